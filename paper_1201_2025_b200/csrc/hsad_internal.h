// Internal helpers shared by the hsad B200 translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "hsad_gpu.h"

namespace hsad_b200 {

// Thread-local "<Name>: message" of the last failure (error.hpp:36-45 format).
hsad_status set_error(hsad_status code, const std::string& message);
const char* status_name(int32_t code);

// Maps a CUDA runtime failure to HSAD_E_CUDA with the CUDA error text.
hsad_status cuda_fail(cudaError_t e, const char* what);

// Stream-ordered scratch (status words, flags, temporaries) comes from a memory pool
// the library owns per device (release threshold: keep), so repeated calls do not
// remap pages and the process's default pool is left untouched (api.cu).
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);
void scratch_free(void* p, cudaStream_t s);
// Frees one scratch allocation on every return path.
struct ScratchGuard {
    cudaStream_t s;
    void* p;
    explicit ScratchGuard(cudaStream_t st, void* q = nullptr) : s(st), p(q) {}
    ScratchGuard(const ScratchGuard&) = delete;
    ScratchGuard& operator=(const ScratchGuard&) = delete;
    ~ScratchGuard() {
        if (p) scratch_free(p, s);
    }
};

#define HSAD_CUDA_TRY(expr)                                              \
    do {                                                                 \
        cudaError_t e__ = (expr);                                        \
        if (e__ != cudaSuccess) return ::hsad_b200::cuda_fail(e__, #expr); \
    } while (0)

#ifdef __CUDACC__
// mbarrier + TMA bulk-copy (cp.async.bulk) helpers shared by the reduce and detect kernels.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Parity wait; a wait that has not completed after 2^26 polls (seconds) traps, so a
// protocol bug fails the launch instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t polls = 0;; ++polls) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (polls == (1u << 26)) __trap();
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
#endif

// Reflection index, detect.cpp:71-76 (host + device).
__host__ __device__ inline int64_t mirror_index(int64_t i, int64_t n) {
    if (n == 1) return 0;
    const int64_t period = 2 * (n - 1);
    i = i < 0 ? -i : i;
    i %= period;
    return i < n ? i : period - i;
}

// Validation of wavelet parameters exactly as wavelet.cpp:51-56 / 122-167 raise
// them for a pixel of `bands` samples; fills the composed target x bands
// linear map (row-major, fp64) when `map` is non-null.
hsad_status wavelet_plan(int32_t bands, int32_t order, int32_t target, std::vector<double>* map);

hsad_status window_validate(const hsad_window& w);

// Raw ENVI cube helpers (ingest.cu): header + byte-count validation with the reference's
// messages, the NonFiniteValue message for a BIP index, and the asynchronous decode + DWT
// of rows [row0, row1) of a resident BSQ / BIL cube (first non-finite -> *status).
hsad_status validate_raw(const hsad_cube_header& h, int64_t raw_bytes);
hsad_status nonfinite_error(const hsad_cube_header& h, unsigned long long first);
cudaError_t reduce_raw_rows(const hsad_cube_header& h, const void* d_raw, int32_t order, int32_t target,
                            void* d_out, int32_t out_bytes, unsigned long long* status, cudaStream_t s,
                            int64_t row0, int64_t row1);

// Device copy of the composed target x bands wavelet map (cached per thread), reduce.cu.
hsad_status device_wavelet_map(int32_t bands, int32_t order, int32_t target, const double** d_map);

// Full-band (bands > 8) LRX / DWRX request, fullband.cu.
struct FbParams {
    const void* cube;
    int elem_bytes;
    int64_t lines, samples;
    int bands;
    int64_t buf_row0;
    int64_t row_begin, row_end;
    int algo;           // HSAD_LRX, HSAD_DWRX or HSAD_DWEST
    int outer;          // LRX window / DWRX outer
    int inner;          // LRX guard (1 = centre only) / DWRX inner
    double ridge;
    void* scores;
    int score_bytes;
    unsigned long long* status;
    int req;            // position of the request in the call (failure ordering)
    int64_t diag_lin;
    double* diag_out;
    double frac;        // DWEST eigen fraction
    int8_t* eigcount;   // DWEST eigen-count map (nullable)
    int chunk;          // samples per shared-memory chunk (set by fullband_launch)
    int mp;             // bordered dimension L+1 rounded up to a multiple of 4
    // tensor-core route (fullband_tc.cu): the raw window Gram of the shifted samples,
    // [row - gram_row0][col][8x8 tile][8][8], and the per-band shift; null = fp64 FMA Gram
    const double* gram;
    int64_t gram_row0;
    const double* shift;
};

// Packed per-pixel failure word (atomicMin across a call): the request's position in
// the call's request list in bits 56..63, the pixel (row*samples + col) in bits 8..55,
// the hsad_status code in bits 0..6 (bit 7: the "inverse overflowed" variant). The
// minimum is the first failing pixel of the first failing request: what the equivalent
// sequential hsad::detect calls report (detect.cpp:127-130, parallel.hpp:17-40).
constexpr unsigned long long kFailPixelMask = (1ull << 48) - 1;
__host__ __device__ inline unsigned long long pack_failure(int req, int64_t lin, int code) {
    return (static_cast<unsigned long long>(req) << 56) |
           ((static_cast<unsigned long long>(lin) & kFailPixelMask) << 8) |
           static_cast<unsigned long long>(code & 0xff);
}
inline int64_t failure_pixel(unsigned long long w) { return static_cast<int64_t>((w >> 8) & kFailPixelMask); }
inline int failure_request(unsigned long long w) { return static_cast<int>(w >> 56); }
inline int failure_code(unsigned long long w) { return static_cast<int>(w & 0x7f); }

// Kernel-side limits.
constexpr int kMaxDetectBands = 8;
constexpr int kMaxBoxes = 4;
constexpr int kMaxRequests = 4;       // per fused detector launch
constexpr int kMaxCallRequests = 16;  // per hsad_detect_multi / hsad_pipeline_host call
constexpr int kMaxRadius = 112;  // window edge <= 225 (block of 256 columns)
constexpr int kMaxReduceBands = 4096;

}  // namespace hsad_b200
