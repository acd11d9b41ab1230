// ENVI ingest on the device: hsad::read_cube (proj/core/src/cube.cpp:198-253).
//
// The reference decodes a raw ENVI cube element by element on the host: validate
// the header (cube.cpp:22-45), check the byte count, then for every (row, col,
// band) in that order read the source element from its interleave position
// (BSQ band*plane + row*samples + col, BIL (row*bands + band)*samples + col, BIP
// (row*samples + col)*bands + band), byte-swap if the file's byte order differs
// from the host's, widen to fp64 and reject non-finite values.
//
// Here the raw file bytes are already in HBM and the whole decode is one
// HBM-bound pass:
//   * BSQ and BIL are batched (bands x columns) -> (columns x bands) transposes
//     (BSQ: one batch of lines*samples columns; BIL: one batch per line), moved
//     through 32 x 32 shared-memory tiles so both the band-plane reads and the
//     BIP writes are coalesced;
//   * BIP is a streaming element-wise decode;
//   * typed, naturally aligned loads (u8/i16/u16/f32/f64), byte swap in
//     registers (PRMT), widen to the output type (fp64 = the reference's
//     HyperCube, or fp32 for sources fp32 holds exactly);
//   * a non-finite value records its BIP linear index with atomicMin, so the
//     error names the first one in the reference's (row, col, band) loop order.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "hsad_internal.h"

namespace hsad_b200 {
namespace {

template <int CODE>
struct Src;
template <> struct Src<1> { using T = uint8_t; };
template <> struct Src<2> { using T = uint16_t; };   // int16 bits
template <> struct Src<4> { using T = uint32_t; };   // float bits
template <> struct Src<5> { using T = uint64_t; };   // double bits
template <> struct Src<12> { using T = uint16_t; };

__device__ __forceinline__ uint16_t bswap16(uint16_t v) {
    return static_cast<uint16_t>(__byte_perm(v, 0, 0x3201) & 0xffffu);
}
__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }
__device__ __forceinline__ uint64_t bswap64(uint64_t v) {
    const uint32_t lo = static_cast<uint32_t>(v), hi = static_cast<uint32_t>(v >> 32);
    return (static_cast<uint64_t>(bswap32(lo)) << 32) | bswap32(hi);
}

// widen<T>(p, swap), cube.cpp:214-224
template <int CODE>
__device__ __forceinline__ double decode(typename Src<CODE>::T raw, bool swap) {
    if constexpr (CODE == 1) {
        return static_cast<double>(raw);
    } else if constexpr (CODE == 2) {
        return static_cast<double>(static_cast<int16_t>(swap ? bswap16(raw) : raw));
    } else if constexpr (CODE == 12) {
        return static_cast<double>(swap ? bswap16(raw) : raw);
    } else if constexpr (CODE == 4) {
        return static_cast<double>(__uint_as_float(swap ? bswap32(raw) : raw));
    } else {
        return __longlong_as_double(static_cast<long long>(swap ? bswap64(raw) : raw));
    }
}

template <int CODE>
__device__ __forceinline__ void check_finite(double v, int64_t bip_index, unsigned long long* status) {
    if constexpr (CODE == 4 || CODE == 5) {
        if (!isfinite(v)) atomicMin(status, static_cast<unsigned long long>(bip_index));
    }
}

constexpr int kTile = 32;
constexpr int kRowsPerPass = 8;

// Batched transpose: in[batch][r][c] (r < R bands, c < C columns) -> out[(batch*C + c)*R + r].
template <int CODE, typename Tout>
__global__ void __launch_bounds__(kTile * kRowsPerPass)
    ingest_transpose_kernel(const typename Src<CODE>::T* __restrict__ in, bool swap, int R, int64_t C,
                            Tout* __restrict__ out, unsigned long long* status) {
    __shared__ Tout tile[kTile][kTile + 1];
    const int64_t batch = blockIdx.z;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kTile;
    const int r0 = blockIdx.y * kTile;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const typename Src<CODE>::T* src = in + batch * R * C;
    // load: lanes along columns (contiguous in BSQ planes / BIL lines)
#pragma unroll
    for (int k = 0; k < kTile; k += kRowsPerPass) {
        const int r = r0 + ty + k;
        const int64_t c = c0 + tx;
        if (r < R && c < C) {
            const double v = decode<CODE>(__ldg(src + static_cast<int64_t>(r) * C + c), swap);
            check_finite<CODE>(v, (batch * C + c) * R + r, status);
            tile[ty + k][tx] = static_cast<Tout>(v);
        }
    }
    __syncthreads();
    // store: lanes along bands (contiguous in BIP)
#pragma unroll
    for (int k = 0; k < kTile; k += kRowsPerPass) {
        const int64_t c = c0 + ty + k;
        const int r = r0 + tx;
        if (r < R && c < C) out[(batch * C + c) * R + r] = tile[tx][ty + k];
    }
}

// Whole-spectrum tiles: one CTA moves PIX consecutive columns x all R bands, so the
// BIP output of the tile is one contiguous R*PIX run (fully coalesced writes) and
// every band row is read as one PIX-column segment (128 B for u8..f32 sources at
// PIX = 32). Loads are issued U bands at a time per warp so enough bytes are in
// flight to cover HBM latency. Used when the tile fits in shared memory.
constexpr int kWideThreads = 256;
constexpr int kWideWarps = kWideThreads / 32;
template <typename Tout>
__host__ __device__ constexpr int wide_pix() { return sizeof(Tout) == 4 ? 64 : 32; }
template <int CODE, typename Tout>
__global__ void __launch_bounds__(kWideThreads)
    ingest_wide_kernel(const typename Src<CODE>::T* __restrict__ in, bool swap, int R, int64_t C,
                       Tout* __restrict__ out, unsigned long long* status) {
    using T = typename Src<CODE>::T;
    constexpr int PIX = wide_pix<Tout>();
    constexpr int CPL = PIX / 32;  // columns per lane
    constexpr int U = sizeof(Tout) == 4 ? 8 : 14;  // band rows in flight per warp (measured)
    extern __shared__ __align__(16) unsigned char s_raw[];
    Tout* tile = reinterpret_cast<Tout*>(s_raw);  // [PIX][R + 1]
    const int stride = R + 1;
    const int64_t batch = blockIdx.y;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * PIX;
    const int ncol = static_cast<int>(C - c0 < PIX ? C - c0 : PIX);
    const T* src = in + batch * R * C + c0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int b0 = warp; b0 < R; b0 += kWideWarps * U) {
        T raw[U][CPL];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
                const int b = b0 + u * kWideWarps, c = lane + 32 * j;
                raw[u][j] = (b < R && c < ncol) ? __ldg(src + static_cast<int64_t>(b) * C + c) : T(0);
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
                const int b = b0 + u * kWideWarps, c = lane + 32 * j;
                if (b < R && c < ncol) {
                    const double v = decode<CODE>(raw[u][j], swap);
                    check_finite<CODE>(v, (batch * C + c0 + c) * R + b, status);
                    tile[c * stride + b] = static_cast<Tout>(v);
                }
            }
    }
    __syncthreads();
    // store: the tile's BIP run [(batch*C + c0) * R, + ncol * R) in order
    Tout* dst = out + (batch * C + c0) * R;
    const int total = ncol * R;
    int c = threadIdx.x / R, b = threadIdx.x % R;
    const int dc = kWideThreads / R, db = kWideThreads % R;
    for (int i = threadIdx.x; i < total; i += kWideThreads) {
        dst[i] = tile[c * stride + b];
        c += dc;
        b += db;
        if (b >= R) {
            b -= R;
            ++c;
        }
    }
}

// BIP source: element-wise decode (grid-stride)
template <int CODE, typename Tout>
__global__ void ingest_bip_kernel(const typename Src<CODE>::T* __restrict__ in, bool swap, int64_t n,
                                  Tout* __restrict__ out, unsigned long long* status) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = decode<CODE>(__ldg(in + i), swap);
        check_finite<CODE>(v, i, status);
        out[i] = static_cast<Tout>(v);
    }
}

template <int CODE, typename Tout>
cudaError_t launch_ingest(const hsad_cube_header& h, const void* raw, bool swap, void* out,
                          unsigned long long* status, cudaStream_t s) {
    using T = typename Src<CODE>::T;
    const T* in = static_cast<const T*>(raw);
    Tout* o = static_cast<Tout*>(out);
    const int64_t plane = static_cast<int64_t>(h.lines) * h.samples;
    if (h.interleave == HSAD_BIP) {
        const int64_t n = plane * h.bands;
        const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
        ingest_bip_kernel<CODE, Tout><<<static_cast<unsigned>(blocks), 256, 0, s>>>(in, swap, n, o, status);
        return cudaGetLastError();
    }
    const int64_t batches = h.interleave == HSAD_BSQ ? 1 : h.lines;
    const int64_t C = h.interleave == HSAD_BSQ ? plane : h.samples;
    const size_t wide_smem = static_cast<size_t>(wide_pix<Tout>()) * (h.bands + 1) * sizeof(Tout);
    if (wide_smem <= 100 * 1024 && batches <= 65535) {
        auto kern = ingest_wide_kernel<CODE, Tout>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(wide_smem));
        if (e != cudaSuccess) return e;
        const dim3 g(static_cast<unsigned>((C + wide_pix<Tout>() - 1) / wide_pix<Tout>()),
                     static_cast<unsigned>(batches));
        kern<<<g, kWideThreads, wide_smem, s>>>(in, swap, h.bands, C, o, status);
        return cudaGetLastError();
    }
    const dim3 grid(static_cast<unsigned>((C + kTile - 1) / kTile),
                    static_cast<unsigned>((h.bands + kTile - 1) / kTile), static_cast<unsigned>(batches));
    if (grid.y > 65535 || grid.z > 65535) return cudaErrorInvalidConfiguration;
    ingest_transpose_kernel<CODE, Tout><<<grid, dim3(kTile, kRowsPerPass), 0, s>>>(in, swap, h.bands, C, o,
                                                                                  status);
    return cudaGetLastError();
}

template <typename Tout>
cudaError_t dispatch_code(const hsad_cube_header& h, const void* raw, bool swap, void* out,
                          unsigned long long* status, cudaStream_t s) {
    switch (h.data_type_code) {
        case 1: return launch_ingest<1, Tout>(h, raw, swap, out, status, s);
        case 2: return launch_ingest<2, Tout>(h, raw, swap, out, status, s);
        case 4: return launch_ingest<4, Tout>(h, raw, swap, out, status, s);
        case 5: return launch_ingest<5, Tout>(h, raw, swap, out, status, s);
        case 12: return launch_ingest<12, Tout>(h, raw, swap, out, status, s);
    }
    return cudaErrorInvalidValue;
}

// ---- fused decode + DWT straight from a raw BSQ / BIL file (read_cube then reduce_cube)
// One CTA = 128 consecutive columns of one batch (BSQ: the whole plane, BIL: one line);
// 4 band groups of 64 threads stream their bands (each thread 2 columns 64 apart: warp
// loads are 32 consecutive columns of one band, coalesced in BSQ/BIL; 16 loads in flight
// per thread), apply the composed target x bands map (shared memory) and combine their
// partial sums in a fixed order into one contiguous BIP run. The BIP fp32/fp64
// intermediate of read_cube is never written.
constexpr int kRawThreads = 64;  // columns per group; each thread owns kRawPPT columns
constexpr int kRawPPT = 2;
constexpr int kRawPix = kRawThreads * kRawPPT;  // columns per CTA
constexpr int kRawGroups = 4;                   // band groups per CTA
template <int CODE, int TARGET>
__global__ void __launch_bounds__(kRawThreads * kRawGroups)
    reduce_raw_kernel(const typename Src<CODE>::T* __restrict__ in, bool swap, int R, int64_t C,
                      int64_t batch0, int64_t c_begin, int64_t c_end,
                      const double* __restrict__ wmap, void* __restrict__ out, int out_bytes,
                      unsigned long long* status) {
    using T = typename Src<CODE>::T;
    extern __shared__ double s_dyn[];
    double* s_w = s_dyn;                                          // [TARGET][R]
    double* s_part = s_dyn + TARGET * R;                          // [groups][kRawPix][TARGET]
    for (int i = threadIdx.x; i < TARGET * R; i += blockDim.x) s_w[i] = wmap[i];
    __syncthreads();
    const int tx = threadIdx.x % kRawThreads, g = threadIdx.x / kRawThreads;
    const int64_t batch = batch0 + blockIdx.y;
    const int64_t cbase = c_begin + static_cast<int64_t>(blockIdx.x) * kRawPix;
    const T* src = in + batch * R * C + cbase;
    bool live[kRawPPT];
#pragma unroll
    for (int m = 0; m < kRawPPT; ++m) live[m] = cbase + tx + m * kRawThreads < c_end;
    double acc[kRawPPT][TARGET];
#pragma unroll
    for (int m = 0; m < kRawPPT; ++m)
#pragma unroll
        for (int j = 0; j < TARGET; ++j) acc[m][j] = 0.0;
    constexpr int U = 8;  // band rows in flight per thread (x kRawPPT columns)
    for (int b0 = g; b0 < R; b0 += kRawGroups * U) {
        T raw[U][kRawPPT];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < kRawPPT; ++m) {
                const int b = b0 + u * kRawGroups;
                raw[u][m] = (live[m] && b < R)
                                ? __ldg(src + static_cast<int64_t>(b) * C + tx + m * kRawThreads)
                                : T(0);
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int b = b0 + u * kRawGroups;
            if (b < R) {
#pragma unroll
                for (int m = 0; m < kRawPPT; ++m) {
                    if (!live[m]) continue;
                    const double v = decode<CODE>(raw[u][m], swap);
                    check_finite<CODE>(v, (batch * C + cbase + tx + m * kRawThreads) * R + b, status);
#pragma unroll
                    for (int j = 0; j < TARGET; ++j) acc[m][j] = fma(s_w[j * R + b], v, acc[m][j]);
                }
            }
        }
    }
#pragma unroll
    for (int m = 0; m < kRawPPT; ++m)
#pragma unroll
        for (int j = 0; j < TARGET; ++j)
            s_part[(g * kRawPix + tx + m * kRawThreads) * TARGET + j] = acc[m][j];
    __syncthreads();
    // combine the band groups in a fixed order; the CTA's output run is contiguous
    const int64_t o0 = (batch * C + cbase) * TARGET;
    const int64_t ncols = c_end - cbase < kRawPix ? c_end - cbase : kRawPix;
    for (int i = threadIdx.x; i < ncols * TARGET; i += blockDim.x) {
        const double v = (s_part[i] + s_part[kRawPix * TARGET + i]) +
                         (s_part[2 * kRawPix * TARGET + i] + s_part[3 * kRawPix * TARGET + i]);
        if (out_bytes == 8) static_cast<double*>(out)[o0 + i] = v;
        else static_cast<float*>(out)[o0 + i] = static_cast<float>(v);
    }
}

// rows [row0, row1) of a BSQ / BIL cube whose full raw image is at `raw`; the outputs
// land at their global BIP positions of `out`
template <int CODE>
cudaError_t launch_reduce_raw(const hsad_cube_header& h, const void* raw, bool swap, int target,
                              const double* wmap, void* out, int out_bytes,
                              unsigned long long* status, cudaStream_t s, int64_t row0, int64_t row1) {
    const int64_t plane = static_cast<int64_t>(h.lines) * h.samples;
    const bool bsq = h.interleave == HSAD_BSQ;
    const int64_t C = bsq ? plane : h.samples;
    const int64_t batch0 = bsq ? 0 : row0, batches = bsq ? 1 : row1 - row0;
    const int64_t c_begin = bsq ? row0 * h.samples : 0, c_end = bsq ? row1 * h.samples : h.samples;
    if (batches > 65535) return cudaErrorInvalidConfiguration;
    if (batches <= 0 || c_end <= c_begin) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>((c_end - c_begin + kRawPix - 1) / kRawPix),
                    static_cast<unsigned>(batches));
    const size_t smem = (static_cast<size_t>(target) * h.bands +
                         static_cast<size_t>(kRawGroups) * kRawPix * target) * sizeof(double);
    const auto* in = static_cast<const typename Src<CODE>::T*>(raw);
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        kern<<<grid, kRawThreads * kRawGroups, smem, s>>>(in, swap, h.bands, C, batch0, c_begin, c_end,
                                                          wmap, out, out_bytes, status);
        return cudaGetLastError();
    };
    switch (target) {
        case 1: return go(reduce_raw_kernel<CODE, 1>);
        case 2: return go(reduce_raw_kernel<CODE, 2>);
        case 4: return go(reduce_raw_kernel<CODE, 4>);
        case 8: return go(reduce_raw_kernel<CODE, 8>);
        case 16: return go(reduce_raw_kernel<CODE, 16>);
    }
    return cudaErrorInvalidValue;
}

int64_t element_size(int code) {  // cube.cpp:22-33
    switch (code) {
        case 1: return 1;
        case 2: return 2;
        case 4: return 4;
        case 5: return 8;
        case 12: return 2;
    }
    return 0;
}

}  // namespace
}  // namespace hsad_b200

namespace hsad_b200 {
// Asynchronous decode + DWT of rows [row0, row1) of a resident BSQ / BIL raw cube into the
// matching rows of d_out; the first non-finite element's BIP index goes to *status
// (atomicMin). Used by hsad_reduce_raw and the raw host pipeline.
cudaError_t reduce_raw_rows(const hsad_cube_header& h, const void* d_raw, int32_t order, int32_t target,
                            void* d_out, int32_t out_bytes, unsigned long long* status, cudaStream_t s,
                            int64_t row0, int64_t row1) {
    const double* d_map = nullptr;
    if (device_wavelet_map(h.bands, order, target, &d_map) != HSAD_OK) return cudaErrorInvalidValue;
    const bool swap = h.byte_order == 1;
    switch (h.data_type_code) {
        case 1: return launch_reduce_raw<1>(h, d_raw, swap, target, d_map, d_out, out_bytes, status, s, row0, row1);
        case 2: return launch_reduce_raw<2>(h, d_raw, swap, target, d_map, d_out, out_bytes, status, s, row0, row1);
        case 4: return launch_reduce_raw<4>(h, d_raw, swap, target, d_map, d_out, out_bytes, status, s, row0, row1);
        case 5: return launch_reduce_raw<5>(h, d_raw, swap, target, d_map, d_out, out_bytes, status, s, row0, row1);
        case 12: return launch_reduce_raw<12>(h, d_raw, swap, target, d_map, d_out, out_bytes, status, s, row0, row1);
    }
    return cudaErrorInvalidValue;
}
}  // namespace hsad_b200

namespace hsad_b200 {
// CubeHeader::validate + the byte count (cube.cpp:22-45, 200-203), same order and messages
hsad_status validate_raw(const hsad_cube_header& h, int64_t raw_bytes) {
    if (h.samples < 1 || h.lines < 1 || h.bands < 1)
        return set_error(HSAD_E_INVALID_VALUE, "samples, lines and bands must all be >= 1");
    const int64_t esize = element_size(h.data_type_code);
    if (esize == 0)
        return set_error(HSAD_E_INVALID_VALUE,
                         "unsupported data type code " + std::to_string(h.data_type_code));
    if (h.byte_order != 0 && h.byte_order != 1)
        return set_error(HSAD_E_INVALID_VALUE, "byte order must be 0 or 1");
    if (h.interleave != HSAD_BSQ && h.interleave != HSAD_BIL && h.interleave != HSAD_BIP)
        return set_error(HSAD_E_INVALID_VALUE, "unknown interleave " + std::to_string(h.interleave));
    const int64_t expected = static_cast<int64_t>(h.samples) * h.lines * h.bands * esize;
    if (raw_bytes != expected)
        return set_error(HSAD_E_SIZE_MISMATCH, "raw data is " + std::to_string(raw_bytes) +
                                                   " bytes, header expects " + std::to_string(expected));
    return HSAD_OK;
}

hsad_status nonfinite_error(const hsad_cube_header& h, unsigned long long first) {
    const int64_t band = static_cast<int64_t>(first % h.bands);
    const int64_t pix = static_cast<int64_t>(first / h.bands);
    return set_error(HSAD_E_NON_FINITE_VALUE, "at (row=" + std::to_string(pix / h.samples) +
                                                  ", col=" + std::to_string(pix % h.samples) +
                                                  ", band=" + std::to_string(band) + ")");
}
}  // namespace hsad_b200

using namespace hsad_b200;

extern "C" hsad_status hsad_reduce_raw(const void* d_raw, int64_t raw_bytes, const hsad_cube_header* header,
                                       int32_t order, int32_t target_bands, void* d_out,
                                       int32_t out_bytes, void* stream) {
    if (!header) return set_error(HSAD_E_INVALID_VALUE, "null header");
    const hsad_cube_header& h = *header;
    hsad_status st = validate_raw(h, raw_bytes);
    if (st != HSAD_OK) return st;
    if (out_bytes != 8 && out_bytes != 4)
        return set_error(HSAD_E_INVALID_VALUE, "out_bytes must be 8 (fp64) or 4 (fp32)");
    st = wavelet_plan(h.bands, order, target_bands, nullptr);
    if (st != HSAD_OK) return st;
    if (!d_raw || !d_out) return set_error(HSAD_E_INVALID_VALUE, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (h.interleave == HSAD_BIP) {
        // BIP: decode (read_cube) into a stream-ordered fp64 cube, then the TMA DWT
        void* tmp = nullptr;
        const size_t n = static_cast<size_t>(h.lines) * h.samples * h.bands;
        HSAD_CUDA_TRY(scratch_alloc(&tmp, n * sizeof(double), s));
        ScratchGuard tmp_guard(s, tmp);
        st = hsad_read_cube(d_raw, raw_bytes, &h, tmp, 8, stream);
        if (st == HSAD_OK)
            st = hsad_reduce(tmp, 8, h.lines, h.samples, h.bands, order, target_bands, d_out, out_bytes, stream);
        return st;
    }
    if (target_bands != 1 && target_bands != 2 && target_bands != 4 && target_bands != 8 &&
        target_bands != 16)
        return set_error(HSAD_E_UNSUPPORTED, "raw-cube reduction supports 1..16 target bands");
    const double* d_map = nullptr;
    st = device_wavelet_map(h.bands, order, target_bands, &d_map);  // plan errors before any launch
    if (st != HSAD_OK) return st;
    unsigned long long* status = nullptr;
    HSAD_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&status), sizeof(unsigned long long), s));
    ScratchGuard status_guard(s, status);
    HSAD_CUDA_TRY(cudaMemsetAsync(status, 0xff, sizeof(unsigned long long), s));
    cudaError_t e = reduce_raw_rows(h, d_raw, order, target_bands, d_out, out_bytes, status, s, 0, h.lines);
    unsigned long long first = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&first, status, sizeof(first), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "hsad_reduce_raw");
    if (first != ~0ull) return nonfinite_error(h, first);
    return HSAD_OK;
}

extern "C" hsad_status hsad_read_cube(const void* d_raw, int64_t raw_bytes, const hsad_cube_header* header,
                                      void* d_out, int32_t out_bytes, void* stream) {
    if (!header) return set_error(HSAD_E_INVALID_VALUE, "null header");
    const hsad_cube_header& h = *header;
    hsad_status vst = validate_raw(h, raw_bytes);
    if (vst != HSAD_OK) return vst;
    if (out_bytes != 8 && out_bytes != 4)
        return set_error(HSAD_E_INVALID_VALUE, "out_bytes must be 8 (fp64) or 4 (fp32)");
    if (out_bytes == 4 && h.data_type_code == 5)
        return set_error(HSAD_E_INVALID_VALUE,
                         "an fp32 cube cannot hold an fp64 source exactly; use out_bytes 8");
    if (!d_raw || !d_out) return set_error(HSAD_E_INVALID_VALUE, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // every supported host is little-endian: swap when the file is big-endian (cube.cpp:205)
    const bool swap = h.byte_order == 1;
    unsigned long long* status = nullptr;
    HSAD_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&status), sizeof(unsigned long long), s));
    ScratchGuard status_guard(s, status);
    HSAD_CUDA_TRY(cudaMemsetAsync(status, 0xff, sizeof(unsigned long long), s));
    cudaError_t e = out_bytes == 8 ? dispatch_code<double>(h, d_raw, swap, d_out, status, s)
                                   : dispatch_code<float>(h, d_raw, swap, d_out, status, s);
    unsigned long long first = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&first, status, sizeof(first), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "hsad_read_cube");
    if (first != ~0ull) return nonfinite_error(h, first);  // cube.cpp:244-247
    return HSAD_OK;
}
