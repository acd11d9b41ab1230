// K1: per-pixel Daubechies reduction of a BIP cube to `target` approximation
// bands (hsad::reduce_cube, proj/core/src/wavelet.cpp:148-167).
//
// The reference pads each spectrum by half-sample mirroring to P = bit_ceil(L)
// and runs log2(P/target) periodic low-pass stages (wavelet.cpp:122-146). That
// cascade is one fixed linear map W (target x L); the host composes it in fp64
// from the same taps and padding rule (api.cu: wavelet_plan), so the kernel is a
// streaming [pixels x L] . [L x target] product in fp64 — ~4 DFMA per input
// element (fewer than the cascade's 2016/189 per element) and HBM-bound.
//
// Layout / mapping (lane-split warp):
//   * a warp owns a group of G = 32/target consecutive pixels; lane l reads bands
//     l, l+32, l+64, ... of each pixel, so every load instruction is a contiguous
//     128 B run of the BIP row (coalesced, no shared memory, no bank conflicts);
//   * lane l keeps its slice of W (target x BPL doubles) in registers;
//   * after the G pixels each lane holds 32 partial sums; a butterfly
//     reduce-scatter over the warp (31 64-bit shuffles) leaves lane l with the
//     total of output (pixel l/target, band l%target), so the store is one
//     contiguous 32 x 8 B run.
// Input fp32 (widened exactly) or fp64; output fp64 or fp32.
#include <cstdint>
#include <vector>

#include "hsad_internal.h"

namespace hsad_b200 {
namespace {

constexpr int kWarps = 8;  // warps per CTA

template <typename T>
__device__ __forceinline__ double load_widen(const T* p) {
    return static_cast<double>(__ldg(p));
}

template <typename Tin, int TARGET, int BPL>
__global__ void __launch_bounds__(kWarps * 32)
    reduce_lanesplit_kernel(const Tin* __restrict__ cube, int64_t npix, int bands,
                            const double* __restrict__ wmap, void* __restrict__ out, int out_bytes) {
    constexpr int G = 32 / TARGET;  // pixels per reduce group
    const int lane = threadIdx.x & 31;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kWarps) + (threadIdx.x >> 5);
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;

    double w[BPL][TARGET];
#pragma unroll
    for (int s = 0; s < BPL; ++s) {
        const int b = lane + 32 * s;
#pragma unroll
        for (int k = 0; k < TARGET; ++k) w[s][k] = b < bands ? wmap[k * bands + b] : 0.0;
    }

    const int64_t ngroups = (npix + G - 1) / G;
    for (int64_t g = warp; g < ngroups; g += nwarps) {
        const int64_t p0 = g * G;
        double v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int64_t p = p0 + j;
            const bool pin = p < npix;
            const Tin* px = cube + p * bands;
            double x[BPL];
#pragma unroll
            for (int s = 0; s < BPL; ++s) {
                const int b = lane + 32 * s;
                x[s] = (pin && b < bands) ? load_widen(px + b) : 0.0;
            }
#pragma unroll
            for (int s = 0; s < BPL; ++s)
#pragma unroll
                for (int k = 0; k < TARGET; ++k) v[j * TARGET + k] = fma(w[s][k], x[s], v[j * TARGET + k]);
        }
        // butterfly reduce-scatter: lane l ends with the warp total of v[l]
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o; ++i) {
                const double send = upper ? v[i] : v[i + o];
                const double keep = upper ? v[i + o] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        const int64_t p = p0 + lane / TARGET;
        if (p < npix) {
            const int64_t o = p0 * TARGET + lane;
            if (out_bytes == 8) static_cast<double*>(out)[o] = v[0];
            else static_cast<float*>(out)[o] = static_cast<float>(v[0]);
        }
    }
}

// ---------------------------------------------------------------------------
// Bulk-staged variant (the default path). A persistent CTA of 8 warps streams
// contiguous tiles of P pixels (P*L*elem bytes, one TMA bulk copy each) through
// a 3-stage shared-memory ring guarded by mbarriers, so ~2 tiles (>100 KB) per SM
// are always in flight regardless of register pressure. Warps consume a stage
// exactly like the lane-split kernel, reading the spectra from shared memory
// (lane l reads band l + 32 s: consecutive words, conflict-free for any L).
constexpr int kStages = 3;

template <typename Tin, int TARGET, int BPL>
__global__ void __launch_bounds__(kWarps * 32, 1)
    reduce_bulk_kernel(const Tin* __restrict__ cube, int64_t npix, int bands, int tile_px,
                       const double* __restrict__ wmap, void* __restrict__ out, int out_bytes) {
    constexpr int G = 32 / TARGET;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
    Tin* stage0 = reinterpret_cast<Tin*>(smem_raw + 128);
    const int64_t stage_elems = static_cast<int64_t>(tile_px) * bands;
    const uint32_t tile_bytes = static_cast<uint32_t>(stage_elems * sizeof(Tin));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    double w[BPL][TARGET];
#pragma unroll
    for (int s = 0; s < BPL; ++s) {
        const int b = lane + 32 * s;
#pragma unroll
        for (int k = 0; k < TARGET; ++k) w[s][k] = b < bands ? wmap[k * bands + b] : 0.0;
    }

    const int64_t full_tiles = npix / tile_px;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            const int64_t t = blockIdx.x + static_cast<int64_t>(s) * gridDim.x;
            if (t < full_tiles) {
                mbar_expect_tx(&bars[s], tile_bytes);
                bulk_g2s(stage0 + s * stage_elems, cube + t * stage_elems, tile_bytes, &bars[s]);
            }
        }
    }
    const int groups = tile_px / G;
    int64_t k = 0;
    for (int64_t t = blockIdx.x; t < full_tiles; t += gridDim.x, ++k) {
        const int s = static_cast<int>(k % kStages);
        mbar_wait(&bars[s], static_cast<uint32_t>((k / kStages) & 1));
        const Tin* tile = stage0 + s * stage_elems;
        for (int gi = warp; gi < groups; gi += kWarps) {
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const Tin* px = tile + static_cast<int64_t>(gi * G + j) * bands;
                double x[BPL];
#pragma unroll
                for (int s2 = 0; s2 < BPL; ++s2) {
                    const int b = lane + 32 * s2;
                    x[s2] = b < bands ? static_cast<double>(px[b]) : 0.0;
                }
#pragma unroll
                for (int s2 = 0; s2 < BPL; ++s2)
#pragma unroll
                    for (int kk = 0; kk < TARGET; ++kk)
                        v[j * TARGET + kk] = fma(w[s2][kk], x[s2], v[j * TARGET + kk]);
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const bool upper = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < o; ++i) {
                    const double send = upper ? v[i] : v[i + o];
                    const double keep = upper ? v[i + o] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            const int64_t oidx = (t * tile_px + gi * G) * TARGET + lane;
            if (out_bytes == 8) static_cast<double*>(out)[oidx] = v[0];
            else static_cast<float*>(out)[oidx] = static_cast<float>(v[0]);
        }
        __syncthreads();  // every warp is done with stage s
        if (threadIdx.x == 0) {
            const int64_t tn = t + static_cast<int64_t>(kStages) * gridDim.x;
            if (tn < full_tiles) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bars[s], tile_bytes);
                bulk_g2s(stage0 + s * stage_elems, cube + tn * stage_elems, tile_bytes, &bars[s]);
            }
        }
    }
}

// Fallback for targets > 8 or very long spectra: one thread per output value.
template <typename Tin>
__global__ void reduce_generic_kernel(const Tin* __restrict__ cube, int64_t npix, int bands,
                                      int target, const double* __restrict__ wmap,
                                      void* __restrict__ out, int out_bytes) {
    const int64_t total = npix * target;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t p = i / target;
        const int k = static_cast<int>(i % target);
        const Tin* px = cube + p * bands;
        const double* wk = wmap + static_cast<int64_t>(k) * bands;
        double acc = 0.0;
        for (int b = 0; b < bands; ++b) acc = fma(wk[b], load_widen(px + b), acc);
        if (out_bytes == 8) static_cast<double*>(out)[i] = acc;
        else static_cast<float*>(out)[i] = static_cast<float>(acc);
    }
}

int grid_for(int64_t work_items, int per_block) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (work_items + per_block - 1) / per_block;
    const int64_t cap = static_cast<int64_t>(sms) * 8;
    return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

int device_sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Pixels per bulk tile: a multiple of 32 (so every warp group is full and the
// tile start stays 16-byte aligned for any band count) with <= 64 KB per stage.
int bulk_tile_px(int bands, int elem) {
    int px = 64;
    while (px > 32 && static_cast<int64_t>(px) * bands * elem > 64 * 1024) px /= 2;
    if (static_cast<int64_t>(px) * bands * elem > 64 * 1024) return 0;
    return px;
}

template <typename Tin, int TARGET, int B>
cudaError_t launch_tb(const Tin* cube, int64_t npix, int bands, const double* wmap, void* out,
                      int out_bytes, cudaStream_t s) {
    constexpr int G = 32 / TARGET;
    const int tile = bulk_tile_px(bands, sizeof(Tin));
    // cp.async.bulk needs a 16-byte aligned source: a cube (or a row strip of one) whose
    // base is not, starts the bulk path at the first pixel that is, and the lane-split
    // kernel (same arithmetic, bit-identical) takes the leading pixels
    int64_t lead = -1;
    const uintptr_t pix_bytes = static_cast<uintptr_t>(bands) * sizeof(Tin);
    for (int64_t p = 0; p < 16 && p < npix; ++p)
        if ((reinterpret_cast<uintptr_t>(cube) + p * pix_bytes) % 16 == 0) {
            lead = p;
            break;
        }
    if (lead > 0) {
        const int grid = grid_for((lead + G - 1) / G, kWarps);
        reduce_lanesplit_kernel<Tin, TARGET, B><<<grid, kWarps * 32, 0, s>>>(
            cube, lead, bands, wmap, out, out_bytes);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        cube += lead * bands;
        out = static_cast<char*>(out) + lead * TARGET * out_bytes;
        npix -= lead;
    }
    int64_t done = 0;
    if (lead >= 0 && tile > 0 && npix >= tile) {
        const int64_t tiles = npix / tile;
        const size_t smem = 128 + static_cast<size_t>(kStages) * tile * bands * sizeof(Tin);
        auto k = reduce_bulk_kernel<Tin, TARGET, B>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const int64_t sms = device_sm_count();
        const int grid = static_cast<int>(tiles < sms ? tiles : sms);
        k<<<grid, kWarps * 32, smem, s>>>(cube, npix, bands, tile, wmap, out, out_bytes);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        done = tiles * tile;
    }
    if (done < npix) {  // tail (and tiny cubes): direct lane-split loads
        const int64_t rest = npix - done;
        const int grid = grid_for((rest + G - 1) / G, kWarps);
        reduce_lanesplit_kernel<Tin, TARGET, B><<<grid, kWarps * 32, 0, s>>>(
            cube + done * bands, rest, bands, wmap,
            static_cast<char*>(out) + done * TARGET * out_bytes, out_bytes);
        return cudaGetLastError();
    }
    return cudaSuccess;
}

template <typename Tin, int TARGET>
cudaError_t launch_target(const Tin* cube, int64_t npix, int bands, const double* wmap, void* out,
                          int out_bytes, cudaStream_t s) {
    const int bpl = (bands + 31) / 32;
    if (bpl <= 1) return launch_tb<Tin, TARGET, 1>(cube, npix, bands, wmap, out, out_bytes, s);
    if (bpl <= 2) return launch_tb<Tin, TARGET, 2>(cube, npix, bands, wmap, out, out_bytes, s);
    if (bpl <= 4) return launch_tb<Tin, TARGET, 4>(cube, npix, bands, wmap, out, out_bytes, s);
    if (bpl <= 6) return launch_tb<Tin, TARGET, 6>(cube, npix, bands, wmap, out, out_bytes, s);
    if (bpl <= 7) return launch_tb<Tin, TARGET, 7>(cube, npix, bands, wmap, out, out_bytes, s);
    if (bpl <= 8) return launch_tb<Tin, TARGET, 8>(cube, npix, bands, wmap, out, out_bytes, s);
    return cudaErrorInvalidValue;
}

template <typename Tin>
cudaError_t launch_reduce(const Tin* cube, int64_t npix, int bands, int target, const double* wmap,
                          void* out, int out_bytes, cudaStream_t s) {
    if (npix == 0) return cudaSuccess;
    if (bands <= 256) {
        if (target == 2) return launch_target<Tin, 2>(cube, npix, bands, wmap, out, out_bytes, s);
        if (target == 4) return launch_target<Tin, 4>(cube, npix, bands, wmap, out, out_bytes, s);
        if (target == 8) return launch_target<Tin, 8>(cube, npix, bands, wmap, out, out_bytes, s);
    }
    reduce_generic_kernel<Tin><<<grid_for(npix * target, 256), 256, 0, s>>>(
        cube, npix, bands, target, wmap, out, out_bytes);
    return cudaGetLastError();
}

// Per-thread cache of the composed map on the device, keyed by (bands, order, target).
struct MapCache {
    int device = -1, bands = 0, order = 0, target = 0;
    double* d_map = nullptr;
    ~MapCache() {
        if (d_map) cudaFree(d_map);
    }
};
thread_local MapCache g_map;

}  // namespace

hsad_status device_wavelet_map(int32_t bands, int32_t order, int32_t target, const double** d_map) {
    int dev = 0;
    HSAD_CUDA_TRY(cudaGetDevice(&dev));
    if (g_map.d_map && g_map.device == dev && g_map.bands == bands && g_map.order == order &&
        g_map.target == target) {
        *d_map = g_map.d_map;
        return HSAD_OK;
    }
    std::vector<double> map;
    hsad_status st = wavelet_plan(bands, order, target, &map);
    if (st != HSAD_OK) return st;
    if (g_map.d_map) {
        cudaFree(g_map.d_map);
        g_map.d_map = nullptr;
    }
    HSAD_CUDA_TRY(cudaMalloc(&g_map.d_map, map.size() * sizeof(double)));
    HSAD_CUDA_TRY(cudaMemcpy(g_map.d_map, map.data(), map.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
    g_map.device = dev;
    g_map.bands = bands;
    g_map.order = order;
    g_map.target = target;
    *d_map = g_map.d_map;
    return HSAD_OK;
}

}  // namespace hsad_b200

using namespace hsad_b200;

extern "C" hsad_status hsad_reduce(const void* d_cube, int32_t elem_bytes, int64_t lines,
                                   int64_t samples, int32_t bands, int32_t order,
                                   int32_t target_bands, void* d_out, int32_t out_bytes,
                                   void* stream) {
    if (elem_bytes != 4 && elem_bytes != 8)
        return set_error(HSAD_E_INVALID_VALUE, "elem_bytes must be 4 or 8");
    if (out_bytes != 4 && out_bytes != 8)
        return set_error(HSAD_E_INVALID_VALUE, "out_bytes must be 4 or 8");
    if (lines < 0 || samples < 0) return set_error(HSAD_E_INVALID_VALUE, "negative cube extent");
    hsad_status st = wavelet_plan(bands, order, target_bands, nullptr);
    if (st != HSAD_OK) return st;
    const int64_t npix = lines * samples;
    if (npix == 0) return HSAD_OK;
    if (!d_cube || !d_out) return set_error(HSAD_E_INVALID_VALUE, "null buffer");
    const double* d_map = nullptr;
    st = device_wavelet_map(bands, order, target_bands, &d_map);
    if (st != HSAD_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = elem_bytes == 4
                        ? launch_reduce(static_cast<const float*>(d_cube), npix, bands,
                                        target_bands, d_map, d_out, out_bytes, s)
                        : launch_reduce(static_cast<const double*>(d_cube), npix, bands,
                                        target_bands, d_map, d_out, out_bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "hsad_reduce kernel launch");
    return HSAD_OK;
}
