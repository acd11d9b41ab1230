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
#include <cstdlib>
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

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

// DMMA variant (TARGET = 4, fp32 cube): Y[8 px x 8] += X[8 px x 4 bands] . Wt[4 x 8]
// with mma.sync.m8n8k4.f64 (DMMA.8x8x4, the fp64 tensor-core path; columns 4..7 of
// Wt are zero). One warp instruction performs the 8 x 4 x 4 useful MACs that take 4
// DFMA instructions per lane in the lane-split kernel, so the DWT costs ~2x fewer
// issue slots. Fragments (PTX mma.m8n8k4 .f64): lane l holds A[l/4][l%4],
// B[l%4][l/4], D[l/4][2(l%4) .. 2(l%4)+1].
// Staging: one bulk copy per pixel into rows of stride L+4 floats (== 4 mod 32 words
// for L % 32 == 0: the 8 rows of an A fragment hit distinct banks); 3-stage ring.
template <int BANDS_PAD>
__global__ void __launch_bounds__(kWarps * 32, 1)
    reduce_dmma_kernel(const float* __restrict__ cube, int64_t npix, int bands, int tile_px,
                       int stride, const double* __restrict__ wmap, double* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
    float* stage0 = reinterpret_cast<float*>(smem_raw + 128);
    const int stage_floats = tile_px * stride;
    double* s_wt = reinterpret_cast<double*>(stage0 + kStages * stage_floats);  // [BANDS_PAD][4]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < BANDS_PAD * 4; i += kWarps * 32) {
        const int k = i >> 2, n = i & 3;
        s_wt[i] = k < bands ? wmap[n * bands + k] : 0.0;
    }
    const int64_t full_tiles = npix / tile_px;
    const uint32_t row_bytes = static_cast<uint32_t>(bands) * 4;
    const uint32_t tile_bytes = row_bytes * tile_px;
    // warp 0 issues a tile: lane 0 arms the barrier, every lane copies tile_px/32 rows
    auto issue = [&](int s, int64_t t) {
        if (lane == 0) mbar_expect_tx(&bars[s], tile_bytes);
        __syncwarp();
        for (int p = lane; p < tile_px; p += 32)
            bulk_g2s(stage0 + s * stage_floats + p * stride, cube + (t * tile_px + p) * bands,
                     row_bytes, &bars[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0)
        for (int s = 0; s < kStages; ++s) {
            const int64_t t = blockIdx.x + static_cast<int64_t>(s) * gridDim.x;
            if (t < full_tiles) issue(s, t);
        }
    const int m = lane >> 2, kq = lane & 3;
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < full_tiles; t += gridDim.x, ++it) {
        const int s = static_cast<int>(it % kStages);
        mbar_wait(&bars[s], static_cast<uint32_t>((it / kStages) & 1));
        const float* tile = stage0 + s * stage_floats;
        for (int gi = warp; gi < tile_px / 8; gi += kWarps) {
            const float* arow = tile + (gi * 8 + m) * stride + kq;
            // four independent accumulator chains (k-steps round-robin) hide DMMA latency
            double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
            for (int k0 = 0; k0 < bands; k0 += 16) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int kk = k0 + 4 * c;
                    const double a = kk + kq < bands ? static_cast<double>(arow[kk]) : 0.0;
                    const double b = (m < 4 && kk < BANDS_PAD) ? s_wt[(kk + kq) * 4 + m] : 0.0;
                    asm volatile(
                        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                        : "+d"(d[c][0]), "+d"(d[c][1])
                        : "d"(a), "d"(b));
                }
            }
            const double d0 = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
            const double d1 = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
            if (kq < 2) {
                const int64_t p = t * tile_px + gi * 8 + m;
                reinterpret_cast<double2*>(out)[p * 2 + kq] = make_double2(d0, d1);
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int64_t tn = t + static_cast<int64_t>(kStages) * gridDim.x;
            if (tn < full_tiles) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(s, tn);
            }
        }
    }
}

// DMMA reduction, register-direct. For a group of 8 pixels and a block of 16 bands
// [k0, k0+16), lane l = (m = l/4, q = l%4) loads x[p0+m][k0+4q .. k0+4q+3] with one
// coalesced float4 (the 8 rows x 64 contiguous bytes of the block) and feeds MMA j
// (j = 0..3) with A[m][q] = x[m][k0+4q+j]: inside each MMA the K index q stands for
// band k0+4q+j, the same for every row, so B[q][n] = W[n][k0+4q+j] (from shared
// memory, padded stride 5 -> conflict-free). Four accumulator chains (one per j).
// Bands must be a multiple of 16 (the fp32 rows stay 16-byte aligned).
__global__ void __launch_bounds__(256)
    reduce_dmma16_kernel(const float* __restrict__ cube, int64_t npix, int bands,
                         const double* __restrict__ wmap, double* __restrict__ out) {
    extern __shared__ double s_wt[];  // [bands][5]
    for (int i = threadIdx.x; i < bands * 4; i += blockDim.x) {
        const int n = i / bands, k = i % bands;
        s_wt[k * 5 + n] = wmap[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int m = lane >> 2, q = lane & 3;
    const int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t groups = npix / 8;
    for (int64_t g = warp; g < groups; g += nwarps) {
        const float4* row = reinterpret_cast<const float4*>(cube + (g * 8 + m) * bands) + q;
        double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 2
        for (int k0 = 0; k0 < bands; k0 += 16) {
            const float4 x4 = __ldg(row + (k0 >> 2));
            const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
            const double* wrow = s_wt + (k0 + 4 * q) * 5 + m;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double a = static_cast<double>(xs[j]);
                const double b = m < 4 ? wrow[j * 5] : 0.0;
                asm volatile(
                    "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(d[j][0]), "+d"(d[j][1])
                    : "d"(a), "d"(b));
            }
        }
        if (q < 2) {
            const double d0 = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
            const double d1 = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
            reinterpret_cast<double2*>(out)[(g * 8 + m) * 2 + q] = make_double2(d0, d1);
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
    int64_t done = 0;
    if (tile > 0 && npix >= tile) {
        const int64_t tiles = npix / tile;
        const size_t smem = 128 + static_cast<size_t>(kStages) * tile * bands * sizeof(Tin);
        auto k = reduce_bulk_kernel<Tin, TARGET, B>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        int64_t sms = device_sm_count();
        if (getenv("HSAD_REDUCE_GRID")) sms = atoi(getenv("HSAD_REDUCE_GRID"));  // probe only
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

// DMMA reduction: fp32 cube, 4 targets, fp64 output, bands a multiple of 4 (per-pixel
// 16-byte bulk copies). Returns cudaErrorNotSupported for other shapes.
cudaError_t launch_reduce_dmma(const float* cube, int64_t npix, int bands, const double* wmap,
                               double* out, cudaStream_t s) {
    if (bands % 16 == 0 && getenv("HSAD_REDUCE_DMMA16")) {
        const int64_t groups = npix / 8;
        int64_t done = 0;
        if (groups > 0) {
            const size_t smem = static_cast<size_t>(bands) * 5 * sizeof(double);
            cudaError_t e = cudaFuncSetAttribute(reduce_dmma16_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            const int grid = device_sm_count() * 8;
            reduce_dmma16_kernel<<<grid, 256, smem, s>>>(cube, npix, bands, wmap, out);
            e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            done = groups * 8;
        }
        if (done < npix) return launch_target<float, 4>(cube + done * bands, npix - done, bands,
                                                        wmap, out + done * 4, 8, s);
        return cudaSuccess;
    }
    if (bands % 4 != 0 || bands > 256) return cudaErrorNotSupported;
    const int tile = 64;
    const int stride = bands + 4;
    int64_t done = 0;
    if (npix >= tile) {
        const int64_t tiles = npix / tile;
        const size_t smem = 128 + static_cast<size_t>(kStages) * tile * stride * sizeof(float) +
                            static_cast<size_t>(256) * 4 * sizeof(double);
        auto k = reduce_dmma_kernel<256>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const int64_t sms = device_sm_count();
        const int grid = static_cast<int>(tiles < sms ? tiles : sms);
        k<<<grid, kWarps * 32, smem, s>>>(cube, npix, bands, tile, stride, wmap, out);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        done = tiles * tile;
    }
    if (done < npix) return launch_target<float, 4>(cube + done * bands, npix - done, bands, wmap,
                                                    out + done * 4, 8, s);
    return cudaSuccess;
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
    if (getenv("HSAD_REDUCE_DMMA") && elem_bytes == 4 && target_bands == 4 && out_bytes == 8) {
        cudaError_t e = launch_reduce_dmma(static_cast<const float*>(d_cube), npix, bands, d_map,
                                           static_cast<double*>(d_out), s);
        if (e == cudaSuccess) return HSAD_OK;
        if (e != cudaErrorNotSupported) return cuda_fail(e, "hsad_reduce dmma launch");
    }
    cudaError_t e = elem_bytes == 4
                        ? launch_reduce(static_cast<const float*>(d_cube), npix, bands,
                                        target_bands, d_map, d_out, out_bytes, s)
                        : launch_reduce(static_cast<const double*>(d_cube), npix, bands,
                                        target_bands, d_map, d_out, out_bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "hsad_reduce kernel launch");
    return HSAD_OK;
}
