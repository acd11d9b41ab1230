// K5t: the full-band window Gram on the 5th-generation tensor cores (tcgen05, kind::i8).
//
// hsad::covariance at L = 189 (proj/core/src/stats.cpp:13-29) is the one dense contraction
// of the path: per pixel C = (1/N) sum_k (x_k - mu)(x_k - mu)^T over the N window samples.
// tcgen05 has no fp64 kind, so the contraction runs as an error-free integer product
// (Ozaki split):
//   1. a per-band shift s_b (the buffer's mean spectrum rounded to fp32) and a power-of-two
//      unit u_b = 2^E_b turn every sample into a 55-bit fixed-point integer
//      q = rint((x - s_b) / u_b), exact for fp32 cubes of ordinary dynamic range; q is cut
//      into 8 balanced base-128 digits d_0..d_7 in [-64, 63] (slices, int8);
//   2. for a pixel pair of bands, sum_k q_i q_j = sum_{p,q} 128^(14-p-q) sum_k d_ip d_jq; the
//      36 digit pairs with p + q <= 7 carry everything above 2^-56 of full scale, and each
//      inner sum is an exact int32 MMA accumulation, grouped by g = p + q into 8 TMEM
//      accumulators;
//   3. integer accumulation is exact, so the window Gram SLIDES along an image row without
//      drift: one CTA keeps a 128 x 64 tile of the Gram (8 groups x 64 columns = the SM's
//      whole 512 TMEM columns) and per pixel step feeds only the entering samples and the
//      negated leaving samples (the outer column pair and the guard / inner-box column pair:
//      2W + 2E samples, one K = 32 chunk for the reference's LRX 15) instead of the whole
//      window;
//   4. after each step the tile is read back (tcgen05.ld), the 8 groups are recombined in
//      int64 as hi * 2^28 + lo and stored as that exact (hi, lo) pair of doubles in the
//      8x8-tile order of fullband_reg_kernel. Band L is a constant one, so row L of the Gram
//      is the exact window sum S of every band; fullband_reg_kernel forms
//      C = (N G - S S^T) / N^2 in double-double arithmetic (one rounding, no cancellation
//      against the shift) and runs the Cholesky.
// Operands are MN-major (band-contiguous, the cube's own BIP order), no swizzle: the digit
// array in global memory is [sign][row][col][slice][192 bands] and a chunk is gathered with
// 16-byte cp.async copies straight into the canonical UMMA layout.
#include <cfloat>
#include <cstdlib>

#include "hsad_internal.h"

namespace hsad_b200 {

hsad_status fullband_reg_launch(FbParams& P, cudaStream_t s);  // fullband.cu

namespace {

constexpr int kTcBands = 192;                          // padded bands = bytes per slice row
constexpr int kTcSlices = 8;
constexpr int kTcSampleBytes = kTcSlices * kTcBands;   // 1536 B per pixel and sign
constexpr int kTcThreads = 256;
constexpr int kTcStages = 3;
constexpr int kTcBlk = 576;                 // one 16-band block: 32 samples x 16 B + 64 B (bank spread)
constexpr int kTcASlice = 8 * kTcBlk;       // A: 128 bands per slice
constexpr int kTcBSlice = 4 * kTcBlk;       // B: 64 bands per slice
constexpr int kTcAStage = kTcSlices * kTcASlice;
constexpr int kTcBStage = kTcSlices * kTcBSlice;
constexpr int kTcStage = kTcAStage + kTcBStage;        // 55296 B
constexpr int kTcSmem = kTcStages * kTcStage + 1024;   // > 114 KB: one CTA (512 TMEM columns) per SM
constexpr int kQBits = 54;                             // |q| < 2^54 (balanced 8 x 7-bit digits reach 0.496 * 2^56)

struct TcParams {
    const int8_t* q;        // digits: [2 signs][qrows][samples][8][192] + one zero sample (address of padding copies)
    int64_t neg_off;        // byte offset of the negated copy
    int64_t zero_off;       // byte offset of the all-zero sample
    int lines, samples;
    int qrow0;              // image row of the digit array's first row
    int row_begin;          // first output row of this launch
    int outer, excl;        // window edge W, excluded centred box edge E (0 = none)
    int seg_len, nseg;      // columns per CTA walk
    int ntile;              // 128 x 64 Gram tiles per pixel (lower triangle of mp x mp)
    int tile_ib[6], tile_jb[6];
    int T;                  // mp / 8: 8x8 output tiles per dimension
    double* gram;           // [rows][samples][T (T + 1) / 2][2: hi, lo][8][8] raw Gram of the shifted samples
    const double* unit;     // [192] u_b
    uint32_t lbo, sbo;      // UMMA descriptor strides (bytes)
};

__device__ __forceinline__ int mirror_tc(int i, int n) {
    if (static_cast<unsigned>(i) < static_cast<unsigned>(n)) return i;
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    i = abs(i) % period;
    return i < n ? i : period - i;
}

// ---- per-band statistics of the buffer rows: sum, min, max ---------------------------
__device__ __forceinline__ long long ordered_key(double v) {
    const long long b = __double_as_longlong(v);
    return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
}
__device__ __forceinline__ double key_value(long long k) {
    return __longlong_as_double(k >= 0 ? k : k ^ 0x7fffffffffffffffLL);
}

constexpr int kTcStatBlocks = 296;
struct TcStats {
    double sum[kTcStatBlocks][kTcBands];  // per-block partial sums (summed in block order: deterministic)
    long long kmin[kTcBands], kmax[kTcBands];
};

__global__ void tc_stats_init(TcStats* st) {
    const int b = threadIdx.x;
    st->kmin[b] = 0x7fffffffffffffffLL;
    st->kmax[b] = static_cast<long long>(0x8000000000000000ULL);
}

__global__ void tc_stats_kernel(const void* cube, int elem_bytes, int64_t npix, int bands, TcStats* st) {
    const int b = threadIdx.x;  // 192 threads, one band each (coalesced over the pixel's spectrum)
    if (b >= bands) return;
    const int64_t per = (npix + gridDim.x - 1) / gridDim.x;
    const int64_t p0 = blockIdx.x * per, p1 = min(p0 + per, npix);
    double sum = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
    for (int64_t p = p0; p < p1; ++p) {
        const double v = elem_bytes == 8 ? static_cast<const double*>(cube)[p * bands + b]
                                         : static_cast<double>(static_cast<const float*>(cube)[p * bands + b]);
        sum += v;
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
    }
    st->sum[blockIdx.x][b] = sum;
    if (p0 < p1) {
        atomicMin(&st->kmin[b], ordered_key(mn));
        atomicMax(&st->kmax[b], ordered_key(mx));
    }
}

// shift[b] = the mean rounded to fp32 (so x - shift is exact for an fp32 cube);
// unit[b] = 2^E with max |x - shift| / unit < 2^54
__global__ void tc_stats_final(const TcStats* st, int nblocks, int64_t npix, int bands, double* shift,
                               double* unit) {
    const int b = threadIdx.x;
    double s = 0.0, u = 1.0;
    if (b < bands) {
        double sum = 0.0;
        for (int i = 0; i < nblocks; ++i) sum += st->sum[i][b];
        s = static_cast<double>(static_cast<float>(sum / static_cast<double>(npix)));
        const double bound = fmax(key_value(st->kmax[b]) - s, s - key_value(st->kmin[b]));
        if (bound > 0.0 && bound < DBL_MAX) u = scalbn(1.0, ilogb(bound) + 1 - kQBits);
    } else if (b == bands) {
        u = 0x1p-49;  // the constant-one band: top digit 1, q = 128^7
    }
    shift[b] = s;
    unit[b] = u;
}

// ---- digits: one thread per (pixel, 4 bands) ------------------------------------------
__global__ void tc_slice_kernel(const void* cube, int elem_bytes, int64_t npix, int bands,
                                const double* __restrict__ shift, const double* __restrict__ unit,
                                int8_t* q, int64_t neg_off) {
    const int64_t item = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (item >= npix * (kTcBands / 4)) return;
    const int64_t p = item / (kTcBands / 4);
    const int g = static_cast<int>(item % (kTcBands / 4));
    uint32_t pos[kTcSlices], neg[kTcSlices];
#pragma unroll
    for (int sl = 0; sl < kTcSlices; ++sl) pos[sl] = neg[sl] = 0u;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int b = 4 * g + h;
        long long v = 0;
        if (b < bands) {
            const double x = elem_bytes == 8 ? static_cast<const double*>(cube)[p * bands + b]
                                             : static_cast<double>(static_cast<const float*>(cube)[p * bands + b]);
            const double y = (x - shift[b]) / unit[b];  // power-of-two divisor: exact
            v = __double2ll_rn(y);
        } else if (b == bands) {
            v = 1ll << 49;  // constant one (unit 2^-49): Gram row `bands` = the window sums
        }
#pragma unroll
        for (int sl = kTcSlices - 1; sl >= 0; --sl) {
            const int d = static_cast<int>((v + 64) & 127) - 64;  // balanced digit in [-64, 63]
            v = (v - d) >> 7;
            pos[sl] |= (static_cast<uint32_t>(d) & 0xffu) << (8 * h);
            neg[sl] |= (static_cast<uint32_t>(-d) & 0xffu) << (8 * h);
        }
    }
    int8_t* dst = q + p * kTcSampleBytes + 4 * g;
#pragma unroll
    for (int sl = 0; sl < kTcSlices; ++sl) {
        *reinterpret_cast<uint32_t*>(dst + sl * kTcBands) = pos[sl];
        *reinterpret_cast<uint32_t*>(dst + neg_off + sl * kTcBands) = neg[sl];
    }
}

// ---- tcgen05 helpers --------------------------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SWIZZLE_NONE (layout type 0), descriptor version 1 (sm_100), MN-major canonical layout:
    // 16 contiguous bands x 8 samples (16 B apart) per core matrix; LBO = next 8 samples,
    // SBO = next 16 bands
    return static_cast<uint64_t>((saddr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// kind::i8 instruction descriptor: D = S32, A = B = S8, both MN-major, M = 128, N = 64
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                              ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kIdescI8), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 8 consecutive accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}

// ---- the sliding window Gram ------------------------------------------------------------
__global__ void __launch_bounds__(kTcThreads, 1) tc_gram_kernel(const TcParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ uint64_t s_done[kTcStages];  // MMAs that read a stage have completed
    __shared__ uint32_t s_tmem;
    __shared__ double s_unit[kTcBands];

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int tile = blockIdx.x % P.ntile, seg = blockIdx.x / P.ntile;
    const int ib = P.tile_ib[tile], jb = P.tile_jb[tile];
    const int r = P.row_begin + blockIdx.y;
    const int c_begin = seg * P.seg_len;
    const int c_end = min(c_begin + P.seg_len, P.samples);
    if (c_begin >= c_end) return;
    unsigned char* stage0 = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~static_cast<uintptr_t>(127));

    if (t < kTcBands) s_unit[t] = P.unit[t];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) {
        for (int i = 0; i < kTcStages; ++i) mbar_init(&s_done[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    const int W = P.outer, R = W / 2, E = P.excl, Re = E / 2;
    const int n_init = (W * W + 31) / 32;
    const int n_step = (2 * W + 2 * E + 31) / 32;
    const int total = n_init + (c_end - c_begin - 1) * n_step;

    // this thread's part of a chunk copy: sample k (8 threads per sample), 16-byte pieces
    const int k = t >> 3, sub = t & 7;
    const int a_blocks = min(8, (kTcBands - ib * 128) / 16);  // 16-band blocks of A that exist
    auto issue_copy = [&](int g) {
        // which sample is entry k of chunk g
        int dr = 0, col = 0, sign = 0;  // sign 0: zero sample
        if (g < n_init) {
            const int idx = g * 32 + k;
            if (idx < W * W) {
                dr = idx / W - R;
                const int dc = idx % W - R;
                col = c_begin + dc;
                sign = (E > 0 && abs(dr) <= Re && abs(dc) <= Re) ? 0 : 1;
            }
        } else {
            const int gs = g - n_init;
            const int c = c_begin + 1 + gs / n_step;  // the new centre column
            const int idx = (gs % n_step) * 32 + k;
            if (idx < W) {
                dr = idx - R, col = c + R, sign = 1;                  // entering outer column
            } else if (idx < 2 * W) {
                dr = idx - W - R, col = c - 1 - R, sign = -1;         // leaving outer column
            } else if (idx < 2 * W + E) {
                dr = idx - 2 * W - Re, col = c + Re, sign = -1;       // entering the excluded box
            } else if (idx < 2 * W + 2 * E) {
                dr = idx - 2 * W - E - Re, col = c - 1 - Re, sign = 1;  // leaving the excluded box
            }
        }
        // padding entries copy nothing: cp.async with src-size 0 zero-fills the 16 bytes
        // (a shared all-zero sample in global memory made every SM hit one L2 line)
        const uint32_t nbytes = sign != 0 ? 16u : 0u;
        int64_t off_b = P.zero_off, off_a = P.zero_off;
        if (sign != 0) {
            const int rr = mirror_tc(r + dr, P.lines) - P.qrow0;
            const int cc = mirror_tc(col, P.samples);
            off_b = (static_cast<int64_t>(rr) * P.samples + cc) * kTcSampleBytes;
            off_a = off_b + (sign < 0 ? P.neg_off : 0);
        }
        unsigned char* sa = stage0 + (g % kTcStages) * kTcStage;
        unsigned char* sb = sa + kTcAStage;
        if (sub < a_blocks) {
            const int8_t* src = P.q + off_a + ib * 128 + sub * 16;
            const uint32_t dst = smem_u32(sa + sub * kTcBlk + k * 16);
#pragma unroll
            for (int sl = 0; sl < kTcSlices; ++sl)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + sl * kTcASlice),
                             "l"(src + sl * kTcBands), "r"(nbytes)
                             : "memory");
        }
        {
            const int m = sub & 3, s0 = sub >> 2;
            const int8_t* src = P.q + off_b + jb * 64 + m * 16;
            const uint32_t dst = smem_u32(sb + m * kTcBlk + k * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int sl = s0 + 2 * i;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + sl * kTcBSlice),
                             "l"(src + sl * kTcBands), "r"(nbytes)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    // epilogue geometry: warp quadrant = TMEM lanes, warp half = 32 of the tile's 64 columns
    const int qd = warp & 3, half = warp >> 2;
    const int i_row = ib * 128 + qd * 32 + lane;  // Gram row (band) of this thread
    const int ti = i_row >> 3, a_in = i_row & 7;
    const int ntile_out = P.T * (P.T + 1) / 2;
    const double ui = i_row < kTcBands ? s_unit[i_row] * 0x1p49 : 0.0;  // u_i * 128^7

    issue_copy(0);
    if (total > 1) issue_copy(1);
    for (int g = 0; g < total; ++g) {
        if (g + 1 < total) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core reads
        tc_fence_before();
        __syncthreads();  // chunk g is in shared memory; the previous pixel's TMEM reads are done
        if (t == 0) {
            tc_fence_after();
            const uint32_t sa = smem_u32(stage0 + (g % kTcStages) * kTcStage);
            const uint32_t sb = sa + kTcAStage;
#pragma unroll 1
            for (int p = 0; p < kTcSlices; ++p) {
                const uint64_t ad = umma_desc(sa + p * kTcASlice, P.lbo, P.sbo);
                for (int q = 0; p + q < kTcSlices; ++q) {
                    const uint64_t bd = umma_desc(sb + q * kTcBSlice, P.lbo, P.sbo);
                    umma_i8(tmem + (p + q) * 64, ad, bd, (g > 0 || p > 0) ? 1u : 0u);
                }
            }
            umma_commit(&s_done[g % kTcStages]);
        }
        // refill the stage chunk g - 1 used (its MMAs were issued one iteration ago)
        if (g + 2 < total) {
            if (g >= 1) mbar_wait(&s_done[(g - 1) % kTcStages], ((g - 1) / kTcStages) & 1);
            issue_copy(g + 2);
        }
        const bool pixel_done = g + 1 >= n_init && (g + 1 - n_init) % n_step == 0;
        if (pixel_done) {
            const int c = c_begin + (g + 1 - n_init) / n_step;
            mbar_wait(&s_done[g % kTcStages], (g / kTcStages) & 1);  // every MMA up to chunk g
            tc_fence_after();
            double* out = P.gram + (static_cast<int64_t>(r - P.row_begin) * P.samples + c) * ntile_out * 128;
#pragma unroll 1
            for (int cb = 0; cb < 4; ++cb) {
                const int j0 = jb * 64 + half * 32 + cb * 8;
                const int tk = j0 >> 3;
                int acc[kTcSlices][8];
                const uint32_t taddr = tmem + (static_cast<uint32_t>(qd * 32) << 16) + half * 32 + cb * 8;
#pragma unroll
                for (int gq = 0; gq < kTcSlices; ++gq) tmem_ld8(taddr + gq * 64, acc[gq]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (ti < P.T && tk <= ti) {
                    // sum_g acc_g 128^(7 - g) = hi 2^28 + lo, both exact in int64 and in fp64:
                    // the entry leaves as the unevaluated pair (hi part, lo part), so the
                    // consumer can subtract the mean product before anything is rounded
                    double vh[8], vl[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        long long hi = acc[0][b], lo = acc[4][b];
#pragma unroll
                        for (int gq = 1; gq < 4; ++gq) {
                            hi = hi * 128 + acc[gq][b];
                            lo = lo * 128 + acc[4 + gq][b];
                        }
                        const double uij = __dmul_rn(ui, s_unit[j0 + b]);  // power of two
                        vh[b] = __dmul_rn(__dmul_rn(static_cast<double>(hi), 0x1p28), uij);
                        vl[b] = __dmul_rn(static_cast<double>(lo), uij);
                    }
                    double2* dst = reinterpret_cast<double2*>(out + (ti * (ti + 1) / 2 + tk) * 128 + a_in * 8);
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        dst[b] = make_double2(vh[2 * b], vh[2 * b + 1]);
                        dst[32 + b] = make_double2(vl[2 * b], vl[2 * b + 1]);
                    }
                }
            }
            tc_fence_before();  // the next iteration's barrier orders these reads before its MMAs
        }
    }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

}  // namespace

// The tensor-core route serves LRX / DWRX whose bordered matrix fits the register-tile
// Cholesky (bands + 1 <= 192). It is selected with HSAD_FB_TC=1: its covariance is exact to
// one rounding, so at kappa ~ 1e6 its scores sit as close to the long-double value as the
// reference's own fp64 arithmetic does (C3: 1.4e-9 vs 1.6e-9) but no longer share the
// reference's rounding, and differ from it by up to 2e-9 on ~1% of the C3 pixels; the default
// fp64 FMA Gram sums the reference's products and stays within the plain 1e-9 bar of it.
bool fullband_tc_applies(const FbParams& P) {
    if (env_int("HSAD_FB_TC", 0) == 0) return false;
    if (P.algo != HSAD_LRX && P.algo != HSAD_DWRX) return false;
    if ((P.bands + 1 + 7) / 8 * 8 > kTcBands) return false;
    if (P.lines > INT32_MAX || P.samples > INT32_MAX) return false;
    return true;
}

// Digits of buffer rows [lo, hi] (image rows), then per row batch: tc_gram_kernel ->
// fullband_reg_kernel with the Gram tiles. If `gram_out` is non-null the Cholesky is
// skipped and the raw tiles of rows [row_begin, row_end) plus shift / unit are returned
// (debug / test entry).
hsad_status fullband_tc_launch(FbParams& P, cudaStream_t s, double* gram_out, double* shift_unit_out) {
    const int R = P.outer / 2;
    int64_t lo = P.lines, hi = -1;
    for (int64_t rr = P.row_begin - R; rr <= P.row_end - 1 + R; ++rr) {
        const int64_t m = mirror_index(rr, P.lines);
        lo = m < lo ? m : lo;
        hi = m > hi ? m : hi;
    }
    const int64_t qrows = hi - lo + 1;
    const int64_t npix = qrows * P.samples;
    const int64_t neg_off = npix * kTcSampleBytes;
    const int64_t zero_off = 2 * neg_off;
    const size_t qbytes = static_cast<size_t>(zero_off) + kTcSampleBytes;

    int8_t* q = nullptr;
    TcStats* st = nullptr;
    double* su = nullptr;  // shift[192], unit[192]
    ScratchGuard gq(s), gs(s), gu(s);
    HSAD_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&q), qbytes, s));
    gq.p = q;
    HSAD_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&st), sizeof(TcStats), s));
    gs.p = st;
    HSAD_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&su), 2 * kTcBands * sizeof(double), s));
    gu.p = su;
    const char* rows0 = static_cast<const char*>(P.cube) +
                        (lo - P.buf_row0) * P.samples * P.bands * static_cast<int64_t>(P.elem_bytes);
    tc_stats_init<<<1, kTcBands, 0, s>>>(st);
    const int sblocks = static_cast<int>(npix < kTcStatBlocks ? npix : kTcStatBlocks);
    tc_stats_kernel<<<sblocks, kTcBands, 0, s>>>(rows0, P.elem_bytes, npix, P.bands, st);
    tc_stats_final<<<1, kTcBands, 0, s>>>(st, sblocks, npix, P.bands, su, su + kTcBands);
    HSAD_CUDA_TRY(cudaMemsetAsync(q + zero_off, 0, kTcSampleBytes, s));
    const int64_t items = npix * (kTcBands / 4);
    tc_slice_kernel<<<static_cast<unsigned>((items + 255) / 256), 256, 0, s>>>(rows0, P.elem_bytes, npix, P.bands,
                                                                              su, su + kTcBands, q, neg_off);
    HSAD_CUDA_TRY(cudaGetLastError());
    if (shift_unit_out)
        HSAD_CUDA_TRY(cudaMemcpyAsync(shift_unit_out, su, 2 * kTcBands * sizeof(double), cudaMemcpyDeviceToDevice, s));

    TcParams G{};
    G.q = q;
    G.neg_off = neg_off;
    G.zero_off = zero_off;
    G.lines = static_cast<int>(P.lines);
    G.samples = static_cast<int>(P.samples);
    G.qrow0 = static_cast<int>(lo);
    G.outer = P.outer;
    G.excl = P.inner;
    const int mp = (P.bands + 1 + 7) / 8 * 8;
    G.T = mp / 8;
    G.ntile = 0;
    for (int ib = 0; ib * 128 < mp; ++ib)
        for (int jb = 0; jb * 64 < mp && jb * 64 <= ib * 128 + 127; ++jb) {
            G.tile_ib[G.ntile] = ib;
            G.tile_jb[G.ntile] = jb;
            ++G.ntile;
        }
    // column segments: enough CTAs for a few waves, walks long enough to amortise the
    // full-window start (W^2 / 32 chunks)
    G.seg_len = env_int("HSAD_TC_SEG", 50);
    if (G.seg_len < 1) G.seg_len = 1;
    G.nseg = (G.samples + G.seg_len - 1) / G.seg_len;
    G.unit = su + kTcBands;
    G.lbo = static_cast<uint32_t>(env_int("HSAD_TC_LBO", 128));
    G.sbo = static_cast<uint32_t>(env_int("HSAD_TC_SBO", kTcBlk));
    HSAD_CUDA_TRY(cudaFuncSetAttribute(tc_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));

    const size_t px_bytes = static_cast<size_t>(G.T) * (G.T + 1) / 2 * 128 * sizeof(double);  // (hi, lo) planes
    const int64_t rows = P.row_end - P.row_begin;
    int64_t batch = static_cast<int64_t>((size_t{4} << 30) / (px_bytes * P.samples));  // <= 4 GB of tiles
    if (const int forced = env_int("HSAD_TC_BATCH_ROWS", 0); forced > 0) batch = forced;  // tests
    if (batch < 1) batch = 1;
    if (batch > rows) batch = rows;
    if (batch > 65535) batch = 65535;
    double* gram = gram_out;
    ScratchGuard gg(s);
    if (!gram) {
        HSAD_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&gram), px_bytes * P.samples * batch, s));
        gg.p = gram;
    }
    for (int64_t rb = P.row_begin; rb < P.row_end; rb += batch) {
        const int64_t re = rb + batch < P.row_end ? rb + batch : P.row_end;
        G.row_begin = static_cast<int>(rb);
        G.gram = gram_out ? gram_out + (rb - P.row_begin) * P.samples * (px_bytes / sizeof(double)) : gram;
        dim3 grid(static_cast<unsigned>(G.nseg * G.ntile), static_cast<unsigned>(re - rb));
        tc_gram_kernel<<<grid, kTcThreads, kTcSmem, s>>>(G);
        HSAD_CUDA_TRY(cudaGetLastError());
        if (gram_out) continue;
        FbParams F = P;
        F.row_begin = rb;
        F.row_end = re;
        // the kernel indexes its score map from its own row_begin
        F.scores = static_cast<char*>(P.scores) + (rb - P.row_begin) * P.samples * static_cast<int64_t>(P.score_bytes);
        F.gram = gram;
        F.gram_row0 = rb;
        F.shift = su;
        hsad_status fst = fullband_reg_launch(F, s);
        if (fst != HSAD_OK) return fst;
    }
    return HSAD_OK;
}

}  // namespace hsad_b200

// Test entry (not in include/hsad_gpu.h): the raw window Gram tiles of the shifted samples
// for every pixel of rows [row_begin, row_end), in fullband_reg_kernel's 8x8-tile order,
// plus shift[192] and unit[192].
extern "C" int32_t hsad_debug_fb_tc_gram(const void* d_cube, int32_t elem_bytes, int64_t lines, int64_t samples,
                                         int32_t bands, int64_t row_begin, int64_t row_end, int32_t outer,
                                         int32_t excl, double* d_gram, double* d_shift_unit, void* stream) {
    hsad_b200::FbParams P{};
    P.cube = d_cube;
    P.elem_bytes = elem_bytes;
    P.lines = lines;
    P.samples = samples;
    P.bands = bands;
    P.buf_row0 = 0;
    P.row_begin = row_begin;
    P.row_end = row_end;
    P.algo = HSAD_LRX;
    P.outer = outer;
    P.inner = excl;
    return hsad_b200::fullband_tc_launch(P, static_cast<cudaStream_t>(stream), d_gram, d_shift_unit);
}
