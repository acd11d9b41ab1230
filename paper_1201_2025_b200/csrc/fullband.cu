// K5+K6: full-band detectors (bands > 8, e.g. BASELINE C3: LRX on the raw 189-band cube).
// hsad::local_rx / hsad::dwrx at any band count (proj/core/src/detect.cpp:159-228 with
// stats.cpp:7-62): explicit window gather, two-pass centred covariance (divisor N),
// ridge delta = r tr(C)/L, Cholesky, quadratic form.
//
// One CTA (256 threads) per output pixel:
//   1. pass 1: window means (threads over bands, samples in the reference's scan order);
//   2. pass 2: centred samples stream through shared memory in chunks (register
//      kernel: raw chunks arrive two ahead by cp.async, then one centring pass); every thread
//      owns up to 5 register-tiled 4x4 blocks of the lower triangle of the Gram
//      matrix and accumulates them in fp64 (N L^2 MACs: the dense contraction);
//   3. the bordered matrix [C + delta I, d; d^T, 0] is written packed (lower, row-major)
//      to shared memory and factorised in place (right-looking Cholesky, one column
//      per step). The last Schur pivot is 0 - d^T (C + delta I)^-1 d, i.e. minus the
//      score, so no triangular solve is needed. D_j = pivots (singular rule as K3).
// Supports bands <= 224 (packed bordered matrix <= 209 KB of shared memory).
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "hsad_internal.h"

#ifdef HSAD_PHASE_TIMERS
__device__ unsigned long long g_fb_cycles[8];
#define FB_MARK(i)                                                              \
    do {                                                                        \
        if (threadIdx.x == 0) {                                                 \
            const long long fb_t1 = clock64();                                  \
            atomicAdd(&g_fb_cycles[i], (unsigned long long)(fb_t1 - fb_t0));    \
            fb_t0 = fb_t1;                                                      \
        }                                                                       \
    } while (0)
#else
#define FB_MARK(i) \
    do {           \
    } while (0)
#endif

namespace hsad_b200 {

constexpr int kFbThreads = 256;
constexpr int kFbMaxBands = 224;
constexpr int kFbMaxTiles = 5;  // 4x4 Gram tiles per thread (lower triangle of 228 x 228)

namespace {

__device__ __forceinline__ int mirror_fb(int i, int n) {
    if (static_cast<unsigned>(i) < static_cast<unsigned>(n)) return i;
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    i = abs(i) % period;
    return i < n ? i : period - i;
}

__device__ __forceinline__ double ld(const FbParams& P, int64_t idx) {
    return P.elem_bytes == 8 ? __ldg(static_cast<const double*>(P.cube) + idx)
                             : static_cast<double>(__ldg(static_cast<const float*>(P.cube) + idx));
}

// element index of window sample s (reference scan order: dr outer, dc inner,
// skipping the excluded centred box of edge `excl`, 0 = none) of pixel (r, c)
__device__ __forceinline__ int64_t sample_base(const FbParams& P, int r, int c, int s, int size,
                                               int excl) {
    const int h = size / 2, eh = excl / 2;
    // the excluded box occupies rows |dr| <= eh, columns |dc| <= eh
    int dr, dc;
    if (excl <= 0) {
        dr = s / size - h;
        dc = s % size - h;
    } else {
        const int top = (h - eh) * size;  // samples in the rows above the excluded band
        if (s < top) {
            dr = s / size - h;
            dc = s % size - h;
        } else {
            const int mid_rows = 2 * eh + 1, per_mid = size - excl;
            const int sm = s - top;
            if (sm < mid_rows * per_mid) {
                dr = sm / per_mid - eh;
                const int k = sm % per_mid;
                dc = k < h - eh ? k - h : k - (h - eh) + eh + 1;
            } else {
                const int sb = sm - mid_rows * per_mid;
                dr = eh + 1 + sb / size;
                dc = sb % size - h;
            }
        }
    }
    const int rr = mirror_fb(r + dr, static_cast<int>(P.lines)) - static_cast<int>(P.buf_row0);
    const int cc = mirror_fb(c + dc, static_cast<int>(P.samples));
    return (static_cast<int64_t>(rr) * P.samples + cc) * P.bands;
}

__device__ __forceinline__ double fb_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    return y * fma(-h * y, y, 1.5);
}

__device__ __forceinline__ int packed(int i, int k) { return i * (i + 1) / 2 + k; }  // k <= i

__global__ void __launch_bounds__(kFbThreads, 1) fullband_kernel(const FbParams P) {
    extern __shared__ double sm[];
    const int L = P.bands, MP = P.mp, CH = P.chunk;
    double* A = sm;                                   // packed (MP x MP lower)
    double* xs = A + packed(MP - 1, MP - 1) + 1;      // [CH][MP] centred samples
    double* mu = xs + static_cast<int64_t>(CH) * MP;  // [2][MP] means (window / inner box)
    double* col = mu + 2 * MP;                        // [MP] current Cholesky column
    __shared__ double s_piv, s_dmax, s_dmin;
    __shared__ int s_bad;

    const int t = threadIdx.x;
    const int c = blockIdx.x;
    const int64_t r = P.row_begin + blockIdx.y;
    if (r >= P.row_end) return;
#ifdef HSAD_PHASE_TIMERS
    long long fb_t0 = clock64();
#endif
    const int ri = static_cast<int>(r);
    // sample sets: LRX background = window minus the guard box (centre when guard 1);
    // DWRX covariance = annulus (outer minus inner box), d = mean(inner) - mean(annulus)
    const int size = P.outer;
    const int excl = P.inner;
    const int N = size * size - excl * excl;

    // element offsets of every window sample (and of the DWRX inner box), once
    int64_t* base = reinterpret_cast<int64_t*>(col + MP);  // [N + excl^2]
    const int NI = P.algo == HSAD_DWRX ? excl * excl : 0;
    for (int k = t; k < N + NI; k += kFbThreads)
        base[k] = k < N ? sample_base(P, ri, c, k, size, excl) : sample_base(P, ri, c, k - N, excl, 0);
    __syncthreads();
    // pass 1: means
    for (int b = t; b < MP; b += kFbThreads) {
        double s = 0.0, si = 0.0;
        if (b < L) {
            for (int k = 0; k < N; ++k) s += ld(P, base[k] + b);
            for (int k = 0; k < NI; ++k) si += ld(P, base[N + k] + b);
        }
        mu[b] = b < L ? s / N : 0.0;
        mu[MP + b] = (b < L && P.algo == HSAD_DWRX) ? si / (excl * excl) : 0.0;
    }
    __syncthreads();
    FB_MARK(0);

    // pass 2: centred Gram, 4x4 tiles of the lower triangle, in groups of
    // kFbThreads * kFbMaxTiles tiles (one group for L <= 196, two for L = 224)
    const int T = MP / 4;
    const int ntiles = T * (T + 1) / 2;
    const double invN = 1.0 / N;
    for (int g0 = 0; g0 < ntiles; g0 += kFbThreads * kFbMaxTiles) {
        int ti[kFbMaxTiles], tj[kFbMaxTiles];
        double acc[kFbMaxTiles][4][4];
#pragma unroll
        for (int u = 0; u < kFbMaxTiles; ++u) {
            const int tile = g0 + t + u * kFbThreads;
            int a = static_cast<int>((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
            while ((a + 1) * (a + 2) / 2 <= tile) ++a;
            while (a * (a + 1) / 2 > tile) --a;
            ti[u] = tile < ntiles ? a : -1;
            tj[u] = tile < ntiles ? tile - a * (a + 1) / 2 : -1;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[u][i][j] = 0.0;
        }
        for (int k0 = 0; k0 < N; k0 += CH) {
            const int nk = min(CH, N - k0);
            __syncthreads();
            for (int e = t; e < nk * MP; e += kFbThreads) {
                const int k = e / MP, b = e % MP;
                xs[e] = b < L ? ld(P, base[k0 + k] + b) - mu[b] : 0.0;
            }
            __syncthreads();
            for (int k = 0; k < nk; ++k) {
                const double* x = xs + k * MP;
#pragma unroll
                for (int u = 0; u < kFbMaxTiles; ++u) {
                    if (ti[u] < 0) continue;
                    const double2 a01 = *reinterpret_cast<const double2*>(x + 4 * ti[u]);
                    const double2 a23 = *reinterpret_cast<const double2*>(x + 4 * ti[u] + 2);
                    const double2 b01 = *reinterpret_cast<const double2*>(x + 4 * tj[u]);
                    const double2 b23 = *reinterpret_cast<const double2*>(x + 4 * tj[u] + 2);
                    const double av[4] = {a01.x, a01.y, a23.x, a23.y};
                    const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[u][i][j] = fma(av[i], bv[j], acc[u][i][j]);
                }
            }
        }
        // covariance (divisor N) into packed lower storage; symmetric by construction
#pragma unroll
        for (int u = 0; u < kFbMaxTiles; ++u) {
            if (ti[u] < 0) continue;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int gi = 4 * ti[u] + i, gj = 4 * tj[u] + j;
                    if (gj <= gi) A[packed(gi, gj)] = acc[u][i][j] * invN;
                }
        }
    }
    __syncthreads();
    FB_MARK(1);
    // displacement d and ridge; border row L holds d, (L, L) = 0; rows > L are inert
    if (t == 0) {
        double tr = 0.0;
        for (int b = 0; b < L; ++b) tr += A[packed(b, b)];
        s_piv = P.ridge * tr / L;  // delta
        s_bad = 0;
        s_dmax = 0.0;
        s_dmin = DBL_MAX;
    }
    __syncthreads();
    const double delta = s_piv;
    double dmaxabs = 0.0;
    for (int b = t; b < MP; b += kFbThreads) {
        if (b < L) {
            A[packed(b, b)] += delta;
            double d;
            if (P.algo == HSAD_LRX) {
                const int rr = mirror_fb(ri, static_cast<int>(P.lines)) - static_cast<int>(P.buf_row0);
                d = ld(P, (static_cast<int64_t>(rr) * P.samples + c) * L + b) - mu[b];
            } else {
                d = mu[MP + b] - mu[b];
            }
            A[packed(L, b)] = d;
            dmaxabs = fmax(dmaxabs, fabs(d));
        } else if (b == L) {
            A[packed(L, L)] = 0.0;  // border corner; rows > L (padding) are never read
        }
    }
    // any non-zero displacement? (detect.cpp:175-177 / 212: zero d skips the inverse)
    const int any_d = __syncthreads_or(dmaxabs > 0.0);
    const int64_t o = (r - P.row_begin) * P.samples + c;
    const int64_t lin = r * P.samples + c;
    if (lin == P.diag_lin && t == 0) *P.diag_out = delta;
    double score = 0.0;
    FB_MARK(2);
    if (any_d) {
        // Blocked right-looking Cholesky of the bordered matrix (rows 0..L; the border
        // row L is updated like any row and its diagonal ends as the Schur complement).
        // Column j of the factor is kept UNSCALED in A (l_ij = A[i][j] * rinv[j]), so a
        // panel step never writes the column it reads: per column one barrier, every
        // thread one row of the panel update. Then every thread applies the rank-PB
        // update to 4x4 tiles of the trailing lower triangle.
        constexpr int PB = 8;
        double* rinv = col;  // [MP] 1 / sqrt(pivot) per factored column
        for (int j0 = 0; j0 < L; j0 += PB) {
            const int jend = min(j0 + PB, L);  // panel columns [j0, jend)
            for (int jj = j0; jj < jend; ++jj) {
                const double p = A[packed(jj, jj)];
                if (!(p > 0.0)) {  // uniform: every thread read the same pivot
                    if (t == 0) s_bad = 1;
                    break;
                }
                const double ri = rsqrt(p);
                if (t == 0) {
                    s_dmax = fmax(s_dmax, fabs(p));
                    s_dmin = fmin(s_dmin, p);
                    rinv[jj] = ri;
                }
                // rows i > jj, columns jj < k < jend, k <= i
                for (int i = jj + 1 + t; i <= L; i += kFbThreads) {
                    const double lij = A[packed(i, jj)] * ri;
                    const int kmax = min(i, jend - 1);
                    for (int k = jj + 1; k <= kmax; ++k)
                        A[packed(i, k)] = fma(-lij, A[packed(k, jj)] * ri, A[packed(i, k)]);
                }
                __syncthreads();
            }
            __syncthreads();
            FB_MARK(4);
            if (s_bad) break;
            // trailing update: rows i in [jend, L], columns k in [jend, i]
            const int n = L + 1 - jend;            // trailing rows
            const int nb = (n + 3) / 4;            // 4-row blocks
            const int nblocks = nb * (nb + 1) / 2;
            const int w = jend - j0;               // panel width
            double rp[PB];
#pragma unroll
            for (int q = 0; q < PB; ++q) rp[q] = q < w ? rinv[j0 + q] : 0.0;
            for (int blk = t; blk < nblocks; blk += kFbThreads) {
                int bi = static_cast<int>((sqrt(8.0 * blk + 1.0) - 1.0) * 0.5);
                while ((bi + 1) * (bi + 2) / 2 <= blk) ++bi;
                while (bi * (bi + 1) / 2 > blk) --bi;
                const int bk = blk - bi * (bi + 1) / 2;
                const int i0 = jend + 4 * bi, k0 = jend + 4 * bk;
                double li[4][PB], lk[4][PB];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int q = 0; q < PB; ++q) {
                        li[a][q] = (i0 + a <= L && q < w) ? A[packed(i0 + a, j0 + q)] * rp[q] : 0.0;
                        lk[a][q] = (k0 + a <= L && q < w) ? A[packed(k0 + a, j0 + q)] * rp[q] : 0.0;
                    }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int i = i0 + a;
                    if (i > L) break;
#pragma unroll
                    for (int b2 = 0; b2 < 4; ++b2) {
                        const int k = k0 + b2;
                        if (k > i) break;
                        double acc = A[packed(i, k)];
#pragma unroll
                        for (int q = 0; q < PB; ++q) acc = fma(-li[a][q], lk[b2][q], acc);
                        A[packed(i, k)] = acc;
                    }
                }
            }
            __syncthreads();
            FB_MARK(5);
        }
        if (t == 0) s_piv = A[packed(L, L)];
        __syncthreads();
        FB_MARK(3);
        if (t == 0) {
            const bool singular = s_bad || !(s_dmax > 0.0) || s_dmin <= s_dmax * 1e-14;
            if (singular) {
                atomicMin(P.status, pack_failure(P.req, lin, HSAD_E_SINGULAR_AFTER_RIDGE));
            } else {
                score = -s_piv;  // Schur complement: 0 - d^T (C + delta I)^-1 d
                if (!isfinite(score)) {
                    atomicMin(P.status, pack_failure(P.req, lin, HSAD_E_SINGULAR_AFTER_RIDGE | 0x80));
                    score = 0.0;
                }
            }
        }
    }
    if (t == 0) {
        score = P.algo == HSAD_LRX ? fmax(score, 0.0) : fabs(score);
        if (P.score_bytes == 8) static_cast<double*>(P.scores)[o] = score;
        else static_cast<float*>(P.scores)[o] = static_cast<float>(score);
    }
}

// ---- register-resident variant (bands + 1 <= 192) ----------------------------
// Same arithmetic contract as fullband_kernel, but the bordered matrix never goes
// to shared memory: thread t owns one 8x8 tile (ti, tk), ti >= tk, of the lower
// triangle. The centred Gram accumulates into that tile (64 fp64 accumulators,
// 16 doubles of shared-memory reads per 64 FMAs), and the right-looking Cholesky
// then runs on the same registers: per column j the owners of tile column j/8
// publish the (unscaled) column c to shared memory (double-buffered, one barrier
// per column), and every live tile applies a_ik -= c_i (c_k / c_j). The pivots
// c_j are the LDLT D_j of the singular rule; the last Schur pivot is -score.
constexpr int kFbRegMaxMp = 192;  // 24 tile rows -> 300 tiles -> <= 320 threads
constexpr int kFbRegThreads = 320;

__global__ void __launch_bounds__(kFbRegThreads, 1) fullband_reg_kernel(const FbParams P) {
    extern __shared__ double sm[];
    const int L = P.bands, MP = P.mp, CH = P.chunk;
    // 8-band blocks are padded so that lanes reading different blocks hit different
    // banks: xs blocks of 10 doubles (16-byte aligned), published columns of 9
    const int S = (MP / 8) * 10;                       // xs row stride
    const int CBP = (MP / 8) * 10;                     // panel column length (padded rows)
    double* xs = sm;                                   // [CH][S] centred samples
    double* mu = xs + static_cast<int64_t>(CH) * S;    // [2][MP] means (window / inner box)
    double* lpt = mu + 2 * MP;                         // [2][8 CBP + 8] Cholesky panels
    double* dg = lpt + 2 * (8 * CBP + 8);              // [MP] diagonal of C / displacement d
    __shared__ double s_piv, s_dmax, s_dmin, s_corner[8];
    __shared__ int s_bad;

    const int t = threadIdx.x;
    const int c = blockIdx.x;
    const int64_t r = P.row_begin + blockIdx.y;
    if (r >= P.row_end) return;
    const int ri = static_cast<int>(r);
#ifdef HSAD_PHASE_TIMERS
    long long fb_t0 = clock64();
#endif
    const int size = P.outer, excl = P.inner;
    const int N = size * size - excl * excl;
    int64_t* base = reinterpret_cast<int64_t*>(dg + MP);  // [N + excl^2]
    const int NI = P.algo == HSAD_DWRX ? excl * excl : 0;
    // tensor-core route: the Gram tiles of this pixel; their border row L (a constant-one
    // band in the digit array) holds the exact window sums of the shifted samples
    const bool tc = P.gram != nullptr;
    const int T = MP / 8;
    const int ntiles = T * (T + 1) / 2;
    const double* gpx = tc ? P.gram + ((r - P.gram_row0) * P.samples + c) * ntiles * 128 : nullptr;
    for (int k = t + (tc ? N : 0); k < N + NI; k += blockDim.x)
        base[k] = k < N ? sample_base(P, ri, c, k, size, excl) : sample_base(P, ri, c, k - N, excl, 0);
    __syncthreads();
    // window means: one band per thread, 8 independent partial sums (8 loads in flight;
    // summation order differs from a sequential loop only at rounding level)
    auto band_sum = [&](int b, int k0, int n) {
        double p[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        int k = 0;
        for (; k + 8 <= n; k += 8)
#pragma unroll
            for (int u = 0; u < 8; ++u) p[u] += ld(P, base[k0 + k + u] + b);
        for (; k < n; ++k) p[0] += ld(P, base[k0 + k] + b);
        return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
    };
    for (int b = t; b < MP; b += blockDim.x) {
        double sum = 0.0;
        if (tc) {
            // S = (hi, lo): the exact window sum of the shifted samples
            const int tl = L >> 3;
            const double* sp = gpx + (tl * (tl + 1) / 2 + (b >> 3)) * 128 + (L & 7) * 8 + (b & 7);
            xs[b] = b < L ? __ldg(sp) : 0.0;
            xs[MP + b] = b < L ? __ldg(sp + 64) : 0.0;
        } else if (b < L) {
            sum = band_sum(b, 0, N);
        }
        const double si = (b < L && NI > 0) ? band_sum(b, N, NI) : 0.0;
        mu[b] = b < L ? (tc ? P.shift[b] + (xs[b] + xs[MP + b]) / N : sum / N) : 0.0;
        mu[MP + b] = (b < L && P.algo == HSAD_DWRX) ? si / (excl * excl) : 0.0;
    }
    __syncthreads();
    FB_MARK(0);

    // this thread's tile of the lower triangle
    // Tiles are dealt to threads column by column (tile column tk = threads
    // [tk T - tk (tk - 1) / 2, ...) in row order): the tiles a Cholesky step has finished
    // with are a prefix of the CTA, so whole warps drop out of the trailing update and the
    // panel of a step sits in one warp (row-major dealing kept every warp issuing the 512-FMA
    // update for a few live lanes until the last steps).
    const bool own = t < ntiles;
    int tk = 0;
#ifndef HSAD_FB_ROWMAJOR_TILES
    while (tk + 1 < T && (tk + 1) * T - (tk + 1) * tk / 2 <= t) ++tk;
    int ti = own ? tk + (t - (tk * T - tk * (tk - 1) / 2)) : 0;
    if (!own) tk = 0;
#else
    int ti = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    tk = own ? t - ti * (ti + 1) / 2 : 0;
    if (!own) ti = 0;
#endif
    double acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
    if (P.gram) {
        // tensor-core route: G = sum_k (x_k - s)(x_k - s)^T came from tc_gram_kernel (exact
        // integer accumulation, one rounding); C = G / N - (mu - s)(mu - s)^T
        if (own) {
            // C = (N G - S S^T) / N^2 with G and S as exact (hi, lo) pairs: the difference is
            // formed in double-double arithmetic and rounded once, so a window whose mean is
            // far from the shift loses nothing to cancellation
            const double2* g2 = reinterpret_cast<const double2*>(gpx + (ti * (ti + 1) / 2 + tk) * 128);
            const double dN = N, invN2 = 1.0 / (dN * dN);
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int i = 8 * ti + a;
                const double ai = xs[i], bi = xs[MP + i];  // 0 for i >= L
#pragma unroll
                for (int b = 0; b < 8; b += 2) {
                    const double2 gh2 = __ldg(g2 + a * 4 + b / 2);
                    const double2 gl2 = __ldg(g2 + 32 + a * 4 + b / 2);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int k = 8 * tk + b + h;
                        const double gh = h ? gh2.y : gh2.x, gl = h ? gl2.y : gl2.x;
                        const double aj = xs[k], bj = xs[MP + k];
                        const double th = dN * gh, te = fma(dN, gh, -th);
                        const double ph = ai * aj, pe = fma(ai, aj, -ph);
                        const double cross = fma(ai, bj, bi * aj);
                        const double sd = th - ph, bb = sd - th;
                        const double e = (th - (sd - bb)) + (-ph - bb);  // two_sum(th, -ph)
                        const double res = sd + (e + (((te + dN * gl) - pe) - cross));
                        acc[a][b + h] = (i < L && k < L) ? res * invN2 : 0.0;
                    }
                }
            }
        }
        __syncthreads();  // xs (the shifted means) is free again
    } else {
#ifdef HSAD_FB_SYNC_CHUNKS
    for (int k0 = 0; k0 < N; k0 += CH) {
        const int nk = min(CH, N - k0);
        __syncthreads();
        // one band per thread, all samples of the chunk (coalesced across the warp,
        // 8 independent loads in flight per thread, no integer division)
        for (int b = t; b < MP; b += blockDim.x) {
            double* dst = xs + (b >> 3) * 10 + (b & 7);
            if (b < L) {
                const double m = mu[b];
#pragma unroll 8
                for (int k = 0; k < nk; ++k) dst[k * S] = ld(P, base[k0 + k] + b) - m;
            } else {
                for (int k = 0; k < nk; ++k) dst[k * S] = 0.0;
            }
        }
        __syncthreads();
#else
    // Chunks of CH window samples arrive in a double-buffered raw stage by cp.async
    // (4/8-byte LDGSTS per element, all threads, no registers held), two chunks
    // ahead; each chunk is then centred and widened into xs by every thread in one
    // short pass, so the global-load latency hides behind the previous chunk's Gram.
    const int EB = P.elem_bytes;
    unsigned char* raw = reinterpret_cast<unsigned char*>(base + size * size);  // after the offsets
    const int raw_stride = CH * L * EB;  // bytes per stage buffer
    const int nchunks = (N + CH - 1) / CH;
    auto issue = [&](int j) {
        const int k0 = j * CH, nk = min(CH, N - k0);
        unsigned char* dstb = raw + (j & 1) * raw_stride;
        const int total = nk * L;
        int k = t / L, b = t % L;
        const int dk = blockDim.x / L, db = blockDim.x % L;
        for (int e = t; e < total; e += blockDim.x) {
            const char* src = static_cast<const char*>(P.cube) + (base[k0 + k] + b) * EB;
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(dstb + e * EB));
            if (EB == 8)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
            k += dk;
            b += db;
            if (b >= L) {
                b -= L;
                ++k;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // padding bands [L, MP) of xs stay zero for every chunk
    for (int e = t; e < CH * (MP - L); e += blockDim.x) {
        const int k = e / (MP - L), b = L + e % (MP - L);
        xs[k * S + (b >> 3) * 10 + (b & 7)] = 0.0;
    }
    issue(0);
    if (nchunks > 1) issue(1);
    for (int j = 0; j < nchunks; ++j) {
        const int k0 = j * CH, nk = min(CH, N - k0);
        if (j + 1 < nchunks) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();  // chunk j landed for every thread; the Gram of chunk j-1 is done
        {
            const unsigned char* srcb = raw + (j & 1) * raw_stride;
            const int total = nk * L;
            int k = t / L, b = t % L;
            const int dk = blockDim.x / L, db = blockDim.x % L;
            for (int e = t; e < total; e += blockDim.x) {
                const double v = EB == 8 ? reinterpret_cast<const double*>(srcb)[e]
                                         : static_cast<double>(reinterpret_cast<const float*>(srcb)[e]);
                xs[k * S + (b >> 3) * 10 + (b & 7)] = v - mu[b];
                k += dk;
                b += db;
                if (b >= L) {
                    b -= L;
                    ++k;
                }
            }
        }
        __syncthreads();  // xs holds chunk j; its raw buffer is free
        if (j + 2 < nchunks) issue(j + 2);
#endif
        if (own) {
            const double* xa = xs + 10 * ti;
            const double* xb = xs + 10 * tk;
            for (int k = 0; k < nk; ++k) {
                double av[8], bv[8];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const double2 a2 = *reinterpret_cast<const double2*>(xa + k * S + 2 * h);
                    const double2 b2 = *reinterpret_cast<const double2*>(xb + k * S + 2 * h);
                    av[2 * h] = a2.x;
                    av[2 * h + 1] = a2.y;
                    bv[2 * h] = b2.x;
                    bv[2 * h + 1] = b2.y;
                }
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
            }
        }
    }
    // covariance (divisor N); diagonal to shared memory for the trace
    const double invN = 1.0 / N;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] *= invN;
    }  // !P.gram
    if (own && ti == tk)
#pragma unroll
        for (int a = 0; a < 8; ++a) dg[8 * ti + a] = acc[a][a];
    __syncthreads();
    FB_MARK(1);
    if (t == 0) {
        double tr = 0.0;
        for (int b = 0; b < L; ++b) tr += dg[b];
        s_piv = P.ridge * tr / L;  // delta
        s_bad = 0;
        s_dmax = 0.0;
        s_dmin = DBL_MAX;
    }
    __syncthreads();
    const double delta = s_piv;
    // displacement d (border row L), ridge on the diagonal
    double dmaxabs = 0.0;
    for (int b = t; b < L; b += blockDim.x) {
        double d;
        if (P.algo == HSAD_LRX) {
            const int rr = mirror_fb(ri, static_cast<int>(P.lines)) - static_cast<int>(P.buf_row0);
            d = ld(P, (static_cast<int64_t>(rr) * P.samples + c) * L + b) - mu[b];
        } else {
            d = mu[MP + b] - mu[b];
        }
        dg[b] = d;
        dmaxabs = fmax(dmaxabs, fabs(d));
    }
    const int any_d = __syncthreads_or(dmaxabs > 0.0);
    if (own) {
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int i = 8 * ti + a;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int k = 8 * tk + b;
                if (i == k && i < L) acc[a][b] += delta;
                if (i == L) acc[a][b] = k < L ? dg[k] : 0.0;  // border row; corner 0
            }
        }
    }
    const int64_t o = (r - P.row_begin) * P.samples + c;
    const int64_t lin = r * P.samples + c;
    if (lin == P.diag_lin && t == 0) *P.diag_out = delta;
    FB_MARK(2);
    double score = 0.0;
    if (any_d) {
        // Blocked right-looking Cholesky on the register tiles, one 8-column tile
        // column jt per step (2 barriers per step, panel buffer double-buffered):
        //   1. the owner of diagonal tile (jt, jt) factors it alone (pivots p_j are the
        //      LDLT D_j of the singular rule) and publishes L_jj and 1/L_jj[c][c];
        //   2. the owners of tiles (ti > jt, jt) solve X = A L_jj^-T in registers and
        //      publish X (the panel) column-major;
        //   3. every tile (ti >= tk > jt) applies acc -= X_ti X_tk^T (512 FMAs; per
        //      panel column two 8-double vectors, 4 LDS.128 each).
        // Columns >= L (border, padding) are never factored; the border corner then
        // holds 0 - d^T (C + delta I)^-1 d = -score.
        const int LT = L >> 3;  // tile column holding the border row/column
        for (int jt = 0; jt <= LT; ++jt) {
            double* lp = lpt + (jt & 1) * (8 * CBP + 8);  // [8][CBP] panel, then [8] 1/diag
            double* rdiag = lp + 8 * CBP;
            if (own && ti == jt && tk == jt) {
                bool bad = false;
                double dmax = s_dmax, dmin = s_dmin;
#pragma unroll
                for (int jc = 0; jc < 8; ++jc) {
                    if (8 * jt + jc < L && !bad) {
                        const double p = acc[jc][jc];
                        if (!(p > 0.0)) {
                            bad = true;
                        } else {
                            dmax = fmax(dmax, fabs(p));
                            dmin = fmin(dmin, p);
                            const double r = fb_rsqrt(p);
                            rdiag[jc] = r;
                            acc[jc][jc] = p * r;
#pragma unroll
                            for (int a2 = jc + 1; a2 < 8; ++a2) acc[a2][jc] *= r;
#pragma unroll
                            for (int b2 = jc + 1; b2 < 8; ++b2)
#pragma unroll
                                for (int a2 = b2; a2 < 8; ++a2)
                                    acc[a2][b2] = fma(-acc[a2][jc], acc[b2][jc], acc[a2][b2]);
                        }
                    }
                }
                s_dmax = dmax;
                s_dmin = dmin;
                if (bad) s_bad = 1;
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2)
#pragma unroll
                    for (int a2 = 0; a2 < 8; ++a2) lp[c2 * CBP + 10 * jt + a2] = a2 >= c2 ? acc[a2][c2] : 0.0;
                if (jt == LT)  // all 8 diagonal entries (a runtime register index would spill acc)
#pragma unroll
                    for (int a2 = 0; a2 < 8; ++a2) s_corner[a2] = acc[a2][a2];
            }
            __syncthreads();
            FB_MARK(4);  // diagonal-block factorisation (critical path)
            if (s_bad || jt == LT) break;  // uniform
            if (own && tk == jt && ti > jt) {
                // forward substitution against L_jj^T, column by column, in place
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2) {
                    const double r = rdiag[c2];
#pragma unroll
                    for (int a2 = 0; a2 < 8; ++a2) {
                        double v = acc[a2][c2];
#pragma unroll
                        for (int b2 = 0; b2 < c2; ++b2) v = fma(-acc[a2][b2], lp[b2 * CBP + 10 * jt + c2], v);
                        acc[a2][c2] = v * r;
                    }
                }
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2)
#pragma unroll
                    for (int a2 = 0; a2 < 8; ++a2) lp[c2 * CBP + 10 * ti + a2] = acc[a2][c2];
            }
            __syncthreads();
            FB_MARK(5);  // panel solves
            if (own && tk > jt) {
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2) {
                    double li[8], lk[8];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const double2 x2 = *reinterpret_cast<const double2*>(lp + c2 * CBP + 10 * ti + 2 * h);
                        const double2 y2 = *reinterpret_cast<const double2*>(lp + c2 * CBP + 10 * tk + 2 * h);
                        li[2 * h] = x2.x;
                        li[2 * h + 1] = x2.y;
                        lk[2 * h] = y2.x;
                        lk[2 * h + 1] = y2.y;
                    }
#pragma unroll
                    for (int a2 = 0; a2 < 8; ++a2)
#pragma unroll
                        for (int b2 = 0; b2 < 8; ++b2) acc[a2][b2] = fma(-li[a2], lk[b2], acc[a2][b2]);
                }
            }
#ifdef HSAD_PHASE_TIMERS
            __syncthreads();  // probe build only: separates the trailing update
            FB_MARK(6);
#endif
        }
        __syncthreads();
        FB_MARK(3);
        if (t == 0) {
            const bool singular = s_bad || !(s_dmax > 0.0) || s_dmin <= s_dmax * 1e-14;
            if (singular) {
                atomicMin(P.status, pack_failure(P.req, lin, HSAD_E_SINGULAR_AFTER_RIDGE));
            } else {
                score = -s_corner[L & 7];
                if (!isfinite(score)) {
                    atomicMin(P.status, pack_failure(P.req, lin, HSAD_E_SINGULAR_AFTER_RIDGE | 0x80));
                    score = 0.0;
                }
            }
        }
    }
    if (t == 0) {
        score = P.algo == HSAD_LRX ? fmax(score, 0.0) : fabs(score);
        if (P.score_bytes == 8) static_cast<double*>(P.scores)[o] = score;
        else static_cast<float*>(P.scores)[o] = static_cast<float>(score);
    }
}

}  // namespace

#ifdef HSAD_PHASE_TIMERS
extern "C" void hsad_fb_phase_cycles(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_fb_cycles, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_fb_cycles, z, sizeof(z));
    }
}
#endif

bool fullband_tc_applies(const FbParams& P);                                  // fullband_tc.cu
hsad_status fullband_tc_launch(FbParams& P, cudaStream_t s, double* gram_out, double* shift_unit_out);

// The register-tile kernel over rows [row_begin, row_end) (bands + 1 <= 192).
hsad_status fullband_reg_launch(FbParams& P, cudaStream_t s) {
    const int64_t rows = P.row_end - P.row_begin;
    if (rows > 65535) return set_error(HSAD_E_UNSUPPORTED, "strip too tall for one launch");
    dim3 grid(static_cast<unsigned>(P.samples), static_cast<unsigned>(rows));
    const int64_t nsamp = static_cast<int64_t>(P.outer) * P.outer;  // >= N + inner^2
    P.mp = ((P.bands + 1) + 7) / 8 * 8;
    P.chunk = 32;
    const size_t smem = (static_cast<size_t>(P.chunk) * (P.mp / 8) * 10 + 3 * P.mp +
                         2 * (8 * (P.mp / 8) * 10 + 8) + nsamp) * 8 +
                        2 * static_cast<size_t>(P.chunk) * P.bands * P.elem_bytes;  // cp.async stage
    HSAD_CUDA_TRY(cudaFuncSetAttribute(fullband_reg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
    const int T = P.mp / 8;
    const int nt = (T * (T + 1) / 2 + 31) / 32 * 32;
    fullband_reg_kernel<<<grid, nt, smem, s>>>(P);
    HSAD_CUDA_TRY(cudaGetLastError());
    return HSAD_OK;
}

// Shared memory and launch shape for one full-band request.
hsad_status fullband_launch(FbParams& P, cudaStream_t s) {
    if (P.bands > kFbMaxBands)
        return set_error(HSAD_E_UNSUPPORTED, "full-band detection supports at most " +
                                                 std::to_string(kFbMaxBands) + " bands");
    const int64_t rows = P.row_end - P.row_begin;
    if (rows > 65535) return set_error(HSAD_E_UNSUPPORTED, "strip too tall for one launch");
    dim3 grid(static_cast<unsigned>(P.samples), static_cast<unsigned>(rows));
    const int64_t nsamp = static_cast<int64_t>(P.outer) * P.outer;  // >= N + inner^2
    const int mp8 = ((P.bands + 1) + 7) / 8 * 8;
    if (mp8 <= kFbRegMaxMp && !getenv("HSAD_FB_PACKED")) {
        // register-resident tiles: shared memory holds only samples and vectors; with
        // HSAD_FB_TC=1 the Gram comes from the tensor cores (fullband_tc.cu)
        P.gram = nullptr;
        if (fullband_tc_applies(P)) return fullband_tc_launch(P, s, nullptr, nullptr);
        return fullband_reg_launch(P, s);
    }
    P.mp = ((P.bands + 1) + 3) / 4 * 4;
    const int64_t tri = static_cast<int64_t>(P.mp) * (P.mp + 1) / 2;
    int chunk = 32;
    auto bytes = [&](int ch) {
        return (tri + static_cast<int64_t>(ch) * P.mp + 3 * P.mp + nsamp) * 8;
    };
    while (chunk > 4 && bytes(chunk) > 220 * 1024) chunk /= 2;
    if (bytes(chunk) > 227 * 1024)
        return set_error(HSAD_E_UNSUPPORTED, "full-band working set exceeds shared memory");
    P.chunk = chunk;
    const size_t smem = static_cast<size_t>(bytes(chunk));
    HSAD_CUDA_TRY(cudaFuncSetAttribute(fullband_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
    fullband_kernel<<<grid, kFbThreads, smem, s>>>(P);
    HSAD_CUDA_TRY(cudaGetLastError());
    return HSAD_OK;
}

}  // namespace hsad_b200
