// K6b: full-band DWEST (hsad::dwest at bands > 8, e.g. the raw 189-band cube of BASELINE
// C3; proj/core/src/detect.cpp:230-276 with symmetric_eigen, proj/core/src/stats.cpp:64-89).
//
// One CTA (256 threads) per output pixel, the whole eigenproblem in shared memory:
//   1. window means of the inner box and of the annulus (two-pass, reference scan order);
//   2. C_diff = C_in - C_ann as ONE signed Gram: every centred sample x contributes
//      w x x^T with w = +1/N_in (inner box) or -1/N_ann (annulus); 4x4 register tiles of
//      the lower triangle, samples staged through shared memory in chunks;
//   3. Householder tridiagonalisation in place (packed lower storage; the reflectors stay
//      in the columns below the sub-diagonal) — the first stage of the Eigen solver the
//      reference calls (SelfAdjointEigenSolver: tridiagonalisation + implicit QR);
//   4. eigenvalues of the tridiagonal T by Sturm-count multisection (all 256 threads probe
//      one point each per round: 8 bits per round): lambda_0 = the largest; the DWEST
//      selection {i : lambda_i > 0, lambda_i >= f lambda_0} is monotone in lambda, so its
//      size is n - count(f lambda_0) and the selected eigenvalues are the top ones;
//   5. eigenvectors of T for the selected eigenvalues by the twisted factorisation
//      (stationary L D L^T + progressive U D U^T of T - lambda I, twist index at the
//      smallest |gamma|), re-orthogonalised within clusters;
//   6. back-transformation by the stored reflectors (one warp per vector), the sign
//      rule (first largest-|.| component positive, stats.cpp:83-85), and the projection
//      sum in the reference's descending order; eigen-count = selection size.
// Supports bands <= kDwMaxBands (the packed matrix and the work vectors in 227 KB).
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <string>

#include "hsad_internal.h"

namespace hsad_b200 {

constexpr int kDwThreads = 256;
constexpr int kDwMaxBands = 200;
constexpr int kDwMaxSel = 64;    // selected eigenvectors per pixel (<= inner^2 - 1; scenes: 1-3)
constexpr int kDwRing = 16;      // eigenvectors kept for re-orthogonalisation within clusters
constexpr int kDwMaxTiles = 5;   // 4x4 Gram tiles per thread (lower triangle of 200 x 200)

namespace {

__device__ __forceinline__ int mirror_dw(int i, int n) {
    if (static_cast<unsigned>(i) < static_cast<unsigned>(n)) return i;
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    i = abs(i) % period;
    return i < n ? i : period - i;
}

__device__ __forceinline__ double ld_dw(const FbParams& P, int64_t idx) {
    return P.elem_bytes == 8 ? __ldg(static_cast<const double*>(P.cube) + idx)
                             : static_cast<double>(__ldg(static_cast<const float*>(P.cube) + idx));
}

__device__ __forceinline__ int pk(int i, int k) { return i * (i + 1) / 2 + k; }  // k <= i

// block-wide sum / max, result in every thread (red: >= 32 doubles of shared memory)
__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kDwThreads / 32; ++i) s += red[i];  // fixed order: deterministic
    return s;
}
__device__ __forceinline__ double block_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = red[0];
    for (int i = 1; i < kDwThreads / 32; ++i) s = fmax(s, red[i]);
    return s;
}

// number of eigenvalues of T (diagonal d, squared off-diagonal e2) below x
__device__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    int c = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = (d[i] - x) - e2[i - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        c += q < 0.0;
    }
    return c;
}

// eigenvalue of ascending index idx in [lo, hi] (count(lo) <= idx < count(hi)) by
// multisection: every thread probes one interior point per round
__device__ double eigenvalue(const double* d, const double* e2, int n, int idx, double lo, double hi,
                             double pivmin, double* red) {
    const int t = threadIdx.x;
    for (int round = 0; round < 9; ++round) {
        const double width = hi - lo;
        if (!(width > 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) || !(width > pivmin)) break;
        const double x = lo + width * (t + 1) / (kDwThreads + 1);
        const int below = sturm_count(d, e2, n, x, pivmin) <= idx;
        const int nb = __syncthreads_count(below);  // points with count <= idx (a prefix)
        __syncthreads();
        if (t == nb - 1) red[0] = x;
        if (t == nb) red[1] = x;
        __syncthreads();
        const double nlo = nb > 0 ? red[0] : lo, nhi = nb < kDwThreads ? red[1] : hi;
        __syncthreads();
        lo = nlo;
        hi = nhi;
    }
    return 0.5 * (lo + hi);
}

}  // namespace

__global__ void __launch_bounds__(kDwThreads, 1) fullband_dwest_kernel(const FbParams P) {
    extern __shared__ double sm[];
    const int L = P.bands, L4 = (P.bands + 3) & ~3, CH = P.chunk;
    double* A = sm;                                    // packed lower L4 x L4
    double* xs = A + pk(L4 - 1, L4 - 1) + 1;           // [CH][L4] centred samples; later work
    double* mu_in = xs + static_cast<int64_t>(CH) * L4;  // [L4] -> m = mean(inner) - mean(annulus)
    double* mu_an = mu_in + L4;                        // [L4]
    double* dg = mu_an + L4;                           // [L4] diagonal of T
    double* e2 = dg + L4;                              // [L4] squared off-diagonal of T
    double* bet = e2 + L4;                             // [L4] reflector scales
    double* vv = bet + L4;                             // [L4] reflector / work
    double* pp = vv + L4;                              // [L4] work
    double* red = pp + L4;                             // [64] reductions
    double* lam = red + 64;                            // [kDwMaxSel] selected eigenvalues
    double* contrib = lam + kDwMaxSel;                 // [kDwMaxSel] signed projections
    int64_t* base = reinterpret_cast<int64_t*>(contrib + kDwMaxSel);  // [outer^2] offsets

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#ifdef HSAD_DW_DEBUG
    long long dbg_t0 = clock64(), dbg_ph[8] = {0};
#define DW_MARK(i) do { long long t1_ = clock64(); dbg_ph[i] += t1_ - dbg_t0; dbg_t0 = t1_; } while (0)
#else
#define DW_MARK(i) do { } while (0)
#endif
    const int c = blockIdx.x;
    const int64_t r = P.row_begin + blockIdx.y;
    if (r >= P.row_end) return;
    const int ri = static_cast<int>(r);
    const int64_t o = (r - P.row_begin) * P.samples + c;
    const int outer = P.outer, inner = P.inner, oh = outer / 2, ih = inner / 2;
    const int NI = inner * inner, N = outer * outer;
    const int NA = N - NI;

    // sample offsets in the reference's scan order: inner box first, then the annulus
    for (int s = t; s < N; s += kDwThreads) {
        const int dr = s / outer - oh, dc = s % outer - oh;
        const bool in_box = abs(dr) <= ih && abs(dc) <= ih;
        // rank within its own set (row-major over the window): inner samples before s
        const int in_before = dr < -ih ? 0 : dr > ih ? NI : (dr + ih) * inner + min(max(dc + ih, 0), inner);
        const int k = in_box ? in_before : NI + (s - in_before);
        const int rr = mirror_dw(ri + dr, static_cast<int>(P.lines)) - static_cast<int>(P.buf_row0);
        const int cc = mirror_dw(c + dc, static_cast<int>(P.samples));
        base[k] = (static_cast<int64_t>(rr) * P.samples + cc) * L;
    }
    __syncthreads();
    // 1. means (reference scan order within each set)
    for (int b = t; b < L4; b += kDwThreads) {
        double si = 0.0, sa = 0.0;
        if (b < L) {
            for (int k = 0; k < NI; ++k) si += ld_dw(P, base[k] + b);
            for (int k = NI; k < N; ++k) sa += ld_dw(P, base[k] + b);
        }
        mu_in[b] = b < L ? si / NI : 0.0;
        mu_an[b] = b < L ? sa / NA : 0.0;
    }
    __syncthreads();

    // 2. signed Gram: C_diff = sum_in x x^T / N_in - sum_ann x x^T / N_ann (centred)
    const int T4 = L4 / 4;
    const int ntiles = T4 * (T4 + 1) / 2;
    {
        int ti[kDwMaxTiles], tj[kDwMaxTiles];
        double acc[kDwMaxTiles][4][4];
#pragma unroll
        for (int u = 0; u < kDwMaxTiles; ++u) {
            const int tile = t + u * kDwThreads;
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
        const double w_in = 1.0 / NI, w_an = -1.0 / NA;
        for (int k0 = 0; k0 < N; k0 += CH) {
            const int nk = min(CH, N - k0);
            __syncthreads();
            for (int e = t; e < nk * L4; e += kDwThreads) {
                const int k = e / L4, b = e % L4;
                const double* mu = k0 + k < NI ? mu_in : mu_an;
                xs[e] = b < L ? ld_dw(P, base[k0 + k] + b) - mu[b] : 0.0;
            }
            __syncthreads();
            for (int k = 0; k < nk; ++k) {
                const double* x = xs + k * L4;
                const double w = k0 + k < NI ? w_in : w_an;
#pragma unroll
                for (int u = 0; u < kDwMaxTiles; ++u) {
                    if (ti[u] < 0) continue;
                    const double2 a01 = *reinterpret_cast<const double2*>(x + 4 * ti[u]);
                    const double2 a23 = *reinterpret_cast<const double2*>(x + 4 * ti[u] + 2);
                    const double2 b01 = *reinterpret_cast<const double2*>(x + 4 * tj[u]);
                    const double2 b23 = *reinterpret_cast<const double2*>(x + 4 * tj[u] + 2);
                    const double av[4] = {w * a01.x, w * a01.y, w * a23.x, w * a23.y};
                    const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[u][i][j] = fma(av[i], bv[j], acc[u][i][j]);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kDwMaxTiles; ++u) {
            if (ti[u] < 0) continue;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int gi = 4 * ti[u] + i, gj = 4 * tj[u] + j;
                    if (gj <= gi) A[pk(gi, gj)] = acc[u][i][j];
                }
        }
    }
    for (int b = t; b < L4; b += kDwThreads) mu_in[b] = mu_in[b] - mu_an[b];  // m_diff
    __syncthreads();
    DW_MARK(0);

    // 3. Householder tridiagonalisation (lower): reflector k zeroes A(k+2.., k)
    for (int k = 0; k + 2 < L; ++k) {
        double part = 0.0;
        for (int i = k + 1 + t; i < L; i += kDwThreads) part = fma(A[pk(i, k)], A[pk(i, k)], part);
        const double nrm2 = block_sum(part, red);
        const double x0 = A[pk(k + 1, k)];
        const double sig = nrm2 - x0 * x0;
        double b = 0.0, alpha = x0, v0 = x0;
        if (sig > 0.0) {
            alpha = -copysign(sqrt(nrm2), x0);
            v0 = x0 - alpha;
            b = 2.0 / (sig + v0 * v0);
        }
        for (int i = k + 1 + t; i < L; i += kDwThreads) vv[i] = i == k + 1 ? v0 : A[pk(i, k)];
        if (t == 0) {
            dg[k] = A[pk(k, k)];
            e2[k] = alpha;  // off-diagonal (squared after the loop)
            bet[k] = b;
        }
        __syncthreads();
        if (t == 0) A[pk(k + 1, k)] = v0;  // column k keeps the reflector
        if (b == 0.0) {
            __syncthreads();
            continue;
        }
        // p = b A_trail v (symmetric, lower packed): one warp per row, lanes over columns,
        // four rows per warp in flight (independent accumulators)
        constexpr int NW = kDwThreads / 32, RU = 4;
        for (int i0 = k + 1 + warp; i0 < L; i0 += NW * RU) {
            double s4[RU];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const int i = i0 + u * NW;
                double acc = 0.0;
                if (i < L) {
                    const double* row = A + pk(i, 0);
                    for (int j = k + 1 + lane; j <= i; j += 32) acc = fma(row[j], vv[j], acc);
                    for (int j = i + 1 + lane; j < L; j += 32) acc = fma(A[pk(j, i)], vv[j], acc);
                }
                s4[u] = acc;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int u = 0; u < RU; ++u) s4[u] += __shfl_xor_sync(0xffffffffu, s4[u], off);
            if (lane == 0)
#pragma unroll
                for (int u = 0; u < RU; ++u)
                    if (i0 + u * NW < L) pp[i0 + u * NW] = b * s4[u];
        }
        __syncthreads();
        part = 0.0;
        for (int i = k + 1 + t; i < L; i += kDwThreads) part = fma(pp[i], vv[i], part);
        const double K = 0.5 * b * block_sum(part, red);
        for (int i = k + 1 + t; i < L; i += kDwThreads) pp[i] = fma(-K, vv[i], pp[i]);  // w
        __syncthreads();
        // A_trail -= v w^T + w v^T (lower triangle): a warp per row, lanes over columns
        for (int i0 = k + 1 + warp; i0 < L; i0 += NW * RU) {
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const int i = i0 + u * NW;
                if (i >= L) break;
                double* row = A + pk(i, 0);
                const double vi = vv[i], wi = pp[i];
                for (int j = k + 1 + lane; j <= i; j += 32) row[j] -= fma(vi, pp[j], wi * vv[j]);
            }
        }
        __syncthreads();
    }
    if (t == 0) {
        if (L >= 2) {
            dg[L - 2] = A[pk(L - 2, L - 2)];
            e2[L - 2] = A[pk(L - 1, L - 2)];
        }
        dg[L - 1] = A[pk(L - 1, L - 1)];
    }
    __syncthreads();
    DW_MARK(1);
    // off-diagonal e_k (sign kept for the vectors) -> squares for the Sturm counts
    double* ev = pp;  // [L4] signed off-diagonal
    for (int i = t; i < L - 1; i += kDwThreads) {
        ev[i] = e2[i];
        e2[i] = e2[i] * e2[i];
    }
    __syncthreads();

    // 4. eigenvalues: Gershgorin interval, largest eigenvalue, selection size
    double glo = DBL_MAX, ghi = -DBL_MAX, emax = 0.0;
    for (int i = t; i < L; i += kDwThreads) {
        const double rad = (i > 0 ? fabs(ev[i - 1]) : 0.0) + (i < L - 1 ? fabs(ev[i]) : 0.0);
        glo = fmin(glo, dg[i] - rad);
        ghi = fmax(ghi, dg[i] + rad);
        if (i < L - 1) emax = fmax(emax, e2[i]);
    }
    glo = -block_max(-glo, red);
    ghi = block_max(ghi, red);
    emax = block_max(emax, red);
    const double tnorm = fmax(fabs(glo), fabs(ghi));
    const double pivmin = DBL_MIN * fmax(1.0, emax);
    const double pad = 2.0 * DBL_EPSILON * tnorm + 2.0 * pivmin;
    glo -= pad;
    ghi += pad;
    const double lmax = eigenvalue(dg, e2, L, L - 1, glo, ghi, pivmin, red);
    int nsel = 0;
    if (lmax > 0.0) {
        const double cut = P.frac * lmax;
        nsel = L - sturm_count(dg, e2, L, cut, pivmin);  // eigenvalues >= cut (> 0)
        if (nsel < 1) nsel = 1;
    }
    if (nsel > kDwMaxSel) {  // uniform
        if (t == 0) atomicMin(P.status, pack_failure(P.req, r * P.samples + c, HSAD_E_UNSUPPORTED));
        nsel = 0;
    }
    if (t == 0) lam[0] = lmax;
    for (int j = 1; j < nsel; ++j) {
        const double lj = eigenvalue(dg, e2, L, L - 1 - j, glo, ghi, pivmin, red);
        if (t == 0) lam[j] = lj;
    }
    __syncthreads();

    DW_MARK(2);
    // 5./6. one selected eigenvector at a time, in descending eigenvalue order:
    //   a. lane 0 of warp 0: eigenvector z of T (twisted factorisation) into a ring of the
    //      last kDwRing vectors kept in the tridiagonal basis;
    //   b. CTA: re-orthogonalise z against the ring vectors of the same cluster, normalise;
    //   c. warp 0: back-transformation v = H_0 ... H_{n-3} z (reflectors in A's columns),
    //      the sign rule (first largest-|.| component positive) and v . m_diff.
    // The xs region (the Gram's sample stage) holds the ring, v and two pivot vectors.
    double* ring = xs;                                         // [kDwRing][L4]
    double* vw = xs + static_cast<int64_t>(kDwRing) * L4;      // [L4] vector being transformed
    double* dpl = vw + L4;                                     // [L4] stationary pivots d+
    double* dmi = dpl + L4;                                    // [L4] progressive pivots d-
    for (int j = 0; j < nsel; ++j) {
        double* z = ring + static_cast<int64_t>(j % kDwRing) * L4;
        if (t == 0) {
            const double lj = lam[j];
            // T - lambda I = L D+ L^T (top down) and U D- U^T (bottom up)
            double dp = dg[0] - lj;
            for (int i = 0; i < L - 1; ++i) {
                if (fabs(dp) < pivmin) dp = -pivmin;
                dpl[i] = dp;
                dp = (dg[i + 1] - lj) - ev[i] / dp * ev[i];
            }
            if (fabs(dp) < pivmin) dp = -pivmin;
            dpl[L - 1] = dp;
            double dm = dg[L - 1] - lj;
            if (fabs(dm) < pivmin) dm = -pivmin;
            dmi[L - 1] = dm;
            int tw = L - 1;
            double gbest = fabs(dpl[L - 1]);  // gamma_{n-1} = d+_{n-1}
            for (int i = L - 2; i >= 0; --i) {
                dm = (dg[i] - lj) - ev[i] / dm * ev[i];
                if (fabs(dm) < pivmin) dm = -pivmin;
                dmi[i] = dm;
                const double gam = dpl[i] + dm - (dg[i] - lj);  // twist at i
                if (fabs(gam) < gbest) {
                    gbest = fabs(gam);
                    tw = i;
                }
            }
            // z_tw = 1; L^T rows above the twist, U^T rows below it
            z[tw] = 1.0;
            for (int i = tw - 1; i >= 0; --i) z[i] = -(ev[i] / dpl[i]) * z[i + 1];
            for (int i = tw; i < L - 1; ++i) z[i + 1] = -(ev[i] / dmi[i + 1]) * z[i];
            for (int i = L; i < L4; ++i) z[i] = 0.0;
        }
        __syncthreads();
        for (int q = j - 1; q >= 0 && q > j - kDwRing; --q) {
            if (fabs(lam[q] - lam[j]) > 1e-3 * tnorm) break;  // clusters are contiguous
            const double* zq = ring + static_cast<int64_t>(q % kDwRing) * L4;
            double part = 0.0;
            for (int i = t; i < L; i += kDwThreads) part = fma(zq[i], z[i], part);
            const double dot = block_sum(part, red);
            for (int i = t; i < L; i += kDwThreads) z[i] = fma(-dot, zq[i], z[i]);
            __syncthreads();
        }
        double part = 0.0;
        for (int i = t; i < L; i += kDwThreads) part = fma(z[i], z[i], part);
        const double inv = 1.0 / sqrt(block_sum(part, red));
        for (int i = t; i < L4; i += kDwThreads) {
            z[i] *= inv;
            vw[i] = z[i];
        }
        __syncthreads();
        if (warp == 0) {
            for (int k = L - 3; k >= 0; --k) {
                const double b = bet[k];
                if (b == 0.0) continue;
                double s2 = 0.0;
                for (int i = k + 1 + lane; i < L; i += 32) s2 = fma(A[pk(i, k)], vw[i], s2);
                for (int off = 16; off > 0; off >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, off);
                const double f = b * s2;
                for (int i = k + 1 + lane; i < L; i += 32) vw[i] = fma(-f, A[pk(i, k)], vw[i]);
                __syncwarp();
            }
            // first index of the largest |component| (stats.cpp:83-85), then v . m
            double best = -1.0, dot = 0.0;
            int bidx = L;
            for (int i = lane; i < L; i += 32) {
                const double a = fabs(vw[i]);
                if (a > best) {
                    best = a;
                    bidx = i;
                }
                dot = fma(vw[i], mu_in[i], dot);
            }
            for (int off = 16; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
                if (ob > best || (ob == best && oi < bidx)) {
                    best = ob;
                    bidx = oi;
                }
                dot += __shfl_xor_sync(0xffffffffu, dot, off);
            }
            if (lane == 0) contrib[j] = vw[bidx] < 0.0 ? -dot : dot;
        }
        __syncthreads();
    }
    DW_MARK(3);
#ifdef HSAD_DW_DEBUG
    if (t == 0 && blockIdx.x == 50 && blockIdx.y == 50)
        printf("dw phases gram %lld tridiag %lld eigvals %lld vectors %lld nsel %d\n", dbg_ph[0], dbg_ph[1],
               dbg_ph[2], dbg_ph[3], nsel);
#endif
    if (t == 0) {
        double proj = 0.0;
        for (int j = 0; j < nsel; ++j) proj += contrib[j];  // descending eigenvalue order
        const double score = fabs(proj);
        if (P.score_bytes == 8) static_cast<double*>(P.scores)[o] = score;
        else static_cast<float*>(P.scores)[o] = static_cast<float>(score);
        if (P.eigcount) P.eigcount[o] = static_cast<int8_t>(nsel);
    }
}

hsad_status fullband_dwest_launch(FbParams& P, cudaStream_t s) {
    if (P.bands > kDwMaxBands)
        return set_error(HSAD_E_UNSUPPORTED, "full-band DWEST supports at most " +
                                                 std::to_string(kDwMaxBands) + " bands");
    const int64_t rows = P.row_end - P.row_begin;
    if (rows > 65535) return set_error(HSAD_E_UNSUPPORTED, "strip too tall for one launch");
    if (rows <= 0 || P.samples <= 0) return HSAD_OK;
    const int L4 = (P.bands + 3) & ~3;
    const int64_t tri = static_cast<int64_t>(L4) * (L4 + 1) / 2;
    const int64_t nsamp = static_cast<int64_t>(P.outer) * P.outer;
    auto bytes = [&](int ch) {
        // xs must also hold the ring + 3 work vectors after the Gram
        const int64_t xs = static_cast<int64_t>(ch > kDwRing + 3 ? ch : kDwRing + 3) * L4;
        return (tri + xs + 7 * static_cast<int64_t>(L4) + 64 + 2 * kDwMaxSel + nsamp) * 8;
    };
    int chunk = 32;
    while (chunk > kDwRing + 3 && bytes(chunk) > 227 * 1024) chunk /= 2;
    if (chunk < kDwRing + 3) chunk = kDwRing + 3;
    if (bytes(chunk) > 227 * 1024)
        return set_error(HSAD_E_UNSUPPORTED, "full-band DWEST working set exceeds shared memory");
    P.chunk = chunk;
    const size_t smem = static_cast<size_t>(bytes(chunk));
    HSAD_CUDA_TRY(cudaFuncSetAttribute(fullband_dwest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
    dim3 grid(static_cast<unsigned>(P.samples), static_cast<unsigned>(rows));
    fullband_dwest_kernel<<<grid, kDwThreads, smem, s>>>(P);
    HSAD_CUDA_TRY(cudaGetLastError());
    return HSAD_OK;
}

}  // namespace hsad_b200
