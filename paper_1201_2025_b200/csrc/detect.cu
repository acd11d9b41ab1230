// K2+K3+K4: fused sliding-window statistics and per-pixel solves for Local RX,
// DWRX and DWEST (hsad::local_rx / dwrx / dwest, proj/core/src/detect.cpp:159-276;
// statistics proj/core/src/stats.cpp:7-89).
//
// The reference gathers every window explicitly (detect.cpp:83-117) and forms a
// two-pass centred covariance per pixel: O(N L^2) per pixel. Here every window
// statistic is a *box sum* of per-pixel moments m(p) = (y, upper(y y^T)), with
// y = x - s shifted by a tile-anchored reference spectrum s (translation
// invariance of the scores makes the shift exact in real arithmetic and removes
// the cancellation of S2/N - mu mu^T). Annulus = outer box - inner box, LRX
// background = box - centre position (or - guard box). Box sums are separable:
//
//   * a CTA owns a column strip of NT = TW + 2*rmax virtual columns (thread t owns
//     virtual column c0 - rmax + t, reflected with mirror_index on *global*
//     coordinates, detect.cpp:71-76) and streams down a chunk of output rows;
//   * each thread keeps the vertical window sums of its column for every box in
//     registers (fp64 running sums: + entering row, - leaving row);
//   * per output row the vertical sums go through shared memory and each output
//     thread adds its 2R+1 horizontal neighbours: the full box sums;
//   * then, still in registers, mean / covariance, ridge, 4x4 Cholesky and the
//     Mahalanobis form (LRX, DWRX) or a cyclic Jacobi eigensolve, descending
//     sort, sign rule and the DWEST selection loop.
//
// Everything is fp64. The per-pixel summation order depends only on global
// coordinates and the chunk anchoring, so row strips that start on a multiple
// of hsad_row_quantum() reproduce the single-GPU map bit for bit.
#include <cfloat>
#include <cstdlib>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "hsad_internal.h"

#ifdef HSAD_PHASE_TIMERS
__device__ unsigned long long g_phase_cycles[8];
#define PT_START() long long pt_t0 = clock64(); unsigned long long pt_acc[5] = {0, 0, 0, 0, 0}
#define PT_MARK(i)                                                    \
    do {                                                              \
        long long pt_t1 = clock64();                                  \
        pt_acc[i] += (unsigned long long)(pt_t1 - pt_t0);             \
        pt_t0 = pt_t1;                                                \
    } while (0)
#define PT_FLUSH() \
    for (int pi = 0; pi < 5; ++pi) atomicAdd(&g_phase_cycles[pi], pt_acc[pi])
#else
#define PT_START()
#define PT_MARK(i)
#define PT_FLUSH()
#endif

namespace hsad_b200 {

hsad_status fullband_launch(FbParams& P, cudaStream_t s);
hsad_status fullband_dwest_launch(FbParams& P, cudaStream_t s);

namespace {

constexpr int kCodeOverflow = 0x80;

// Boxes of at least this radius use the lane-pair horizontal sums (K = 1 kernels)
#ifndef HSAD_PAIR_RADIUS
#define HSAD_PAIR_RADIUS 2
#endif
constexpr int kPairRadius = HSAD_PAIR_RADIUS;
// Pivot ratio of C + delta I above which an LRX / DWRX pixel is recomputed two-pass
// (repair_pixel, in the counting pass).
constexpr double kRepairKappa = 1e4;
constexpr int kIllConditioned = 0x100;  // chol_quad: solved, but flag the pixel for the repair

struct ReqDev {
    int algo;         // hsad_algorithm
    int box_a;        // LRX: window box; dual: outer box
    int box_b;        // LRX: guard box or -1 (centre only); dual: inner box
    double n_a;       // LRX: background count; dual: inner count
    double n_b;       // dual: annulus count
    double ridge;
    double frac;
    void* scores;
    int score_bytes;
    int8_t* eigcount;
};

struct DetectParams {
    const void* cube;
    int elem_bytes;
    int64_t lines, samples;
    int64_t buf_row0, buf_rows;
    int64_t row_begin, row_end;
    int64_t chunk;
    int tw;
    int rmax;
    int nbox;
    int radius[kMaxBoxes];
    int nreq;
    ReqDev req[kMaxRequests];
    int std_layout;  // box 0 = LRX/outer window for every request, box 1 = inner box
    const float* raw;      // FUSE: the fp32 full-band cube (same buffer rows as `cube`) ...
    int raw_bands;         // ... its band count,
    const double* wmap;    // ... and the composed wavelet map (4 x raw_bands)
    int trio;        // std layout with exactly one LRX, one DWRX and one DWEST request ...
    int trio_q[3];   // ... at these request positions (solve_trio interleaves their solves)
    ReqDev treq[3];  // ... and their copies in LRX, DWRX, DWEST order: compile-time indices, so the
                     // solver reads ridge / fraction / map pointers straight from the constant bank
    int staged;      // STD kernel: the update rows arrive in shared memory by TMA bulk copies
    unsigned char* zflag;  // per-CTA "saw an all-zero spectrum" (fast pass -> counting pass)
    int has_dual;
    double n_in, n_ann;  // standard-layout dual counts
    unsigned long long* status;
    int req_base;       // position of req[0] in the call's request list (failure ordering)
    int64_t diag_lin;   // >= 0: pixel whose ridge delta is written to diag_out ...
    int diag_req;       // ... by this request (call position) only
    double* diag_out;
};

template <int L>
struct Dim {
    static constexpr int NC = L + L * (L + 1) / 2;  // moment channels
    static constexpr int NC2 = (NC + 1) / 2;        // channel pairs
    static constexpr int S2 = NC2 | 1;              // odd double2 stride: conflict-free LDS.128
};

// TMA row stage of the STD kernel: entering + leaving row of every box, strip width
__host__ __device__ inline size_t stage_bytes(int nbox, int64_t ncol, int bands) {
    return static_cast<size_t>(2 * nbox) * ncol * bands * sizeof(double);
}
constexpr int kFuseMapBytes = 256 * 4 * 8;  // fused DWT: the wavelet map for <= 256 bands

// nonzero-count table: NBOX x ncol ints, in double2 (16-byte) units
__host__ __device__ inline int nz_pairs(int nbox, int ncol) { return (nbox * ncol * 4 + 15) / 16; }

// Fast pass (ZC = false): set when the CTA has loaded an all-zero spectrum. Such a CTA's
// tile is recomputed by the counting pass (ZC = true), so its own error reports
// (possibly from rounding residue in all-zero windows) are suppressed.
__shared__ int s_zero_seen;

__device__ __forceinline__ void report(const DetectParams& P, int q, int64_t row, int64_t col,
                                       int code) {
    if (s_zero_seen) return;
    atomicMin(P.status, pack_failure(P.req_base + q, row * P.samples + col, code));
}

// Reflection on int32 coordinates with the in-range case first (detect.cpp:71-76).
__device__ __noinline__ int mirror32_slow(int i, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    i = abs(i) % period;
    return i < n ? i : period - i;
}
__device__ __forceinline__ int mirror32(int i, int n) {
    return static_cast<unsigned>(i) < static_cast<unsigned>(n) ? i : mirror32_slow(i, n);
}

// y = spectrum at (global row vrow, this thread's data column) as fp64;
// F64: the cube is known to be fp64 (no fp32 branch in the code)
// CG: the cube is written by this kernel (fused DWT): coherent L2 loads, not the
// read-only path
template <int L, bool F64 = false, bool CG = false>
__device__ __forceinline__ void load_row(const DetectParams& P, const char* colbase,
                                         int64_t row_bytes, int vrow, double (&y)[L]) {
    const int drow = mirror32(vrow, static_cast<int>(P.lines)) - static_cast<int>(P.buf_row0);
    const char* p = colbase + static_cast<int64_t>(drow) * row_bytes;
    if (F64 || P.elem_bytes == 8) {
        const double* d = reinterpret_cast<const double*>(p);
        if constexpr (L % 2 == 0) {
#pragma unroll
            for (int i = 0; i < L; i += 2) {
                const double2 v = CG ? __ldcg(reinterpret_cast<const double2*>(d + i))
                                     : __ldg(reinterpret_cast<const double2*>(d + i));
                y[i] = v.x;
                y[i + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < L; ++i) y[i] = __ldg(d + i);
        }
    } else {
        const float* f = reinterpret_cast<const float*>(p);
#pragma unroll
        for (int i = 0; i < L; ++i) y[i] = static_cast<double>(__ldg(f + i));
    }
}

// 1 if the (unshifted) spectrum has any nonzero band (-0.0 == 0.0), integer ops only
template <int L>
__device__ __forceinline__ int nonzero(const double (&x)[L]) {
    uint32_t lo = 0, hi = 0;  // OR of the 32-bit halves (LOP3), sign bits dropped
#pragma unroll
    for (int i = 0; i < L; ++i) {
        lo |= static_cast<uint32_t>(__double2loint(x[i]));
        hi |= static_cast<uint32_t>(__double2hiint(x[i]));
    }
    return ((hi & 0x7fffffffu) | lo) != 0u;
}

// m = (y, y_i y_j for i <= j), y already shifted
template <int L>
__device__ __forceinline__ void add_moments(double (&acc)[Dim<L>::NC], const double (&y)[L],
                                            double sign) {
    int c = L;
#pragma unroll
    for (int i = 0; i < L; ++i) acc[i] = fma(sign, y[i], acc[i]);
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = i; j < L; ++j) {
            acc[c] = fma(sign * y[i], y[j], acc[c]);
            ++c;
        }
}

template <int L>
__device__ __forceinline__ int tri(int i, int j) {  // packed upper index, i <= j
    return L + i * L - i * (i - 1) / 2 + (j - i);
}

// fp64 reciprocal: MUFU seed + two Newton steps (~1 ulp; the IEEE divide is a
// 20-instruction subroutine and nothing here needs correct rounding).
__device__ __forceinline__ double fast_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// fp64 reciprocal with one Newton step (~2^-44 relative): enough where the result
// only scales a correction that is itself ~1e-4 of its operand (polish angles)
__device__ __forceinline__ double rcp1(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return fma(y, fma(-x, y, 1.0), y);
}

// fp64 reciprocal square root: MUFU seed + two Newton steps (~1 ulp); CUDA's
// rsqrt(double) adds special-case handling this code never needs (x > 0 finite).
__device__ __forceinline__ double fast_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    return y * fma(-h * y, y, 1.5);
}

// max / min by compare-and-select (3 instructions; fmax / fmin cost ~8 with their NaN
// rules). For operands that are never NaN.
__device__ __forceinline__ double max_sel(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double min_sel(double a, double b) { return a < b ? a : b; }

// mean and covariance (divisor N) from box sums: C = S2/N - mu mu^T
// (== stats.cpp:13-29 in exact arithmetic on the shifted values). Symmetric
// matrices are stored as their upper triangle only (c[i][j], i <= j).
//
// A window whose samples are all exactly zero (no-data fill) has, in the reference's
// two-pass arithmetic, mean 0 and covariance 0 exactly; the shifted sums would leave
// rounding residue there, so `zero` (from the per-box count of nonzero spectra)
// selects the exact covariance 0. The callers resolve the cases where the mean's
// residue would decide the result (all-zero background and centre, both DWRX boxes).
template <int L>
__device__ __forceinline__ void mean_cov(const double (&s)[Dim<L>::NC], double n, double (&mu)[L],
                                         double (&c)[L][L], bool zero) {
    const double inv = fast_rcp(n);
#pragma unroll
    for (int i = 0; i < L; ++i) mu[i] = __dmul_rn(s[i], inv);  // never fused into the uses
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = i; j < L; ++j) c[i][j] = zero ? 0.0 : fma(-mu[i], mu[j], s[tri<L>(i, j)] * inv);
}

// regularized_inverse + quadratic form (stats.cpp:31-62, detect.cpp:179-180):
// delta = ridge tr(C)/L, Cholesky of C + delta I, score = |L^-1 d|^2.
// Singular rule on the pivots D_j = L_jj^2 (stats.cpp:45-48): a non-positive
// pivot, or min D <= 1e-14 max D. Only 1/L_jj is ever needed, so each column
// costs one fp64 rsqrt (MUFU seed + Newton) instead of an IEEE sqrt + divide.
// Returns 0 or an error code.
template <int L>
__device__ __forceinline__ int chol_quad(double (&a)[L][L], const double (&d)[L], double ridge,
                                         double& score, double& delta) {
    // a: upper triangle of C on entry; overwritten with U (C + delta I = U^T U)
    double tr = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) tr += a[i][i];
    delta = (L & (L - 1)) == 0 ? __dmul_rn(__dmul_rn(ridge, tr), 1.0 / L) : __ddiv_rn(__dmul_rn(ridge, tr), L);
#pragma unroll
    for (int i = 0; i < L; ++i) a[i][i] += delta;
    bool ok = true;
    double z[L], piv[L];
#pragma unroll
    for (int j = 0; j < L; ++j) {
        double p = a[j][j];
#pragma unroll
        for (int k = 0; k < j; ++k) p = fma(-a[k][j], a[k][j], p);
        ok = ok && (p > 0.0);
        piv[j] = p;
        // a non-positive pivot makes rinv inf / NaN; the pixel is rejected below
        const double rinv = fast_rsqrt(p);
#pragma unroll
        for (int i = j + 1; i < L; ++i) {
            double v = a[j][i];
#pragma unroll
            for (int k = 0; k < j; ++k) v = fma(-a[k][i], a[k][j], v);
            a[j][i] = v * rinv;
        }
        double zj = d[j];
#pragma unroll
        for (int k = 0; k < j; ++k) zj = fma(-a[k][j], z[k], zj);
        z[j] = zj * rinv;
    }
    if (!ok) return HSAD_E_SINGULAR_AFTER_RIDGE;
    double dmax = piv[0], dmin = piv[0];  // all pivots positive here
#pragma unroll
    for (int j = 1; j < L; ++j) {
        dmax = max_sel(dmax, piv[j]);
        dmin = min_sel(dmin, piv[j]);
    }
    if (dmin <= dmax * 1e-14) return HSAD_E_SINGULAR_AFTER_RIDGE;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j) s = fma(z[j], z[j], s);
    if (!isfinite(s)) return HSAD_E_SINGULAR_AFTER_RIDGE | kCodeOverflow;
    score = s;
#ifdef HSAD_NO_REPAIR
    return 0;
#else
    return dmax > kRepairKappa * dmin ? kIllConditioned : 0;
#endif
}


// Explicit fused multiply-add for float and double. Every product that feeds a sum on
// the score path is either fused here or formed with a __dmul_rn intrinsic (which
// the compiler never contracts), so all kernel instantiations round identically:
// the staged and the global-load kernels must produce bit-identical maps.
__device__ __forceinline__ float mad(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double mad(double a, double b, double c) { return __fma_rn(a, b, c); }

// Symmetric L x L matrices are kept as their upper triangle only (a[i][j], i <= j);
// sym(a, i, j) addresses element (i, j) for any order with compile-time indices,
// so rotations never write the mirrored copy.
template <int L, typename T>
__device__ __forceinline__ T& sym(T (&a)[L][L], int i, int j) {
    return i <= j ? a[i][j] : a[j][i];
}

// One Jacobi rotation zeroing (p, q) with tan t and cos c (sin = t c):
// A <- J^T A J on the upper triangle, V <- V J.
template <int L, typename T>
__device__ __forceinline__ void rotate_tc(T (&a)[L][L], T (&v)[L][L], int p, int q, T t, T c) {
    const T apq = a[p][q];
    const T s = t * c;
    a[p][p] = mad(-t, apq, a[p][p]);
    a[q][q] = mad(t, apq, a[q][q]);
    a[p][q] = T(0);
#pragma unroll
    for (int k = 0; k < L; ++k) {
        if (k == p || k == q) continue;
        T& akp = sym<L, T>(a, k, p);
        T& akq = sym<L, T>(a, k, q);
        const T x = akp, y = akq;
        akp = mad(c, x, -(s * y));
        akq = mad(s, x, c * y);
    }
#pragma unroll
    for (int k = 0; k < L; ++k) {
        const T vkp = v[k][p], vkq = v[k][q];
        v[k][p] = mad(c, vkp, -(s * vkq));
        v[k][q] = mad(s, vkp, c * vkq);
    }
}

// fp32 Jacobi angle (MUFU only): t = sgn(th)/(|th| + sqrt(th^2 + 1)),
// th = (a_qq - a_pp)/(2 a_pq); a_pq == 0 gives the identity rotation.
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Jacobi angle: t = tan(phi) of the rotation zeroing a_pq, written as
//   t = 2 a_pq sgn(h) / (|h| + sqrt(h^2 + 4 a_pq^2)),  h = a_qq - a_pp
// (the tan-half-angle form without the a_pq / h quotient): one rsqrt and one
// reciprocal, and a_pq == 0 gives t = 0 (identity rotation) directly. Only h = a_pq = 0
// makes the denominator vanish; that case is selected to t = 0.
__device__ __forceinline__ float jacobi_t32(float app, float aqq, float apq) {
    const float h = aqq - app;
    const float apq2 = apq + apq;
    const float r2 = mad(apq2, apq2, h * h);
    // h = apq = 0: r2 * rsqrt(r2) is NaN and fmaxf keeps FLT_MIN, so t = 0 * huge = 0
    const float den = fmaxf(mad(r2, rsqrtf(r2), fabsf(h)), FLT_MIN);
    const float t = apq2 * rcp_approx(den);
    // sign of h (for h = +-0 either sign zeroes a_pq)
    return __int_as_float(__float_as_int(t) ^ (__float_as_int(h) & 0x80000000));
}

// fp64 general-path angle (fast rcp/rsqrt, ~1 ulp)
__device__ __forceinline__ double jacobi_t64(double app, double aqq, double apq) {
    const double h = aqq - app;
    const double r2 = fma(4.0 * apq, apq, h * h);
    const double den = mad(r2, fast_rsqrt(r2), fabs(h));
    double t = 2.0 * apq * fast_rcp(den);
    t = h < 0.0 ? -t : t;
    return den > 0.0 ? t : 0.0;
}

// The polish sweep's general angle (some lane of the warp still has a large angle):
// rare after the fp32 stage, so kept out of line to spare the instruction cache.
__device__ __noinline__ void polish_angle_general(double app, double aqq, double apq, bool small,
                                                  double& t, double& c) {
    const double h = aqq - app;
    t = small ? (apq == 0.0 ? 0.0 : apq * fast_rcp(h)) : jacobi_t64(app, aqq, apq);
    if (small) t = t * fma(-t, t, 1.0);
    c = fast_rsqrt(fma(t, t, 1.0));
}

// Pairs of one sweep; for L = 4 in parallel order (rounds of two disjoint pairs
// {(0,1),(2,3)}, {(0,2),(1,3)}, {(0,3),(1,2)} whose angles are independent).
template <int L>
struct SweepOrder {
    static constexpr int N = L * (L - 1) / 2;
    int p[N > 0 ? N : 1], q[N > 0 ? N : 1];
    constexpr SweepOrder() : p(), q() {
        if constexpr (L == 4) {
            const int pp[6] = {0, 2, 0, 1, 0, 1}, qq[6] = {1, 3, 2, 3, 3, 2};
            for (int i = 0; i < 6; ++i) {
                p[i] = pp[i];
                q[i] = qq[i];
            }
        } else {
            int n = 0;
            for (int i = 0; i < L - 1; ++i)
                for (int j = i + 1; j < L; ++j) {
                    p[n] = i;
                    q[n] = j;
                    ++n;
                }
        }
    }
};

template <int L>
__device__ __forceinline__ void sweep32(float (&a)[L][L], float (&v)[L][L]) {
    constexpr SweepOrder<L> ord;
#pragma unroll
    for (int i = 0; i < SweepOrder<L>::N; ++i) {
        const int p = ord.p[i], q = ord.q[i];
        const float t = jacobi_t32(a[p][p], a[q][q], a[p][q]);
        rotate_tc<L, float>(a, v, p, q, t, rsqrtf(fmaf(t, t, 1.0f)));
    }
}

// L = 4 fp32 sweep with the eigenvector matrix held as packed column halves
// vv[j][h] = (V[2h][j], V[2h+1][j]): each column rotation is four FFMA2/FMUL2 pairs
// instead of eight scalar multiply-adds (Blackwell fp32x2).
__device__ __forceinline__ void sweep32_4(float (&a)[4][4], float2 (&vv)[4][2]) {
    constexpr SweepOrder<4> ord;
#pragma unroll
    for (int i = 0; i < SweepOrder<4>::N; ++i) {
        const int p = ord.p[i], q = ord.q[i];
        const float t = jacobi_t32(a[p][p], a[q][q], a[p][q]);
        const float c = rsqrtf(fmaf(t, t, 1.0f));
        const float s = t * c;
        const float apq = a[p][q];
        a[p][p] = mad(-t, apq, a[p][p]);
        a[q][q] = mad(t, apq, a[q][q]);
        a[p][q] = 0.0f;
        const float2 c2 = make_float2(c, c), s2 = make_float2(s, s), ns2 = make_float2(-s, -s);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k == p || k == q) continue;
            float& akp = sym<4, float>(a, k, p);
            float& akq = sym<4, float>(a, k, q);
            const float x = akp, y = akq;
            akp = mad(c, x, -(s * y));
            akq = mad(s, x, c * y);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float2 vp = vv[p][h], vq = vv[q][h];
            vv[p][h] = __ffma2_rn(c2, vp, __fmul2_rn(ns2, vq));
            vv[q][h] = __ffma2_rn(s2, vp, __fmul2_rn(c2, vq));
        }
    }
}

// fp64 polish sweep on a nearly diagonal matrix. When every lane of the warp
// has |a_pq| < 1e-4 |a_qq - a_pp| the angle comes from the series
// t = x (1 - x^2), x = a_pq / (a_qq - a_pp), and c = 1 - t^2/2 (both exact to
// fp64 for |x| < 1e-4); otherwise the general formula. The choice is
// warp-uniform so the cheap path costs no divergence.
template <int L>
__device__ __forceinline__ void sweep64(double (&a)[L][L], double (&v)[L][L]) {
    constexpr SweepOrder<L> ord;
#pragma unroll
    for (int i = 0; i < SweepOrder<L>::N; ++i) {
        const int p = ord.p[i], q = ord.q[i];
        const double apq = a[p][q], h = a[q][q] - a[p][p];
        const bool small = fabs(apq) < 1e-4 * fabs(h) || apq == 0.0;
        double t, c;
        if (__all_sync(__activemask(), small)) {
            const double x = apq == 0.0 ? 0.0 : apq * rcp1(h);  // 1 Newton step suffices here
            t = x * fma(-x, x, 1.0);
            c = fma(-0.5 * t, t, 1.0);
        } else {
            polish_angle_general(a[p][p], a[q][q], apq, small, t, c);
        }
        rotate_tc<L, double>(a, v, p, q, t, c);
    }
}

// symmetric_eigen (stats.cpp:64-89) for the small DWEST matrix, unsorted:
//   1. three parallel-order Jacobi sweeps in fp32 on the max-normalised matrix;
//   2. fp64 modified Gram-Schmidt of those vectors -> orthonormal Q,
//      B = Q^T A Q in fp64 (off-diagonal ~1e-6 |A|);
//   3. two fp64 polish sweeps on B (quadratic convergence to fp64 accuracy),
//      accumulated into Q.
// Returns eigenvalues w (diagonal of B) and eigenvectors V (columns), in no
// particular order: the DWEST selection below does not need them sorted.
// Stage 1 (fp32): Jacobi sweeps on the max-normalised matrix -> approximate vectors.
// UNROLL: the sweeps fully unrolled, so a caller can interleave independent work.
template <int L, bool UNROLL = false>
__device__ __forceinline__ void dwest_f32_stage(const double (&A)[L][L], float (&v32)[L][L]) {
    double amax = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = i; j < L; ++j) amax = fmax(amax, fabs(A[i][j]));
    const double scale = amax > 0.0 ? fast_rcp(amax) : 1.0;
    float a32[L][L];
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = 0; j < L; ++j) {
            a32[i][j] = j >= i ? static_cast<float>(A[i][j] * scale) : 0.0f;
            v32[i][j] = i == j ? 1.0f : 0.0f;
        }
#ifndef HSAD_F32_SWEEPS
#define HSAD_F32_SWEEPS 3
#endif
    if constexpr (L == 4) {  // measured -1.8% on the C5 sweep vs the scalar rotation
        float2 vv[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            vv[j][0] = make_float2(j == 0 ? 1.0f : 0.0f, j == 1 ? 1.0f : 0.0f);
            vv[j][1] = make_float2(j == 2 ? 1.0f : 0.0f, j == 3 ? 1.0f : 0.0f);
        }
        if constexpr (UNROLL) {
#pragma unroll
            for (int sweep = 0; sweep < HSAD_F32_SWEEPS; ++sweep) sweep32_4(a32, vv);
        } else {
#pragma unroll 1
            for (int sweep = 0; sweep < HSAD_F32_SWEEPS; ++sweep) sweep32_4(a32, vv);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v32[0][j] = vv[j][0].x;
            v32[1][j] = vv[j][0].y;
            v32[2][j] = vv[j][1].x;
            v32[3][j] = vv[j][1].y;
        }
    } else {
#pragma unroll 1
        for (int sweep = 0; sweep < (L <= 4 ? HSAD_F32_SWEEPS : 6); ++sweep) sweep32<L>(a32, v32);
    }
}

// Stage 2 (fp64): Gram-Schmidt of the fp32 vectors, B = Q^T A Q, polish sweeps.
// EXTRA: one more sweep after the off-diagonal test passes. The test is relative to |B|, so a
// pair of eigenvalues much closer than |B| keeps a rotation error of ~1e-12 |B| / gap; the
// 4-band fallback route, which exists for exactly such pairs, takes the extra (quadratically
// convergent) sweep.
template <int L, bool EXTRA = false>
__device__ __forceinline__ void dwest_f64_stage(const double (&A)[L][L], const float (&v32)[L][L],
                                                double (&V)[L][L], double (&w)[L]) {
    // modified Gram-Schmidt in fp64
#pragma unroll
    for (int j = 0; j < L; ++j) {
#pragma unroll
        for (int k = 0; k < L; ++k) V[k][j] = static_cast<double>(v32[k][j]);
#pragma unroll
        for (int i = 0; i < j; ++i) {
            double dot = 0.0;
#pragma unroll
            for (int k = 0; k < L; ++k) dot = fma(V[k][i], V[k][j], dot);
#pragma unroll
            for (int k = 0; k < L; ++k) V[k][j] = fma(-dot, V[k][i], V[k][j]);
        }
        double nrm = 0.0;
#pragma unroll
        for (int k = 0; k < L; ++k) nrm = fma(V[k][j], V[k][j], nrm);
        const double r = fast_rsqrt(nrm);
#pragma unroll
        for (int k = 0; k < L; ++k) V[k][j] *= r;
    }
    // B = V^T A V (upper triangle), one column of A V at a time
    double B[L][L];
#pragma unroll
    for (int j = 0; j < L; ++j) {
        double w[L];
#pragma unroll
        for (int i = 0; i < L; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < L; ++k) acc = fma(i <= k ? A[i][k] : A[k][i], V[k][j], acc);
            w[i] = acc;
        }
#pragma unroll
        for (int i = 0; i <= j; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < L; ++k) acc = fma(V[k][i], w[k], acc);
            B[i][j] = acc;
        }
    }
    // polish sweeps (warp-uniform) until the off-diagonal mass is below
    // (1e-12 |B|)^2: eigenvalues are then exact to ~1e-24 |B| and eigenvectors to
    // ~1e-12 / relative gap, three orders inside the 1e-9 score gate. After the fp32
    // stage (off ~1e-7) one quadratic sweep gets there; larger matrices leave fp32
    // less converged and take more
#pragma unroll 1
    for (int sweep = 0; sweep < 8; ++sweep) {
#ifdef HSAD_PHASE_TIMERS
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[7], 1ull);  // warp polish sweeps
#endif
        sweep64<L>(B, V);
        {
            double off = 0.0, dia = 0.0;
#pragma unroll
            for (int i = 0; i < L; ++i) {
                dia = fma(B[i][i], B[i][i], dia);
#pragma unroll
                for (int j = i + 1; j < L; ++j) off = fma(B[i][j], B[i][j], off);
            }
            if (__all_sync(__activemask(), off <= 1e-24 * dia)) break;
        }
    }
    if constexpr (EXTRA) sweep64<L>(B, V);
#pragma unroll
    for (int i = 0; i < L; ++i) w[i] = B[i][i];
}

template <int L, bool EXTRA = false>
__device__ __forceinline__ void dwest_eigen(const double (&A)[L][L], double (&V)[L][L], double (&w)[L]) {
    float v32[L][L];
    dwest_f32_stage<L>(A, v32);
    dwest_f64_stage<L, EXTRA>(A, v32, V, w);
}

__device__ __forceinline__ void store_score(const ReqDev& R, int64_t o, double s) {
    if (R.score_bytes == 8) static_cast<double*>(R.scores)[o] = s;
    else static_cast<float*>(R.scores)[o] = static_cast<float>(s);
}

// ---- accuracy repair of ill-conditioned LRX / DWRX pixels ----------------------------
// The shifted one-pass covariance S2/N - mu mu^T carries ~|y|^2/|C| times the rounding
// of the reference's two-pass form, and an ill-conditioned C + delta I amplifies it. A
// pixel whose Cholesky pivot ratio exceeds kRepairKappa is therefore recomputed with
// the reference's own arithmetic: the window gathered in its row-major scan order
// (detect.cpp:83-117, reflection on global coordinates), mean, two-pass centred
// covariance / N (stats.cpp:7-29), then the same ridge, Cholesky quadratic form and
// singular rule. The fast pass only marks the CTA (like a zero spectrum); the counting
// pass, which recomputes marked CTAs, repairs such pixels in place. Rare on real
// scenes (none on the C5 sweep), common only in sample-starved windows (3x3 boxes at
// mirrored corners).
template <int L>
__device__ __forceinline__ void load_px(const DetectParams& P, int64_t r, int64_t c, double (&x)[L]) {
    const int64_t rr = mirror_index(r, P.lines) - P.buf_row0;
    const int64_t cc = mirror_index(c, P.samples);
    const int64_t i = (rr * P.samples + cc) * L;
    if (P.elem_bytes == 8) {
#pragma unroll
        for (int b = 0; b < L; ++b) x[b] = static_cast<const double*>(P.cube)[i + b];
    } else {
#pragma unroll
        for (int b = 0; b < L; ++b) x[b] = static_cast<double>(static_cast<const float*>(P.cube)[i + b]);
    }
}

// window samples: |dr|, |dc| <= outer, minus |dr|, |dc| <= hole (hole < 0: none)
template <int L, typename Fn>
__device__ __forceinline__ void for_window(const DetectParams& P, int64_t r, int64_t c, int outer, int hole,
                                           Fn&& fn) {
    for (int dr = -outer; dr <= outer; ++dr)
        for (int dc = -outer; dc <= outer; ++dc) {
            if (abs(dr) <= hole && abs(dc) <= hole) continue;
            double x[L];
            load_px<L>(P, r + dr, c + dc, x);
            fn(x);
        }
}

template <int L>
__device__ __forceinline__ void window_mean_cov(const DetectParams& P, int64_t r, int64_t c, int outer,
                                                int hole, double n, double (&mu)[L], double (&cv)[L][L]) {
#pragma unroll
    for (int i = 0; i < L; ++i) mu[i] = 0.0;
    for_window<L>(P, r, c, outer, hole, [&](const double (&x)[L]) {
#pragma unroll
        for (int i = 0; i < L; ++i) mu[i] += x[i];
    });
#pragma unroll
    for (int i = 0; i < L; ++i) mu[i] /= n;
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = i; j < L; ++j) cv[i][j] = 0.0;
    for_window<L>(P, r, c, outer, hole, [&](const double (&x)[L]) {
        double d[L];
#pragma unroll
        for (int i = 0; i < L; ++i) d[i] = x[i] - mu[i];
#pragma unroll
        for (int i = 0; i < L; ++i)
#pragma unroll
            for (int j = i; j < L; ++j) cv[i][j] = fma(d[i], d[j], cv[i][j]);
    });
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = i; j < L; ++j) cv[i][j] /= n;
}

// Two-pass LRX / DWRX score of one pixel (returns 0 or an error code).
template <int L>
__device__ __noinline__ int repair_pixel(const DetectParams& P, const ReqDev& R, int64_t r, int64_t col,
                                         double& score) {
    double mu[L], cv[L][L], d[L];
    if (R.algo == HSAD_LRX) {
        const int hole = R.box_b < 0 ? 0 : P.radius[R.box_b];
        window_mean_cov<L>(P, r, col, P.radius[R.box_a], hole, R.n_a, mu, cv);
        double x[L];
        load_px<L>(P, r, col, x);
#pragma unroll
        for (int i = 0; i < L; ++i) d[i] = x[i] - mu[i];
    } else {
        double mu_in[L], cin[L][L];
        window_mean_cov<L>(P, r, col, P.radius[R.box_b], -1, R.n_a, mu_in, cin);
        window_mean_cov<L>(P, r, col, P.radius[R.box_a], P.radius[R.box_b], R.n_b, mu, cv);
#pragma unroll
        for (int i = 0; i < L; ++i) d[i] = mu_in[i] - mu[i];
    }
    double dmax = 0.0, delta = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) dmax = fmax(dmax, fabs(d[i]));
    score = 0.0;
    if (!(dmax > 0.0)) return 0;
    const int code = chol_quad<L>(cv, d, R.ridge, score, delta);
    return code == kIllConditioned ? 0 : code;
}

// ---- per-detector solves on window statistics ---------------------------------

// LRX (detect.cpp:168-188) on background sums bg, count n: score = max(d^T (C+dI)^-1 d, 0)
template <int L, bool ZC>
__device__ __forceinline__ void lrx_solve(const DetectParams& P, int q, const ReqDev& R,
                                          const double (&bg)[Dim<L>::NC], double n_bg, bool bg_zero,
                                          int nzc, const double (&yc)[L], int64_t r, int64_t col,
                                          int64_t o, int64_t lin) {
    if (bg_zero) {  // C = 0, delta = 0: d = 0 -> 0 (detect.cpp:175-177), else singular
        if (nzc) report(P, q, r, col, HSAD_E_SINGULAR_AFTER_RIDGE);
        store_score(R, o, 0.0);
        return;
    }
    double mu[L], cm[L][L], dv[L];
    mean_cov<L>(bg, n_bg, mu, cm, false);
    bool dnz = false;  // max |d_i| > 0 (detect.cpp:175)
#pragma unroll
    for (int i = 0; i < L; ++i) {
        dv[i] = yc[i] - mu[i];
        dnz = dnz | (fabs(dv[i]) > 0.0);
    }
    double score = 0.0;
    if (dnz) {
        double delta = 0.0;
        int code = chol_quad<L>(cm, dv, R.ridge, score, delta);
        if (code == kIllConditioned) {
            if constexpr (ZC) code = repair_pixel<L>(P, R, r, col, score);
            else s_zero_seen = 1, code = 0;  // the counting pass recomputes this CTA
        }
        if (P.diag_lin >= 0 && lin == P.diag_lin && P.req_base + q == P.diag_req) *P.diag_out = delta;
        if (code) {
            report(P, q, r, col, code);
            score = 0.0;
        }
    }
    store_score(R, o, fmax(score, 0.0));
}

// inner-box / annulus statistics shared by DWRX and DWEST (detect.cpp:204-213, 244-253)
template <int L>
struct DualStats {
    double c_out[L][L], cd[L][L], md[L];  // upper triangles; cd = C_in - C_ann
    bool mnz;                             // max |m_diff| > 0 (detect.cpp:211)
};
template <int L>
__device__ __forceinline__ void dual_stats(const double (&s_in)[Dim<L>::NC],
                                           const double (&s_box)[Dim<L>::NC], double n_in,
                                           double n_ann, bool in_zero, bool ann_zero,
                                           DualStats<L>& D) {
    constexpr int NC = Dim<L>::NC;
    double sann[NC], mu_in[L], mu_out[L];
#pragma unroll
    for (int c = 0; c < NC; ++c) sann[c] = s_box[c] - s_in[c];
    mean_cov<L>(s_in, n_in, mu_in, D.cd, in_zero);
    mean_cov<L>(sann, n_ann, mu_out, D.c_out, ann_zero);
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = i; j < L; ++j) D.cd[i][j] -= D.c_out[i][j];
    D.mnz = false;
    const bool both_zero = in_zero && ann_zero;  // m_diff = 0 - 0 exactly
#pragma unroll
    for (int i = 0; i < L; ++i) {
        D.md[i] = both_zero ? 0.0 : mu_in[i] - mu_out[i];
        D.mnz = D.mnz | (fabs(D.md[i]) > 0.0);
    }
}

// DWRX (detect.cpp:204-223): |m^T (C_ann + dI)^-1 m|
template <int L, bool ZC>
__device__ __forceinline__ void dwrx_solve(const DetectParams& P, int q, const ReqDev& R,
                                           const DualStats<L>& D, int64_t r, int64_t col, int64_t o,
                                           int64_t lin) {
    double score = 0.0;
    if (D.mnz) {
        double a[L][L];
#pragma unroll
        for (int i = 0; i < L; ++i)
#pragma unroll
            for (int j = i; j < L; ++j) a[i][j] = D.c_out[i][j];
        double delta = 0.0;
        int code = chol_quad<L>(a, D.md, R.ridge, score, delta);
        if (code == kIllConditioned) {
            if constexpr (ZC) code = repair_pixel<L>(P, R, r, col, score);
            else s_zero_seen = 1, code = 0;  // the counting pass recomputes this CTA
        }
        if (P.diag_lin >= 0 && lin == P.diag_lin && P.req_base + q == P.diag_req) *P.diag_out = delta;
        if (code) {
            report(P, q, r, col, code);
            score = 0.0;
        }
    }
    store_score(R, o, fabs(score));
}

// DWEST (detect.cpp:242-271): selection and projection from a full eigendecomposition.
// With eigenvalues sorted descending the reference loop sums v_i . m_diff while
// lambda_i > 0 && lambda_i >= f lambda0 and stops at the first failure
// (detect.cpp:255-262). The condition is monotone in lambda_i, so the summed set
// is exactly {i : lambda_i > 0, lambda_i >= f lambda0}: no sort needed. Sign rule
// (stats.cpp:83-85): v_i is flipped so its first largest-|.| component is positive.
template <int L>
__device__ __forceinline__ void dwest_select(double frac, const double (&md)[L], const double (&vec)[L][L],
                                             const double (&w)[L], double& score, int& count) {
    double lmax = w[0];
#pragma unroll
    for (int i = 1; i < L; ++i) lmax = fmax(lmax, w[i]);
    score = 0.0;
    count = 0;
    if (lmax > 0.0) {
        const double cut = frac * lmax;
        double proj = 0.0;
#pragma unroll
        for (int i = 0; i < L; ++i) {
            double best = fabs(vec[0][i]), lead = vec[0][i], dot = vec[0][i] * md[0];
#pragma unroll
            for (int k = 1; k < L; ++k) {
                const double av = fabs(vec[k][i]);
                lead = av > best ? vec[k][i] : lead;
                best = fmax(best, av);
                dot = fma(vec[k][i], md[k], dot);
            }
            const bool take = w[i] > 0.0 && !(w[i] < cut);
            proj += take ? (lead < 0.0 ? -dot : dot) : 0.0;
            count += take ? 1 : 0;
        }
        score = fabs(proj);
    }
}

// The general eigensolve route (any L; for L = 4 the fallback of dwest4_fast, out of
// line so the rare path stays out of the hot loop's instruction-cache footprint).
template <int L>
__device__ __forceinline__ void dwest_jacobi_body(const double (&A)[L][L], const double (&md)[L], double frac,
                                                  double& score, int& count) {
    double vec[L][L], w[L];
    dwest_eigen<L, L == 4>(A, vec, w);
    dwest_select<L>(frac, md, vec, w, score, count);
}
__device__ __forceinline__ void dwest4_scale(const double (&A)[4][4], double (&S)[4][4]);
__device__ __noinline__ void dwest_jacobi4(const double (&A)[4][4], const double (&md)[4], double frac,
                                           double& score, int& count) {
    double S[4][4];  // the power-of-two-scaled matrix, like the two-pair route: eigenvectors and the
    dwest4_scale(A, S);  // selection are scale-free, and tiny or huge covariances neither under- nor overflow
    dwest_jacobi_body<4>(S, md, frac, score, count);
}

// ---- DWEST for 4 bands without a full eigendecomposition -----------------------------
// Only the eigenpairs with lambda >= f lambda_max > 0 enter the score (one for ~83% of
// the C5 pixels, two for ~16%, three for 0.03%), so the 4 x 4 problem is solved for the
// selected pairs only (up to three), each to fp64 backward-stable accuracy (eps |A| / gap,
// like the reference's QL iteration):
//   1. scale by a power of two (exact) so max |a_ij| is in [1, 2);
//   2. tridiagonalise: one Householder reflector (column 0) + one plane rotation;
//   3. monic characteristic polynomial of the tridiagonal T; lambda_1 by Laguerre's
//      iteration from the Gershgorin bound (monotone and cubically convergent for a
//      real-rooted polynomial), lambda_2 the same way on the deflated cubic from
//      lambda_1; each then polished by Newton steps on T's three-term recurrence (a
//      backward-stable evaluation of det(T - x I), which the power-basis form is not);
//   4. eigenvector of T by the twisted factorisation in product form: column k* of
//      adj(T - lambda I) with the largest diagonal entry theta_k phi_{k+1} (leading and
//      trailing principal minors), mapped back through the rotation and the reflector;
//   5. sign rule, projection, count.
// A third selected eigenvalue (lambda_3 from the remaining quadratic, polished the same
// way) gets its own pass. Pixels the route cannot settle — an eigenvalue within 1e-6 of
// the cutoff, four selected eigenvalues, a selected eigenvalue closer than kDw4Gap (in
// units of |A|) to a neighbour, an iteration that did not converge — take the general
// Jacobi route instead (a few 1e-4 of C5).
constexpr double kDw4Gap = 3e-5;
constexpr double kDw4LagTol = 1e-6;

// sqrt of x >= 0 without the IEEE sqrt subroutine (0 -> 0)
__device__ __forceinline__ double sqrt_pos(double x) { return __dmul_rn(x, fast_rsqrt(x + DBL_MIN)); }
// One Laguerre step a = n p / (p' + w sqrt(D)) with D = p'^2 - n/(n-1) p p'' (so that
// w = n - 1). Right of the largest root of a real-rooted monic polynomial p, p' > 0 and
// the iteration descends monotonically, so the sign of the root is fixed. sqrt and the
// quotient come straight from the MUFU seeds (~2^-20): an error of that size in a step
// only shows up as a 1e-6 |a| error of the iterate, and the Newton polish on the
// recurrence follows. D <= 0 (all roots equal, e.g. the zero matrix) gives NaN, which
// fails every convergence test below: such pixels take the general route.
__device__ __forceinline__ double laguerre_step(double p, double dp, double D, double w, double n) {
    double rs, rc;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(D));
    const double den = fma(__dmul_rn(D, w), rs, dp);
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(den));
    return __dmul_rn(__dmul_rn(p, n), rc);
}

struct Tri4 {
    double d[4], e[3], f[3];  // diagonal, off-diagonal, off-diagonal squared
    double v0, v1, v2, beta;  // reflector on coordinates 1..3: H = I - beta v v^T
    double c, s;              // rotation on coordinates 2, 3
};

// det(T - x I) and its derivative by the three-term recurrence
__device__ __forceinline__ void tri4_eval(const Tri4& T, double x, double& p, double& dp) {
    const double g0 = T.d[0] - x, g1 = T.d[1] - x, g2 = T.d[2] - x, g3 = T.d[3] - x;
    const double t1 = g0;
    const double t2 = fma(g1, t1, -T.f[0]);
    const double u2 = -g1 - t1;                                // dt2 = g1 dt1 - t1, dt1 = -1
    const double t3 = fma(g2, t2, __dmul_rn(-T.f[1], t1));
    const double u3 = fma(g2, u2, T.f[1] - t2);                // g2 dt2 - t2 - f1 dt1
    p = fma(g3, t3, __dmul_rn(-T.f[2], t2));
    dp = fma(g3, u3, fma(-T.f[2], u2, -t3));
}

// Newton polish of an eigenvalue estimate on the recurrence; returns false when it did
// not settle (a multiple root: the caller falls back)
__device__ __forceinline__ bool tri4_polish(const Tri4& T, double& x) {
    double st = 1.0;
#pragma unroll 1
    for (int it = 0; it < 4 && fabs(st) > 1e-9; ++it) {
        double p, dp;
        tri4_eval(T, x, p, dp);
        st = dp != 0.0 ? __dmul_rn(p, fast_rcp(dp)) : 0.0;
        x -= st;
    }
    return fabs(st) <= 1e-9;
}

// signed projection sigma (v . md) of T's eigenvector at lam, back in A's coordinates
__device__ __forceinline__ double tri4_project(const Tri4& T, double lam, const double (&md)[4]) {
    const double g0 = T.d[0] - lam, g1 = T.d[1] - lam, g2 = T.d[2] - lam, g3 = T.d[3] - lam;
    const double th1 = g0;
    const double th2 = fma(g1, th1, -T.f[0]);
    const double th3 = fma(g2, th2, __dmul_rn(-T.f[1], th1));
    const double ph3 = g3;
    const double ph2 = fma(g2, ph3, -T.f[2]);
    const double ph1 = fma(g1, ph2, __dmul_rn(-T.f[1], ph3));
    // adj(T - lam I), upper triangle
    const double t01 = __dmul_rn(T.e[0], T.e[1]), t12 = __dmul_rn(T.e[1], T.e[2]);
    const double h1 = __dmul_rn(th1, T.e[1]);
    const double a00 = ph1, a11 = __dmul_rn(th1, ph2), a22 = __dmul_rn(th2, ph3), a33 = th3;
    const double a01 = __dmul_rn(-T.e[0], ph2), a02 = __dmul_rn(t01, ph3), a03 = __dmul_rn(-t01, T.e[2]);
    const double a12 = __dmul_rn(-h1, ph3), a13 = __dmul_rn(th1, t12), a23 = __dmul_rn(-th2, T.e[2]);
    // the column with the largest diagonal entry (the twist index)
    double best = fabs(a00), z0 = a00, z1 = a01, z2 = a02, z3 = a03;
    bool b = fabs(a11) > best;
    best = b ? fabs(a11) : best;
    z0 = b ? a01 : z0, z1 = b ? a11 : z1, z2 = b ? a12 : z2, z3 = b ? a13 : z3;
    b = fabs(a22) > best;
    best = b ? fabs(a22) : best;
    z0 = b ? a02 : z0, z1 = b ? a12 : z1, z2 = b ? a22 : z2, z3 = b ? a23 : z3;
    b = fabs(a33) > best;
    z0 = b ? a03 : z0, z1 = b ? a13 : z1, z2 = b ? a23 : z2, z3 = b ? a33 : z3;
    // back through the rotation (coordinates 2, 3) and the reflector (coordinates 1..3)
    const double y2 = fma(T.c, z2, __dmul_rn(-T.s, z3));
    const double y3 = fma(T.s, z2, __dmul_rn(T.c, z3));
    const double tt = __dmul_rn(T.beta, fma(T.v2, y3, fma(T.v1, y2, __dmul_rn(T.v0, z1))));
    const double x0 = z0, x1 = fma(-tt, T.v0, z1), x2 = fma(-tt, T.v1, y2), x3 = fma(-tt, T.v2, y3);
    const double n2 = fma(x3, x3, fma(x2, x2, fma(x1, x1, __dmul_rn(x0, x0))));
    const double dot = fma(x3, md[3], fma(x2, md[2], fma(x1, md[1], __dmul_rn(x0, md[0]))));
    // sign rule: the first largest-|.| component positive
    double lead = x0, bl = fabs(x0);
    b = fabs(x1) > bl;
    lead = b ? x1 : lead, bl = b ? fabs(x1) : bl;
    b = fabs(x2) > bl;
    lead = b ? x2 : lead, bl = b ? fabs(x2) : bl;
    lead = fabs(x3) > bl ? x3 : lead;
    const double pr = __dmul_rn(dot, fast_rsqrt(n2 + DBL_MIN));
    return lead < 0.0 ? -pr : pr;
}

// 1. exact power-of-two scaling: max |a_ij| -> [1, 2) (upper triangle)
__device__ __forceinline__ void dwest4_scale(const double (&A)[4][4], double (&S)[4][4]) {
    unsigned hmax = 0u;  // only the exponent of max |a_ij| matters: compare the high words
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i; j < 4; ++j) hmax = max(hmax, static_cast<unsigned>(__double2hiint(A[i][j])) & 0x7fffffffu);
    const int ex = static_cast<int>(hmax >> 20);
    const double sc = __hiloint2double((2046 - ex) << 20, 0);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i; j < 4; ++j) S[i][j] = A[i][j] * sc;
}

// Returns false when the pixel needs the general route.
__device__ __forceinline__ bool dwest4_fast(const double (&A)[4][4], const double (&md)[4], double frac,
                                            double& score, int& count) {
    double S[4][4];
    dwest4_scale(A, S);
    const double a00 = S[0][0], a01 = S[0][1], a02 = S[0][2], a03 = S[0][3];
    const double a11 = S[1][1], a12 = S[1][2], a13 = S[1][3];
    const double a22 = S[2][2], a23 = S[2][3], a33 = S[3][3];
    // 2. tridiagonal form
    Tri4 T;
    {
        const double nx = sqrt_pos(fma(a03, a03, fma(a02, a02, __dmul_rn(a01, a01))));
        const double alpha = a01 >= 0.0 ? -nx : nx;
        T.v0 = a01 - alpha, T.v1 = a02, T.v2 = a03;
        const double vv = fma(T.v2, T.v2, fma(T.v1, T.v1, __dmul_rn(T.v0, T.v0)));
        T.beta = vv > 0.0 ? 2.0 * fast_rcp(vv) : 0.0;
        const double p0 = __dmul_rn(T.beta, fma(a13, T.v2, fma(a12, T.v1, __dmul_rn(a11, T.v0))));
        const double p1 = __dmul_rn(T.beta, fma(a23, T.v2, fma(a22, T.v1, __dmul_rn(a12, T.v0))));
        const double p2 = __dmul_rn(T.beta, fma(a33, T.v2, fma(a23, T.v1, __dmul_rn(a13, T.v0))));
        const double K = __dmul_rn(0.5 * T.beta, fma(T.v2, p2, fma(T.v1, p1, __dmul_rn(T.v0, p0))));
        const double w0 = fma(-K, T.v0, p0), w1 = fma(-K, T.v1, p1), w2 = fma(-K, T.v2, p2);
        const double b11 = fma(-2.0 * T.v0, w0, a11);
        const double b12 = fma(-w0, T.v1, fma(-T.v0, w1, a12));
        const double b13 = fma(-w0, T.v2, fma(-T.v0, w2, a13));
        const double b22 = fma(-2.0 * T.v1, w1, a22);
        const double b23 = fma(-w1, T.v2, fma(-T.v1, w2, a23));
        const double b33 = fma(-2.0 * T.v2, w2, a33);
        T.d[0] = a00, T.e[0] = alpha, T.d[1] = b11;
        const double r2 = fma(b13, b13, __dmul_rn(b12, b12));
        const double rinv = fast_rsqrt(r2 + DBL_MIN);
        T.c = r2 > 0.0 ? __dmul_rn(b12, rinv) : 1.0;
        T.s = r2 > 0.0 ? __dmul_rn(b13, rinv) : 0.0;
        T.e[1] = __dmul_rn(r2, rinv);
        const double cc = __dmul_rn(T.c, T.c), ss = __dmul_rn(T.s, T.s), cs2 = __dmul_rn(2.0 * T.c, T.s);
        T.d[2] = fma(ss, b33, fma(cs2, b23, __dmul_rn(cc, b22)));
        T.d[3] = fma(cc, b33, fma(-cs2, b23, __dmul_rn(ss, b22)));
        T.e[2] = fma(0.5 * cs2, b33 - b22, __dmul_rn(cc - ss, b23));
#pragma unroll
        for (int i = 0; i < 3; ++i) T.f[i] = __dmul_rn(T.e[i], T.e[i]);
    }
    // 3. monic characteristic polynomial x^4 + c3 x^3 + c2 x^2 + c1 x + c0
    const double p21 = -(T.d[0] + T.d[1]), p20 = fma(T.d[0], T.d[1], -T.f[0]);
    const double p32 = p21 - T.d[2];
    const double p31 = fma(-T.d[2], p21, p20 - T.f[1]);
    const double p30 = fma(T.f[1], T.d[0], __dmul_rn(-T.d[2], p20));
    const double c3 = p32 - T.d[3];
    const double c2 = fma(-T.d[3], p32, p31 - T.f[2]);
    const double c1 = fma(-T.f[2], p21, fma(-T.d[3], p31, p30));
    const double c0 = fma(-T.f[2], p20, __dmul_rn(-T.d[3], p30));
    //    lambda_1: Laguerre from the Gershgorin upper bound
    const double ae0 = fabs(T.e[0]), ae2 = fabs(T.e[2]);  // e[1] >= 0
    double x = max_sel(max_sel(T.d[0] + ae0, T.d[1] + (ae0 + T.e[1])), max_sel(T.d[2] + (T.e[1] + ae2), T.d[3] + ae2));
    bool ok = true;
    {
        const double k3 = 3.0 * c3, k2 = 2.0 * c2;
        double a = 1.0;
        int it = 0;
#pragma unroll 1
        for (; it < 12 && fabs(a) > kDw4LagTol; ++it) {
            const double p = fma(fma(fma(x + c3, x, c2), x, c1), x, c0);
            const double dp = fma(fma(fma(4.0, x, k3), x, k2), x, c1);
            const double hp = fma(fma(6.0, x, k3), x, c2);  // p'' / 2
            // a = n p / (p' + sqrt((n-1)((n-1) p'^2 - n p p''))), n = 4
            a = laguerre_step(p, dp, fma(__dmul_rn(p, -8.0 / 3.0), hp, __dmul_rn(dp, dp)), 3.0, 4.0);
            x -= a;
        }
        ok = fabs(a) <= kDw4LagTol;
    }
    double lam1 = x;
    ok = tri4_polish(T, lam1) && ok;
    score = 0.0;
    count = 0;
    if (!(lam1 > 0.0)) return ok;  // no positive eigenvalue: score 0 (detect.cpp:254)
    //    lambda_2 on the deflated cubic x^3 + q2 x^2 + q1 x + q0, from lambda_1
    const double q2 = c3 + lam1, q1 = fma(lam1, q2, c2), q0 = fma(lam1, q1, c1);
    {
        const double k2 = 2.0 * q2;
        double a = 1.0;
        int it = 0;
        x = lam1;
#pragma unroll 1
        for (; it < 12 && fabs(a) > kDw4LagTol; ++it) {
            const double p = fma(fma(x + q2, x, q1), x, q0);
            const double dp = fma(fma(3.0, x, k2), x, q1);
            const double hp = fma(3.0, x, q2);  // p'' / 2
            a = laguerre_step(p, dp, fma(__dmul_rn(p, -3.0), hp, __dmul_rn(dp, dp)), 2.0, 3.0);  // n = 3
            x -= a;
        }
        ok = ok && fabs(a) <= kDw4LagTol;
    }
    double lam2 = x;
    ok = tri4_polish(T, lam2) && ok;
    //    lambda_3 >= lambda_4 from the remaining quadratic x^2 + r1 x + r0
    const double r1 = q2 + lam2, r0 = fma(lam2, r1, q1);
    double lam3 = 0.5 * (sqrt_pos(fmax(fma(r1, r1, -4.0 * r0), 0.0)) - r1);
    const double cut = __dmul_rn(frac, lam1);
    const double margin = fma(1e-6, cut, 1e-9);  // an eigenvalue this close to the cutoff: general route
    const bool take2 = lam2 > 0.0 && !(lam2 < cut);
    bool take3 = false;
    if (take2 && lam3 > cut + margin) {  // a third selected eigenvalue (0.03% of the C5 pixels)
        take3 = true;
        const double lam4 = -r1 - lam3;  // before the polish: the quadratic's own pair
        ok = tri4_polish(T, lam3) && ok && lam4 < cut - margin && lam3 - lam4 >= kDw4Gap;
    } else {
        ok = ok && lam3 < cut - margin;
    }
    // the route settles the pixel when no eigenvalue sits at the cutoff and every selected
    // eigenvalue is clear of its neighbours
    ok = ok && lam1 - lam2 >= kDw4Gap && (!take2 || lam2 - lam3 >= kDw4Gap);
    // 4./5. eigenvectors, sign rule, projection: one pass per selected eigenvalue
    count = take3 ? 3 : take2 ? 2 : 1;
    double proj = 0.0;
#pragma unroll 1
    for (int k = 0; k < count; ++k) proj += tri4_project(T, k == 0 ? lam1 : k == 1 ? lam2 : lam3, md);
    score = fabs(proj);
    return ok;
}

// DWEST score and eigen-count of one pixel from C_in - C_ann and m_in - m_ann
template <int L>
__device__ __forceinline__ void dwest_score(const double (&A)[L][L], const double (&md)[L], double frac,
                                            double& score, int& count) {
    if constexpr (L == 4) {
        double s1 = 0.0;
        int c1 = 0;
#ifndef HSAD_DWEST_JACOBI
        if (!dwest4_fast(A, md, frac, s1, c1))
#endif
        {
            // the out-of-line route takes its arguments in local memory: copy them here, in the
            // rare branch, so the common path keeps the statistics in registers
            double Ac[4][4], mc[4], s2;
            int c2;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                mc[i] = md[i];
#pragma unroll
                for (int j = i; j < 4; ++j) Ac[i][j] = A[i][j];
            }
            dwest_jacobi4(Ac, mc, frac, s2, c2);
            s1 = s2;
            c1 = c2;
        }
        score = s1;
        count = c1;
    } else {
        dwest_jacobi_body<L>(A, md, frac, score, count);
    }
}

template <int L>
__device__ __forceinline__ void dwest_solve(const ReqDev& R, const DualStats<L>& D, int64_t o) {
    double score;
    int count;
    dwest_score<L>(D.cd, D.md, R.frac, score, count);
    store_score(R, o, score);
    if (R.eigcount) R.eigcount[o] = static_cast<int8_t>(count);
}

// symmetric_eigen + the DWEST selection loop (stats.cpp:64-89, detect.cpp:252-263) on a
// batch of 4 x 4 matrices: one thread per (C_diff, m_diff) pair, the same device code
// path as the fused detector (hsad_dwest_pairs).
__global__ void dwest_pairs_kernel(const double* __restrict__ cdiff, const double* __restrict__ mdiff,
                                   int64_t n, double frac, double* __restrict__ scores,
                                   int8_t* __restrict__ counts, int8_t* __restrict__ route) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double A[4][4], md[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        md[r] = mdiff[i * 4 + r];
#pragma unroll
        for (int c = r; c < 4; ++c) A[r][c] = cdiff[i * 16 + r * 4 + c];  // upper triangle
    }
    double score;
    int count;
    bool fast = dwest4_fast(A, md, frac, score, count);
#ifdef HSAD_DWEST_JACOBI
    fast = false;
#endif
    if (!fast) dwest_jacobi4(A, md, frac, score, count);
    scores[i] = score;
    if (counts) counts[i] = static_cast<int8_t>(count);
    if (route) route[i] = fast ? 0 : 1;
}

template <int NBOX>
__device__ __forceinline__ int select_cnt(const int (&cnt)[NBOX], int k) {
    int v = cnt[0];
#pragma unroll
    for (int kk = 1; kk < NBOX; ++kk)
        if (k == kk) v = cnt[kk];
    return v;
}

template <int L, int NBOX>
__device__ __forceinline__ void select_box(const double (&S)[NBOX][Dim<L>::NC], int k,
                                           double (&out)[Dim<L>::NC]) {
#pragma unroll
    for (int c = 0; c < Dim<L>::NC; ++c) out[c] = S[0][c];
#pragma unroll
    for (int kk = 1; kk < NBOX; ++kk)
        if (k == kk) {
#pragma unroll
            for (int c = 0; c < Dim<L>::NC; ++c) out[c] = S[kk][c];
        }
}

// The standard trio (one LRX on the outer window, one DWRX and one DWEST on (outer,
// inner)): the three solves without the per-request dispatch of the general path, the
// LRX and DWRX Cholesky chains side by side so the scheduler can interleave them. Same
// per-value arithmetic as lrx_solve / dwrx_solve / dwest_solve, so results are
// bit-identical to those paths.
template <int L, bool ZC>
__device__ __forceinline__ void solve_trio(const DetectParams& P, const ReqDev* s_req,
                                           const double (&S0)[Dim<L>::NC], const double (&S1)[Dim<L>::NC],
                                           int cnt0, int cnt1, int nzc, const double (&yc)[L], int64_t r,
                                           int64_t col, int64_t o, int64_t lin) {
    constexpr int NC = Dim<L>::NC;
    const int qL = P.trio_q[0], qR = P.trio_q[1];
    const ReqDev& RL = P.treq[0];
    const ReqDev& RR = P.treq[1];
    const ReqDev& RE = P.treq[2];
    double bg[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) bg[c] = S0[c];
    add_moments<L>(bg, yc, -1.0);
    const bool bg_zero = ZC && cnt0 - nzc == 0;
    double muL[L], cm[L][L], dv[L];
    mean_cov<L>(bg, RL.n_a, muL, cm, false);
    bool dnzL = false;
#pragma unroll
    for (int i = 0; i < L; ++i) {
        dv[i] = yc[i] - muL[i];
        dnzL = dnzL | (fabs(dv[i]) > 0.0);
    }
    DualStats<L> D;
    dual_stats<L>(S1, S0, P.n_in, P.n_ann, ZC && cnt1 == 0, ZC && cnt0 - cnt1 == 0, D);
    double a[L][L];
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = i; j < L; ++j) a[i][j] = D.c_out[i][j];
    // the LRX and DWRX solves
    double scoreL = 0.0, deltaL = 0.0, scoreR = 0.0, deltaR = 0.0;
    int codeL = chol_quad<L>(cm, dv, RL.ridge, scoreL, deltaL);
    int codeR = chol_quad<L>(a, D.md, RR.ridge, scoreR, deltaR);
    // LRX epilogue (lrx_solve)
    if (bg_zero) {
        if (nzc) report(P, qL, r, col, HSAD_E_SINGULAR_AFTER_RIDGE);
        store_score(RL, o, 0.0);
    } else {
        double score = 0.0;
        if (dnzL) {
            score = scoreL;
            if (codeL == kIllConditioned) {
                if constexpr (ZC) codeL = repair_pixel<L>(P, RL, r, col, score);
                else s_zero_seen = 1, codeL = 0;
            }
            if (codeL) {
                report(P, qL, r, col, codeL);
                score = 0.0;
            }
        }
        store_score(RL, o, fmax(score, 0.0));
    }
    // DWRX epilogue (dwrx_solve)
    {
        double score = 0.0;
        if (D.mnz) {
            score = scoreR;
            if (codeR == kIllConditioned) {
                if constexpr (ZC) codeR = repair_pixel<L>(P, RR, r, col, score);
                else s_zero_seen = 1, codeR = 0;
            }
            if (codeR) {
                report(P, qR, r, col, codeR);
                score = 0.0;
            }
        }
        store_score(RR, o, fabs(score));
    }
    // DWEST (dwest_solve)
#ifdef HSAD_EXP_NODWEST  // experiment: the kernel without the eigensolve (lower bound)
    store_score(RE, o, D.cd[0][0]);
#else
    dwest_solve<L>(RE, D, o);
#endif
}

// Per-pixel solves of every request from the box sums S (detect.cpp:168-271).
// Requests come from shared memory (s_req). In the standard layout — box 0 the
// shared outer/LRX window, box 1 the inner box, LRX excluding only the centre —
// box indices are compile-time and the inner/annulus statistics are computed
// once for DWRX and DWEST; other layouts select boxes at run time.
template <int L, int NBOX, bool STD, bool ZC, bool TRIO = false>
__device__ __forceinline__ void solve_pixel(const DetectParams& P, const ReqDev* s_req,
                                            const double (&S)[NBOX][Dim<L>::NC],
                                            const int (&cnt)[NBOX], int nzc, const double (&yc)[L],
                                            int64_t r, int64_t col) {
    // cnt[k]: nonzero spectra in box k; nzc: the centre spectrum is nonzero
    constexpr int NC = Dim<L>::NC;
    const int64_t o = (r - P.row_begin) * P.samples + col;
    const int64_t lin = r * P.samples + col;
    if constexpr (TRIO && NBOX == 2) {  // a kernel for the trio alone (no general paths: smaller code)
        solve_trio<L, ZC>(P, s_req, S[0], S[1], cnt[0], cnt[1], nzc, yc, r, col, o, lin);
        return;
    }
    if (STD || P.std_layout) {
        if constexpr (NBOX == 2) {
            if (P.trio) {
                solve_trio<L, ZC>(P, s_req, S[0], S[1], cnt[0], cnt[1], nzc, yc, r, col, o, lin);
                return;
            }
        }
        for (int q = 0; q < P.nreq; ++q) {
            const ReqDev& R = s_req[q];
            if (R.algo != HSAD_LRX) continue;
            double bg[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) bg[c] = S[0][c];
            add_moments<L>(bg, yc, -1.0);
            lrx_solve<L, ZC>(P, q, R, bg, R.n_a, ZC && cnt[0] - nzc == 0, nzc, yc, r, col, o, lin);
        }
#ifdef HSAD_PHASE_TIMERS
        long long q0 = clock64();  // phases 5/6 sampled on thread 0 of each CTA (x128)
#endif
        if constexpr (NBOX >= 2) {
            if (P.has_dual) {
                DualStats<L> D;
                dual_stats<L>(S[1], S[0], P.n_in, P.n_ann, ZC && cnt[1] == 0, ZC && cnt[0] - cnt[1] == 0, D);
                for (int q = 0; q < P.nreq; ++q)  // DWRX first: C_ann dies before the eigensolve
                    if (s_req[q].algo == HSAD_DWRX) dwrx_solve<L, ZC>(P, q, s_req[q], D, r, col, o, lin);
#ifdef HSAD_PHASE_TIMERS
                long long q1 = clock64();
                if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[5], 128ull * (q1 - q0));
#endif
                for (int q = 0; q < P.nreq; ++q)
                    if (s_req[q].algo == HSAD_DWEST) dwest_solve<L>(s_req[q], D, o);
#ifdef HSAD_PHASE_TIMERS
                if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[6], 128ull * (clock64() - q1));
#endif
            }
        }
        return;
    }
    if constexpr (!STD) {  // general layouts: boxes selected at run time
        for (int q = 0; q < P.nreq; ++q) {
            const ReqDev& R = s_req[q];
            if (R.algo == HSAD_LRX) {
                double bg[NC];
                select_box<L, NBOX>(S, R.box_a, bg);
                int nz_bg = select_cnt<NBOX>(cnt, R.box_a);
                if (R.box_b < 0) {
                    add_moments<L>(bg, yc, -1.0);
                    nz_bg -= nzc;
                } else {
                    double g[NC];
                    select_box<L, NBOX>(S, R.box_b, g);
#pragma unroll
                    for (int c = 0; c < NC; ++c) bg[c] -= g[c];
                    nz_bg -= select_cnt<NBOX>(cnt, R.box_b);
                }
                lrx_solve<L, ZC>(P, q, R, bg, R.n_a, ZC && nz_bg == 0, nzc, yc, r, col, o, lin);
            } else {
                double s_in[NC], s_box[NC];
                select_box<L, NBOX>(S, R.box_b, s_in);
                select_box<L, NBOX>(S, R.box_a, s_box);
                const int nz_in = select_cnt<NBOX>(cnt, R.box_b);
                const int nz_box = select_cnt<NBOX>(cnt, R.box_a);
                DualStats<L> D;
                dual_stats<L>(s_in, s_box, R.n_a, R.n_b, ZC && nz_in == 0, ZC && nz_box - nz_in == 0, D);
                if (R.algo == HSAD_DWRX) dwrx_solve<L, ZC>(P, q, R, D, r, col, o, lin);
                else dwest_solve<L>(R, D, o);
            }
        }
    }
}

// Column-strip streaming kernel. A CTA of NT threads owns TW = NT*K output columns
// (thread t: strip columns [tK, tK+K)) plus rmax halo columns on each side, and
// walks down a chunk of output rows:
//   1. vertical window sums of every strip column (+halo) for every box live in
//      shared memory; each step, thread t updates columns t, t+NT, ... with the
//      entering row minus the leaving row (fp64 moments of shifted spectra);
//   2. barrier; thread t slides a horizontal running sum over its K columns
//      (2R+1 terms once, then +1/-1 per column), so each output costs O(1) per
//      box instead of O(R); at each of its columns it solves LRX/DWRX/DWEST;
//   3. barrier before the next row's update.
// Smem column stride: S2 double2 per column plus one pad pair after every K
// columns, so the per-thread segments (stride K columns) hit distinct banks.
// Fused DWT: one reduced row of the strip (global row `grow`, already
// inside the image) from the fp32 full-band rows, written to the reduced buffer. The
// arithmetic is K1's lane-split kernel's exactly (reduce.cu: lane l accumulates bands
// l + 32 s in s order for each of 8 pixels, then the same 31-shuffle butterfly), so the
// reduced values are bit-identical to hsad_reduce's. Warps take groups of 8 strip columns.
__device__ __forceinline__ void fused_dwt_row(const DetectParams& P, const double* wsm, int64_t grow,
                                              int64_t c0, int ncol) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int RB = P.raw_bands, bpl = (RB + 31) >> 5;
    const int64_t drow = grow - P.buf_row0;
    double* red = const_cast<double*>(static_cast<const double*>(P.cube));
    for (int g = warp; g * 8 < ncol; g += nwarps) {
        double v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = min(g * 8 + j, ncol - 1);  // a repeated column past the strip: dropped below
            const int dcol = mirror32(static_cast<int>(c0 - P.rmax + c), static_cast<int>(P.samples));
            const float* px = P.raw + (drow * P.samples + dcol) * RB;
#pragma unroll 8
            for (int s2 = 0; s2 < 8; ++s2) {
                if (s2 >= bpl) break;
                const int b = lane + 32 * s2;
                const double x = b < RB ? static_cast<double>(__ldg(px + b)) : 0.0;
                const double* w = wsm + (s2 * 32 + lane) * 4;
#pragma unroll
                for (int k = 0; k < 4; ++k) v[j * 4 + k] = fma(w[k], x, v[j * 4 + k]);
            }
        }
        // butterfly reduce-scatter (reduce.cu): lane l ends with output l = (pixel l/4, band l%4)
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
        const int c = g * 8 + (lane >> 2);
        if (c < ncol) {
            const int dcol = mirror32(static_cast<int>(c0 - P.rmax + c), static_cast<int>(P.samples));
            red[(drow * P.samples + dcol) * 4 + (lane & 3)] = v[0];
        }
    }
    // the rows are read back by this CTA's TMA bulk copies (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int L, int NBOX, int K, bool STD, bool ZC, bool FUSE = false, bool TRIO = false>
// 4 resident CTAs (16 warps) per SM: the per-pixel solves are chains of dependent
// fp64 operations, and extra warps hide their latency better than the registers
// a larger budget would save (measured: 4.35 vs 5.52 ms for LRX+DWRX+DWEST on C5).
#ifndef HSAD_DET_NT
#define HSAD_DET_NT 128  // threads (= output columns at K = 1) per CTA
#endif
#ifndef HSAD_DET_MINB
#define HSAD_DET_MINB 4
#endif
__device__ __forceinline__ void detect_tile(const DetectParams& P, int bx, int by, int nbx) {
    constexpr int NC = Dim<L>::NC;
    constexpr int NC2 = Dim<L>::NC2;
    constexpr int S2 = Dim<L>::S2;
    extern __shared__ double2 s_v2[];
    __shared__ ReqDev s_req[kMaxRequests];
    __shared__ uint64_t s_bar;  // STD: stage-full barrier of the row-update copies

    const int t = threadIdx.x;
    const int NT = blockDim.x;
    if constexpr (ZC) {  // counting pass after a fast pass: only the CTAs that met zeros
        if (P.zflag && !P.zflag[static_cast<int64_t>(by) * nbx + bx]) return;
    }
    if (t < P.nreq) s_req[t] = P.req[t];  // dynamic request index -> shared memory
    if (t == 0) s_zero_seen = 0;
    __syncthreads();

    const int ncol = P.tw + 2 * P.rmax;            // strip columns incl. halo
    // pairs per box: S2 (odd) per column + one pad pair per K columns when K > 1,
    // so a thread-to-thread stride of K*S2 + 1 pairs stays odd (conflict-free LDS.128)
    const int box_stride = ncol * S2 + (K > 1 ? ncol / K + 1 : 0);
    auto vslot = [&](int k, int c) -> double2* {    // c: strip column index 0..ncol-1
        return s_v2 + k * box_stride + c * S2 + (K > 1 ? c / K : 0);
    };
    const int64_t c0 = static_cast<int64_t>(bx) * P.tw;  // first output column
    const int64_t ra = P.row_begin + static_cast<int64_t>(by) * P.chunk;
    const int64_t rb = min(ra + P.chunk, P.row_end);
    if (ra >= rb) return;
    const int64_t row_bytes = P.samples * L * P.elem_bytes;

    const int64_t st_lo = c0 - P.rmax > 0 ? c0 - P.rmax : 0;
    const int64_t st_hi = c0 + P.tw + P.rmax < P.samples ? c0 + P.tw + P.rmax : P.samples;
    // per strip column and box: nonzero spectra in the column's vertical window (kept
    // like the window sums: + entering row, - leaving row)
    int* s_nz = reinterpret_cast<int*>(s_v2 + NBOX * box_stride);  // [NBOX][ncol]
    double* stage = reinterpret_cast<double*>(s_v2 + NBOX * box_stride + nz_pairs(NBOX, ncol));
    const double* wsm = stage + stage_bytes(NBOX, ncol, L) / sizeof(double);  // FUSE: wavelet map
    if constexpr (FUSE) {
        // the composed map, band-major: wsm[b][k] (lane-contiguous for the DWT)
        double* w = const_cast<double*>(wsm);
        for (int e = t; e < 256 * 4; e += NT) {
            const int b = e >> 2, k = e & 3;
            w[e] = b < P.raw_bands ? P.wmap[k * P.raw_bands + b] : 0.0;
        }
        __syncthreads();
        // warm-up: the reduced rows the first window and the first staged update read
        for (int64_t d = -P.radius[0]; d <= P.radius[0] + 1; ++d)
            fused_dwt_row(P, wsm, mirror32(static_cast<int>(ra + d), static_cast<int>(P.lines)), c0, ncol);
        __syncthreads();
    }
    // tile-anchored shift: the spectrum at (ra, c0)
    double shift[L];
    {
        double y[L];
        load_row<L, STD, FUSE>(P, static_cast<const char*>(P.cube) + c0 * L * P.elem_bytes, row_bytes,
                    static_cast<int>(ra), y);
#pragma unroll
        for (int i = 0; i < L; ++i) shift[i] = y[i];
    }
    auto colbase_of = [&](int c) -> const char* {  // strip column -> data column base
        const int64_t vcol = c0 - P.rmax + c;
        const int dcol = mirror32(static_cast<int>(vcol), static_cast<int>(P.samples));
        return static_cast<const char*>(P.cube) + static_cast<int64_t>(dcol) * L * P.elem_bytes;
    };
    auto shifted = [&](const char* cb, int64_t vrow, double (&y)[L]) -> int {
        load_row<L, STD, FUSE>(P, cb, row_bytes, static_cast<int>(vrow), y);
        const int nz = nonzero<L>(y);
#pragma unroll
        for (int i = 0; i < L; ++i) y[i] -= shift[i];
        return nz;
    };

    // STD (fp64 cube): the entering and leaving rows of every box for the update of
    // row rr are copied by one thread with TMA bulk copies (cp.async.bulk, one per
    // row: the strip's clipped column range is contiguous in BIP) into a shared
    // stage while the CTA still solves row rr - 1, so the update reads shared
    // memory instead of waiting on L2/HBM. stage[(2k + dir) * ncol + col][L].
    auto issue_rows = [&](int64_t rr) {  // thread 0 only
        const uint32_t seg = static_cast<uint32_t>((st_hi - st_lo) * L * sizeof(double));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&s_bar, seg * 2 * NBOX);
#pragma unroll
        for (int k = 0; k < NBOX; ++k) {
            const int R = P.radius[k];
#pragma unroll
            for (int dir = 0; dir < 2; ++dir) {
                const int vrow = static_cast<int>(dir == 0 ? rr + R : rr - 1 - R);
                const int64_t drow = mirror32(vrow, static_cast<int>(P.lines)) - P.buf_row0;
                const double* src = static_cast<const double*>(P.cube) + (drow * P.samples + st_lo) * L;
                bulk_g2s(stage + static_cast<int64_t>(2 * k + dir) * ncol * L, src, seg, &s_bar);
            }
        }
    };
    uint32_t st_phase = 0;
    if constexpr (STD) {
        if (t == 0) {
            mbar_init(&s_bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            if (ra + 1 < rb) issue_rows(ra + 1);
        }
    }

    // initial vertical sums over rows [ra - R_k, ra + R_k]
    for (int c = t; c < ncol; c += NT) {
        const char* cb = colbase_of(c);
#pragma unroll
        for (int k = 0; k < NBOX; ++k) {
            double v[NC];
#pragma unroll
            for (int i = 0; i < NC; ++i) v[i] = 0.0;
            const int R = P.radius[k];
            int nzc = 0;
            for (int d = -R; d <= R; ++d) {
                double y[L];
                nzc += shifted(cb, ra + d, y);
                add_moments<L>(v, y, 1.0);
            }
            if constexpr (ZC) s_nz[k * ncol + c] = nzc;
            else if (k == 0 && nzc != 2 * R + 1) s_zero_seen = 1;
            double2* dst = vslot(k, c);
#pragma unroll
            for (int c2 = 0; c2 < NC2; ++c2)
                dst[c2] = make_double2(v[2 * c2], 2 * c2 + 1 < NC ? v[2 * c2 + 1] : 0.0);
        }
    }

    const int seg0 = t * K;  // first output strip column of this thread (relative to rmax)
    PT_START();
    const bool owner1 = K == 1 && seg0 < P.tw && c0 + seg0 < P.samples;
    const char* own_cb = colbase_of(P.rmax + seg0);
    // stage column of strip column c: every column a valid output's window reads mirrors
    // into [lo, hi); the clamp only guards the unused tail columns of a strip that runs past
    // the image. Row-invariant: the thread's first column's is kept across the row loop.
    auto scol_of = [&](int c) {
        return min(max(mirror32(static_cast<int>(c0 - P.rmax + c), static_cast<int>(P.samples)) -
                           static_cast<int>(st_lo),
                       0),
                   static_cast<int>(st_hi - st_lo) - 1);
    };
    const int scol_t = scol_of(t);
    // K = 1 on an fp64 cube: the centre spectrum of row r through a running pointer (the row is
    // inside the image and the buffer: no reflection)
    const double* own_p = reinterpret_cast<const double*>(own_cb + (ra - P.buf_row0) * row_bytes);
    for (int64_t r = ra; r < rb; ++r) {
        // K = 1: fetch the centre spectrum first; its latency hides behind the
        // vertical update, the barrier and the horizontal sums
        // (raw values: the shift and the zero test wait until the spectrum is used, so
        // the load is in flight across the update and the barrier)
        double yc1[L];
        if constexpr (STD && !FUSE && L % 2 == 0) {
            if (owner1) {
#pragma unroll
                for (int i = 0; i < L; i += 2) {
                    const double2 v = __ldg(reinterpret_cast<const double2*>(own_p + i));
                    yc1[i] = v.x;
                    yc1[i + 1] = v.y;
                }
            }
            own_p += P.samples * L;
        } else {
            if (owner1) load_row<L, STD, FUSE>(P, own_cb, row_bytes, static_cast<int>(r), yc1);
        }
        if (r > ra) {
            if constexpr (STD) {
                mbar_wait(&s_bar, st_phase);
                st_phase ^= 1;
            }
            for (int c = t; c < ncol; c += NT) {
                const char* cb = colbase_of(c);
                const int scol = c == t ? scol_t : scol_of(c);
#pragma unroll
                for (int k = 0; k < NBOX; ++k) {
                    const int R = P.radius[k];
                    double yin[L], yout[L], dm[NC];
                    int nz_in, nz_out;
                    if constexpr (STD) {
                        const double* si = stage + (static_cast<int64_t>(2 * k) * ncol + scol) * L;
                        const double* so = si + static_cast<int64_t>(ncol) * L;
#pragma unroll
                        for (int i = 0; i < L; i += 2) {
                            const double2 a = *reinterpret_cast<const double2*>(si + i);
                            const double2 b = *reinterpret_cast<const double2*>(so + i);
                            yin[i] = a.x;
                            yin[i + 1] = a.y;
                            yout[i] = b.x;
                            yout[i + 1] = b.y;
                        }
                        nz_in = nonzero<L>(yin);
                        nz_out = nonzero<L>(yout);
#pragma unroll
                        for (int i = 0; i < L; ++i) {
                            yin[i] -= shift[i];
                            yout[i] -= shift[i];
                        }
                    } else {
                        nz_in = shifted(cb, r + R, yin);
                        nz_out = shifted(cb, r - 1 - R, yout);
                    }
                    // fast pass: every spectrum of any window enters box 0 (the widest, in
                    // the standard layout) or sits in its initial window, so checking box 0's
                    // entering rows finds every zero spectrum
                    if constexpr (ZC) s_nz[k * ncol + c] += nz_in - nz_out;
                    else if (k == 0 && !nz_in) s_zero_seen = 1;
                    // m(yin) - m(yout), rounded as add_moments(+yin) then add_moments(-yout) onto 0
                    {
                        int cc = L;
#pragma unroll
                        for (int i = 0; i < L; ++i) dm[i] = yin[i] - yout[i];
#pragma unroll
                        for (int i = 0; i < L; ++i)
#pragma unroll
                            for (int j = i; j < L; ++j) dm[cc++] = fma(-yout[i], yout[j], __dmul_rn(yin[i], yin[j]));
                    }
                    double2* dst = vslot(k, c);
#pragma unroll
                    for (int c2 = 0; c2 < NC2; ++c2) {
                        double2 v = dst[c2];
                        v.x += dm[2 * c2];
                        if (2 * c2 + 1 < NC) v.y += dm[2 * c2 + 1];
                        dst[c2] = v;
                    }
                }
            }
        }
        PT_MARK(0);  // vertical update
        __syncthreads();
        if constexpr (STD) {  // the stage is consumed: fetch the next row's update rows
            if (t == 0 && r > ra && r + 1 < rb) issue_rows(r + 1);  // ra + 1: issued at start
        }
        PT_MARK(1);  // barrier A
        // K = 1: every lane forms its horizontal sums (the lane pairs exchange halves
        // with shuffles), then lanes outside the image skip the solves
        if (K == 1 || (seg0 < P.tw && c0 + seg0 < P.samples)) {
            double S[NBOX][NC];
            int cnt[NBOX];
            // horizontal window of the first column of the segment
#pragma unroll
            for (int k = 0; k < NBOX; ++k) {
#pragma unroll
                for (int i = 0; i < NC; ++i) S[k][i] = 0.0;
                const int R = P.radius[k];
                int ck = 0;
                if constexpr (ZC) {
                    for (int d = -R; d <= R; ++d) ck += s_nz[k * ncol + P.rmax + seg0 + d];
                }
                if (K == 1 && R >= kPairRadius) {
                    // Lane pair (even column c, odd column c + 1): the windows share the
                    // 2R columns [c + 1 - R, c + R]. The even lane sums [c + 1 - R, c]
                    // (walking down from c), the odd lane [c + 1, c + R] (walking up),
                    // they swap halves, and each adds its own edge column (c - R or
                    // c + 1 + R): R + 1 column reads per box instead of 2R + 1, and the
                    // opposite walking directions keep the LDS.128 conflict-free. The
                    // core is (lower half + upper half) in both lanes, so each pixel's
                    // summation order depends only on its global column parity.
                    const bool odd = (t & 1) != 0;
                    const int own = P.rmax + seg0;
                    double h[NC];
                    {  // d = 0 (R >= kPairRadius >= 1): the lane's own column starts the sum
                        const double2* src = vslot(k, own);
#pragma unroll
                        for (int c2 = 0; c2 < NC2; ++c2) {
                            const double2 v = src[c2];
                            h[2 * c2] = v.x;
                            if (2 * c2 + 1 < NC) h[2 * c2 + 1] = v.y;
                        }
                    }
                    for (int d = 1; d < R; ++d) {
                        const double2* src = vslot(k, odd ? own + d : own - d);
#pragma unroll
                        for (int c2 = 0; c2 < NC2; ++c2) {
                            const double2 v = src[c2];
                            h[2 * c2] += v.x;
                            if (2 * c2 + 1 < NC) h[2 * c2 + 1] += v.y;
                        }
                    }
                    const double2* e = vslot(k, odd ? own + R : own - R);
#pragma unroll
                    for (int c2 = 0; c2 < NC2; ++c2) {
                        const double2 v = e[c2];
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int i = 2 * c2 + hh;
                            if (i >= NC) break;
                            const double other = __shfl_xor_sync(0xffffffffu, h[i], 1);
                            const double core = odd ? other + h[i] : h[i] + other;
                            S[k][i] = core + (hh == 0 ? v.x : v.y);
                        }
                    }
                } else {
                    for (int d = -R; d <= R; ++d) {
                        const double2* src = vslot(k, P.rmax + seg0 + d);
#pragma unroll
                        for (int c2 = 0; c2 < NC2; ++c2) {
                            const double2 v = src[c2];
                            S[k][2 * c2] += v.x;
                            if (2 * c2 + 1 < NC) S[k][2 * c2 + 1] += v.y;
                        }
                    }
                }
                cnt[k] = ck;
            }
            // K = 1: the window sums are in registers and nothing below reads the shared
            // vertical sums, so the row's second barrier sits here, where the warps arrive
            // together, and a warp that finishes its solves early goes straight on to the next
            // row's update (its own columns) while the others still solve.
            if constexpr (K == 1 && !FUSE) __syncthreads();
#pragma unroll 1
            for (int j = 0; j < K; ++j) {
                const int sc = seg0 + j;
                const int64_t col = c0 + sc;
                if (sc >= P.tw || col >= P.samples) break;
                if (j > 0) {
#pragma unroll
                    for (int k = 0; k < NBOX; ++k) {
                        const int R = P.radius[k];
                        if constexpr (ZC)
                            cnt[k] += s_nz[k * ncol + P.rmax + sc + R] - s_nz[k * ncol + P.rmax + sc - 1 - R];
                        const double2* in = vslot(k, P.rmax + sc + R);
                        const double2* out = vslot(k, P.rmax + sc - 1 - R);
#pragma unroll
                        for (int c2 = 0; c2 < NC2; ++c2) {
                            const double2 a = in[c2], b = out[c2];
                            S[k][2 * c2] += a.x - b.x;
                            if (2 * c2 + 1 < NC) S[k][2 * c2 + 1] += a.y - b.y;
                        }
                    }
                }
                double yc[L];
                int nzc;
                if (K == 1) {
#pragma unroll
                    for (int i = 0; i < L; ++i) yc[i] = yc1[i];
                    nzc = nonzero<L>(yc);
#pragma unroll
                    for (int i = 0; i < L; ++i) yc[i] -= shift[i];
                } else {
                    nzc = shifted(colbase_of(P.rmax + sc), r, yc);
                }
                PT_MARK(2);  // horizontal + centre load
                solve_pixel<L, NBOX, STD, ZC, TRIO>(P, s_req, S, cnt, nzc, yc, r, col);
                PT_MARK(3);  // solves
            }
        }
        if constexpr (FUSE) {  // the entering row of the TMA copies issued at step r + 1
            if (r + 2 < rb)
                fused_dwt_row(P, wsm, mirror32(static_cast<int>(r + 2 + P.radius[0]), static_cast<int>(P.lines)),
                              c0, ncol);
        }
        if constexpr (K > 1 || FUSE) __syncthreads();
        PT_MARK(4);  // barrier B
    }
    if constexpr (K == 1 && !FUSE) __syncthreads();  // s_zero_seen of the last row's solves
    if constexpr (!ZC) {
        if (t == 0 && s_zero_seen && P.zflag)
            P.zflag[static_cast<int64_t>(by) * nbx + bx] = 1;
    }
    if constexpr (STD) {  // the stage barrier is re-initialised by the next tile of a persistent CTA
        __syncthreads();
        if (t == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&s_bar)) : "memory");
    }
    PT_FLUSH();
}

template <int L, int NBOX, int K, bool STD, bool ZC, bool FUSE = false, bool TRIO = false>
__global__ void __launch_bounds__(HSAD_DET_NT, (L <= 5 ? HSAD_DET_MINB : 1)) detect_kernel(const DetectParams P) {
    detect_tile<L, NBOX, K, STD, ZC, FUSE, TRIO>(P, blockIdx.x, blockIdx.y, gridDim.x);
}

// The counting pass after a fast pass recomputes only the tiles the fast pass flagged
// (usually none): one wave of persistent CTAs walks the flag array instead of a full
// grid of CTAs that exit at once (measured ~33 us per launch for the full grid).
template <int L, int NBOX, int K, bool STD>
__global__ void __launch_bounds__(HSAD_DET_NT, (L <= 5 ? HSAD_DET_MINB : 1))
    detect_kernel_flagged(const DetectParams P, int nbx, int nby) {
    const int64_t n = static_cast<int64_t>(nbx) * nby;
    for (int64_t vb = blockIdx.x; vb < n; vb += gridDim.x) {
        if (!P.zflag[vb]) continue;  // uniform per CTA
        detect_tile<L, NBOX, K, STD, true>(P, static_cast<int>(vb % nbx), static_cast<int>(vb / nbx), nbx);
        __syncthreads();
    }
}


template <int L, int NB>
cudaError_t launch_lk(const DetectParams& P, dim3 grid, int nt, int kcols, cudaStream_t s) {
    const int ncol = P.tw + 2 * P.rmax;
    auto go = [&](auto kern, int K, bool staged, bool two_pass, bool fused = false) -> cudaError_t {
        const size_t smem = (static_cast<size_t>(NB) * (ncol * Dim<L>::S2 + (K > 1 ? ncol / K + 1 : 0)) +
                             nz_pairs(NB, ncol)) * sizeof(double2) +
                            (staged ? stage_bytes(NB, ncol, L) : 0) + (fused ? kFuseMapBytes : 0);
        if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        if (two_pass) {
            kern<<<grid, nt, smem, s>>>(P);
        } else {
            DetectParams Q = P;
            Q.zflag = nullptr;  // single counting pass over every CTA
            kern<<<grid, nt, smem, s>>>(Q);
        }
        return cudaGetLastError();
    };
    // the counting pass over the flagged tiles: one wave of persistent CTAs
    auto go_flagged = [&](auto kern, int K) -> cudaError_t {
        const size_t smem = (static_cast<size_t>(NB) * (ncol * Dim<L>::S2 + (K > 1 ? ncol / K + 1 : 0)) +
                             nz_pairs(NB, ncol)) * sizeof(double2) + stage_bytes(NB, ncol, L);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t n = static_cast<int64_t>(grid.x) * grid.y;
        const int ctas = static_cast<int>(n < 4LL * sms ? n : 4LL * sms);
        kern<<<ctas, nt, smem, s>>>(P, static_cast<int>(grid.x), static_cast<int>(grid.y));
        return cudaGetLastError();
    };
    if constexpr (L == 4) {  // multi-column segments only on the 4-band (DWT) hot path
        // standard request layout (box 0 outer/LRX, box 1 inner) on an fp64 cube: a
        // kernel without the general box-selection path and the fp32 load path
        // (smaller code: fewer instruction-cache misses, measured -5% on C5)
        if constexpr (NB <= 2) {
            if (P.staged) {  // fast pass, then the counting pass over CTAs that met zeros
                auto both = [&](auto fast, auto flagged, int K) -> cudaError_t {
                    cudaError_t e = go(fast, K, true, true);
                    return e != cudaSuccess ? e : go_flagged(flagged, K);
                };
                if constexpr (NB == 2) {
                    if (P.raw && kcols == 1) {  // fused DWT fast pass (the counting pass reads the rows it wrote)
                        cudaError_t e = go(detect_kernel<L, NB, 1, true, false, true>, 1, true, true, true);
                        return e != cudaSuccess ? e : go_flagged(detect_kernel_flagged<L, NB, 1, true>, 1);
                    }
                }
                if constexpr (NB == 2) {
                    if (P.trio) {  // the standard trio's own kernel (smaller code)
                        if (kcols == 4) return both(detect_kernel<L, NB, 4, true, false, false, true>, detect_kernel_flagged<L, NB, 4, true>, 4);
                        if (kcols == 2) return both(detect_kernel<L, NB, 2, true, false, false, true>, detect_kernel_flagged<L, NB, 2, true>, 2);
                        if (kcols == 1) return both(detect_kernel<L, NB, 1, true, false, false, true>, detect_kernel_flagged<L, NB, 1, true>, 1);
                    }
                }
                if (kcols == 4) return both(detect_kernel<L, NB, 4, true, false>, detect_kernel_flagged<L, NB, 4, true>, 4);
                if (kcols == 2) return both(detect_kernel<L, NB, 2, true, false>, detect_kernel_flagged<L, NB, 2, true>, 2);
                if (kcols == 1) return both(detect_kernel<L, NB, 1, true, false>, detect_kernel_flagged<L, NB, 1, true>, 1);
            }
        }
        if (kcols == 4) return go(detect_kernel<L, NB, 4, false, true>, 4, false, false);
        if (kcols == 2) return go(detect_kernel<L, NB, 2, false, true>, 2, false, false);
    }
    if (kcols == 1) return go(detect_kernel<L, NB, 1, false, true>, 1, false, false);
    return cudaErrorInvalidValue;
}

template <int L>
cudaError_t launch_l(const DetectParams& P, dim3 grid, int nt, int kcols, cudaStream_t s) {
    switch (P.nbox) {
#ifndef HSAD_FAST_BUILD  // A/B builds of the C5 sweep kernel only (scripts/build_variant.sh)
        case 1: return launch_lk<L, 1>(P, grid, nt, kcols, s);
#endif
        case 2: return launch_lk<L, 2>(P, grid, nt, kcols, s);
#ifndef HSAD_FAST_BUILD
        case 3: return launch_lk<L, 3>(P, grid, nt, kcols, s);
        case 4: return launch_lk<L, 4>(P, grid, nt, kcols, s);
#endif
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_bands(int bands, const DetectParams& P, dim3 grid, int nt, int kcols,
                         cudaStream_t s) {
    switch (bands) {
#ifndef HSAD_FAST_BUILD
        case 1: return launch_l<1>(P, grid, nt, kcols, s);
        case 2: return launch_l<2>(P, grid, nt, kcols, s);
        case 3: return launch_l<3>(P, grid, nt, kcols, s);
#endif
        case 4: return launch_l<4>(P, grid, nt, kcols, s);
#ifndef HSAD_FAST_BUILD
        case 5: return launch_l<5>(P, grid, nt, kcols, s);
        case 6: return launch_l<6>(P, grid, nt, kcols, s);
        case 7: return launch_l<7>(P, grid, nt, kcols, s);
        case 8: return launch_l<8>(P, grid, nt, kcols, s);
#endif
    }
    return cudaErrorInvalidValue;
}

// The staged (standard-layout fp64) kernel runs as a fast pass plus a counting pass
// that recomputes only the CTAs which met an all-zero spectrum; their per-CTA flags
// live in a stream-ordered scratch allocation.
cudaError_t launch_detect(int bands, const DetectParams& P0, dim3 grid, int nt, int kcols,
                          cudaStream_t s) {
    DetectParams P = P0;
    P.zflag = nullptr;
    unsigned char* flags = nullptr;
    if (P.staged) {
        const size_t n = static_cast<size_t>(grid.x) * grid.y;
        cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&flags), n, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(flags, 0, n, s);
        if (e != cudaSuccess) return e;
        P.zflag = flags;
    }
    const cudaError_t e = launch_bands(bands, P, grid, nt, kcols, s);
    if (flags) scratch_free(flags, s);
    return e;
}

const char* algo_name(int a) {
    return a == HSAD_LRX ? "local_rx" : a == HSAD_DWRX ? "dwrx" : a == HSAD_DWEST ? "dwest" : "?";
}

struct Plan {
    DetectParams P{};
    int nt = HSAD_DET_NT;
    int kcols = 1;
    dim3 grid;
};

// Validate requests (detect.cpp:119-125, 233-234) and resolve the distinct box radii.
hsad_status plan_requests(const hsad_detect_request* reqs, int n, Plan& plan) {
    if (n < 1 || n > kMaxRequests)
        return set_error(HSAD_E_INVALID_VALUE,
                         "between 1 and " + std::to_string(kMaxRequests) + " requests per call");
    if (!reqs) return set_error(HSAD_E_INVALID_VALUE, "null request list");
    DetectParams& P = plan.P;
    P.nbox = 0;
    auto box_of = [&](int size) -> int {
        const int r = size / 2;
        for (int k = 0; k < P.nbox; ++k)
            if (P.radius[k] == r) return k;
        if (P.nbox == kMaxBoxes) return -1;
        P.radius[P.nbox] = r;
        return P.nbox++;
    };
    P.nreq = n;
    for (int q = 0; q < n; ++q) {
        const hsad_detect_request& r = reqs[q];
        ReqDev& d = P.req[q];
        hsad_status st = window_validate(r.window);
        if (st != HSAD_OK) return st;
        if (r.algorithm == HSAD_LRX) {
            if (r.window.mode != HSAD_WINDOW_SINGLE)
                return set_error(HSAD_E_CONFIG_MISMATCH, "local_rx requires a single window");
            const int w = r.window.single_size;
            const int g = r.guard <= 0 ? 1 : r.guard;
            if (g % 2 == 0 || g >= w)
                return set_error(HSAD_E_INVALID_VALUE,
                                 "guard window must be odd, >= 1 and < window, got " +
                                     std::to_string(g));
            if (!(r.ridge >= 0.0))
                return set_error(HSAD_E_INVALID_VALUE, "ridge fraction must be nonnegative");
            d.box_a = box_of(w);
            d.box_b = g == 1 ? -1 : box_of(g);
            d.n_a = static_cast<double>(w) * w - static_cast<double>(g) * g;
            d.n_b = 0.0;
        } else if (r.algorithm == HSAD_DWRX || r.algorithm == HSAD_DWEST) {
            if (r.window.mode != HSAD_WINDOW_DUAL)
                return set_error(HSAD_E_CONFIG_MISMATCH,
                                 std::string(algo_name(r.algorithm)) + " requires a dual window");
            if (r.algorithm == HSAD_DWEST && !(r.eigen_fraction > 0.0 && r.eigen_fraction <= 1.0))
                return set_error(HSAD_E_INVALID_VALUE, "eigen fraction must be in (0, 1]");
            if (r.algorithm == HSAD_DWRX && !(r.ridge >= 0.0))
                return set_error(HSAD_E_INVALID_VALUE, "ridge fraction must be nonnegative");
            d.box_a = box_of(r.window.outer_size);
            d.box_b = box_of(r.window.inner_size);
            d.n_a = static_cast<double>(r.window.inner_size) * r.window.inner_size;
            d.n_b = static_cast<double>(r.window.outer_size) * r.window.outer_size - d.n_a;
        } else {
            return set_error(HSAD_E_INVALID_VALUE, "unknown algorithm");
        }
        if (d.box_a < 0 || (r.algorithm != HSAD_LRX && d.box_b < 0) ||
            (r.algorithm == HSAD_LRX && r.guard > 1 && d.box_b < 0))
            return set_error(HSAD_E_UNSUPPORTED,
                             "more than " + std::to_string(kMaxBoxes) + " distinct window sizes");
        d.algo = r.algorithm;
        d.ridge = r.ridge;
        d.frac = r.eigen_fraction;
        d.scores = r.d_scores;
        d.score_bytes = r.score_bytes;
        d.eigcount = r.algorithm == HSAD_DWEST ? r.d_eigcount : nullptr;
        if (r.score_bytes != 4 && r.score_bytes != 8)
            return set_error(HSAD_E_INVALID_VALUE, "score_bytes must be 4 or 8");
    }
    // standard layout: every LRX uses box 0 with the centre excluded and every dual
    // request uses (outer, inner) = (box 0, box 1) -> select-free solves in the kernel
    P.std_layout = 1;
    P.has_dual = 0;
    P.n_in = P.n_ann = 0.0;
    for (int q = 0; q < n; ++q) {
        const ReqDev& d = P.req[q];
        if (d.algo == HSAD_LRX) {
            if (d.box_a != 0 || d.box_b != -1) P.std_layout = 0;
        } else {
            if (d.box_a != 0 || d.box_b != 1) P.std_layout = 0;
            P.has_dual = 1;
            P.n_in = d.n_a;
            P.n_ann = d.n_b;
        }
    }
    // the standard trio: one LRX, one DWRX, one DWEST (solve_trio)
    P.trio = 0;
    if (P.std_layout && P.nbox == 2 && n == 3) {
        int seen[3] = {-1, -1, -1};
        for (int q = 0; q < n; ++q) seen[P.req[q].algo] = q;
        if (seen[0] >= 0 && seen[1] >= 0 && seen[2] >= 0 && !getenv("HSAD_NO_TRIO")) {
            P.trio = 1;
            for (int a = 0; a < 3; ++a) {
                P.trio_q[a] = seen[a];
                P.treq[a] = P.req[seen[a]];
            }
        }
    }
    P.rmax = 0;
    for (int k = 0; k < P.nbox; ++k) P.rmax = P.radius[k] > P.rmax ? P.radius[k] : P.rmax;
    if (P.rmax > kMaxRadius)
        return set_error(HSAD_E_UNSUPPORTED, "window edge above " +
                                                 std::to_string(2 * kMaxRadius + 1) +
                                                 " is outside this build's kernel limits");
    return HSAD_OK;
}

}  // namespace

// Output columns per thread (before the shared-memory fit check): wide images
// amortise the horizontal window over more columns.
int kcols_for(int64_t samples) { return samples >= 2048 ? 4 : samples >= 512 ? 2 : 1; }

extern "C" hsad_status hsad_reduce(const void* d_cube, int32_t elem_bytes, int64_t lines,
                                   int64_t samples, int32_t bands, int32_t order,
                                   int32_t target_bands, void* d_out, int32_t out_bytes,
                                   void* stream);

int64_t row_quantum(int64_t lines, int64_t samples) {
    // chunk height: large enough to amortise the 2R+1-row warm-up, small enough
    // that the grid fills the GPU twice (148 SMs); depends on the image only
    const int sms = 148;
    const int64_t tw = HSAD_DET_NT * kcols_for(samples);
    const int64_t strips = (samples + tw - 1) / tw;
    // 32 measured best on C5 (24..128 sweep: within 1% of 24, 3.6% faster than 64)
#ifndef HSAD_ROW_QUANTUM
#define HSAD_ROW_QUANTUM 32
#endif
    int64_t q = HSAD_ROW_QUANTUM;
    while (q > 2 && strips * ((lines + q - 1) / q) < 2 * sms) q /= 2;
    return q;
}

namespace {

// hsad_reduce_detect's reduction, folded into the first detector launch (fused_dwt_row)
// when HSAD_FUSE=1 and the launch qualifies: the fp32 cube, its bands and the composed
// map. Opt-in because it measured 7x slower than hsad_reduce + the launch (C5 sweep,
// first window pair: 37.8 ms vs 5.16 ms): without shared memory left for a TMA ring of
// the 120 KB raw row each CTA reduces per step, the full-band loads sit in the
// latency-bound detector loop (f1).
struct FuseArgs {
    const float* raw;
    int bands, order, target;
    const double* map;
    bool fused = false;    // the first launch computed the reduction
    bool reduced = false;  // hsad_reduce ran before it
    cudaEvent_t after_reduce = nullptr;  // recorded on the stream right after hsad_reduce (group fork)
    bool after_reduce_recorded = false;
};

// Side streams for the request groups of one asynchronous call: the groups read the same
// cube and write their own maps, so groups 1.. run on side streams forked from the caller's
// stream and joined back into it (the tail of one launch fills with the head of the next:
// C5 sweep detectors 7.14 -> 6.87 ms). Per host thread and device, created on first use.
struct GroupFork {
    static constexpr int kSide = 3;
    int device = -1;
    cudaStream_t side[kSide] = {};
    cudaEvent_t ready = nullptr, done[kSide] = {};
    bool ok = false;
    GroupFork() = default;
    GroupFork(const GroupFork&) = delete;
    GroupFork& operator=(const GroupFork&) = delete;
    ~GroupFork() {  // at thread exit (hsad_pipeline_sharded's workers); errors at process teardown are moot
        for (int i = 0; i < kSide; ++i) {
            if (side[i]) cudaStreamDestroy(side[i]);
            if (done[i]) cudaEventDestroy(done[i]);
        }
        if (ready) cudaEventDestroy(ready);
    }
};
GroupFork* group_fork() {
    thread_local std::vector<std::unique_ptr<GroupFork>> ctx;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    for (auto& gp : ctx)
        if (gp->device == dev) return gp->ok ? gp.get() : nullptr;
    ctx.push_back(std::make_unique<GroupFork>());
    GroupFork& g = *ctx.back();
    g.device = dev;
    bool ok = cudaEventCreateWithFlags(&g.ready, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < GroupFork::kSide && ok; ++i)
        ok = cudaStreamCreateWithFlags(&g.side[i], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&g.done[i], cudaEventDisableTiming) == cudaSuccess;
    g.ok = ok;
    return ok ? &g : nullptr;
}

// One fused launch: <= kMaxRequests requests over <= kMaxBoxes window sizes.
hsad_status detect_group_impl(const void* d_cube, int32_t elem_bytes, int64_t lines,
                              int64_t samples, int32_t bands, int64_t buf_row0, int64_t buf_rows,
                              int64_t row_begin, int64_t row_end,
                              const hsad_detect_request* requests, int32_t n_requests,
                              int req_base, uint64_t* d_status, hsad_pixel_error* err,
                              cudaStream_t s, FuseArgs* fuse = nullptr) {
    if (err) {
        err->code = HSAD_OK;
        err->row = err->col = -1;
    }
    // the reduction when it is not fused into this launch (every early return below)
    auto reduce_first = [&]() -> hsad_status {
        if (!fuse) return HSAD_OK;
        FuseArgs* f = fuse;
        fuse = nullptr;
        f->reduced = true;
        const hsad_status rs = hsad_reduce(f->raw, 4, buf_rows, samples, f->bands, f->order, f->target,
                                           const_cast<void*>(d_cube), 8, s);
        if (rs == HSAD_OK && f->after_reduce && cudaEventRecord(f->after_reduce, s) == cudaSuccess)
            f->after_reduce_recorded = true;  // later groups may start here, next to this one
        return rs;
    };
    Plan plan;
    hsad_status st = plan_requests(requests, n_requests, plan);
    if (st != HSAD_OK) return st;
    if (elem_bytes != 4 && elem_bytes != 8)
        return set_error(HSAD_E_INVALID_VALUE, "elem_bytes must be 4 or 8");
    // bands > 8: the full-band path (K5/K6, fullband.cu) for LRX / DWRX
    const bool fullband = bands > kMaxDetectBands;
    if (bands < 1) return set_error(HSAD_E_INVALID_VALUE, "cube has no bands");
    if (lines < 0 || samples < 0 || row_begin < 0 || row_end > lines || row_begin > row_end)
        return set_error(HSAD_E_INVALID_VALUE, "row range outside the image");
    if (row_begin == row_end || samples == 0) return reduce_first();
    // rows the windows touch must be resident in the buffer
    int64_t need0 = 0, need_rows = 0;
    st = hsad_strip_rows(lines, row_begin, row_end, requests, n_requests, &need0, &need_rows);
    if (st != HSAD_OK) return st;
    if (need0 < buf_row0 || need0 + need_rows > buf_row0 + buf_rows)
        return set_error(HSAD_E_OUT_OF_BOUNDS,
                         "buffer rows [" + std::to_string(buf_row0) + ", " +
                             std::to_string(buf_row0 + buf_rows) + ") do not cover the window rows [" +
                             std::to_string(need0) + ", " + std::to_string(need0 + need_rows) + ")");
    for (int q = 0; q < n_requests; ++q)
        if (!requests[q].d_scores) return set_error(HSAD_E_INVALID_VALUE, "null score buffer");
    // DWEST with a 1-pixel inner box: covariance(inner) throws TooFewSamples at the
    // first pixel (stats.cpp:15-17 via detect.cpp:252-253)
    for (int q = 0; q < n_requests; ++q)
        if (requests[q].algorithm == HSAD_DWEST && requests[q].window.inner_size == 1) {
            if (err) {
                err->code = HSAD_E_TOO_FEW_SAMPLES;
                err->row = row_begin;
                err->col = 0;
            }
            // detect.cpp:127-130 rethrows with the inner "<Name>: " kept
            const hsad_status rs = reduce_first();
            if (rs != HSAD_OK) return rs;
            return set_error(HSAD_E_TOO_FEW_SAMPLES,
                             "TooFewSamples: covariance needs at least 2 samples, got 1 at pixel (" +
                                 std::to_string(row_begin) + ", 0)");
        }

    DetectParams& P = plan.P;
    P.cube = d_cube;
    P.elem_bytes = elem_bytes;
    P.lines = lines;
    P.samples = samples;
    P.buf_row0 = buf_row0;
    P.buf_rows = buf_rows;
    P.row_begin = row_begin;
    P.row_end = row_end;
    P.chunk = row_quantum(lines, samples);
    // 128 threads x K output columns; shrink K until the per-box vertical sums
    // (strip + halo columns) fit comfortably in shared memory
    plan.nt = HSAD_DET_NT;
    int kc = bands == 4 ? kcols_for(samples) : 1;
    auto smem_for = [&](int k) {
        const int64_t ncol = static_cast<int64_t>(HSAD_DET_NT) * k + 2 * P.rmax;
        const int s2 = ((bands + bands * (bands + 1) / 2 + 1) / 2) | 1;
        return (static_cast<int64_t>(P.nbox) * (ncol * s2 + (k > 1 ? ncol / k + 1 : 0)) +
                nz_pairs(P.nbox, static_cast<int>(ncol))) * 16;
    };
    // <= 56 KB keeps 4 CTAs per SM (228 KB shared memory); K shrinks to fit
#ifndef HSAD_DET_SMEM_KB
#define HSAD_DET_SMEM_KB 56
#endif
    const int64_t smem_cap = getenv("HSAD_SMEM_CAP_KB") ? atoi(getenv("HSAD_SMEM_CAP_KB")) * 1024
                                                        : HSAD_DET_SMEM_KB * 1024;
    while (kc > 1 && smem_for(kc) > smem_cap) kc /= 2;
    if (!fullband && smem_for(kc) > 227 * 1024)
        return set_error(HSAD_E_UNSUPPORTED,
                         "window statistics for " + std::to_string(P.nbox) + " window sizes up to " +
                             std::to_string(2 * P.rmax + 1) + " at " + std::to_string(bands) +
                             " bands exceed shared memory; split the requests");
    if (fullband) kc = 1;
    plan.kcols = kc;
    P.tw = HSAD_DET_NT * kc;
    // STD kernel (standard layout, fp64 4-band cube) with the TMA row stage, if the
    // stage fits next to the window sums under the 4-CTA/SM budget
    P.staged = P.std_layout && elem_bytes == 8 && bands == 4 && P.nbox <= 2 &&
               smem_for(kc) + static_cast<int64_t>(stage_bytes(P.nbox, P.tw + 2 * P.rmax, bands)) <=
                   smem_cap &&
               !getenv("HSAD_NO_STAGE");
    P.req_base = req_base;
    P.raw = nullptr;
    P.raw_bands = 0;
    P.wmap = nullptr;
    if (fuse) {
        const int64_t ncol = P.tw + 2 * P.rmax;
        const bool fits = smem_for(kc) + static_cast<int64_t>(stage_bytes(P.nbox, ncol, bands)) +
                              kFuseMapBytes <= smem_cap;
        // the fused launch writes exactly the rows its windows read: it must be the whole buffer
        if (P.staged && kc == 1 && P.nbox == 2 && bands == 4 && fuse->bands <= 256 && fits &&
            need0 == buf_row0 && need_rows == buf_rows && !fullband && getenv("HSAD_FUSE")) {
            P.raw = fuse->raw;
            P.raw_bands = fuse->bands;
            P.wmap = fuse->map;
            fuse->fused = true;
            fuse = nullptr;
        } else {
            st = reduce_first();
            if (st != HSAD_OK) return st;
        }
    }
    P.diag_lin = -1;
    P.diag_req = -1;
    P.diag_out = nullptr;
    const int64_t strips = (samples + P.tw - 1) / P.tw;
    const int64_t chunks = (row_end - row_begin + P.chunk - 1) / P.chunk;
    if (chunks > 65535) return set_error(HSAD_E_UNSUPPORTED, "image too tall for one launch");
    plan.grid = dim3(static_cast<unsigned>(strips), static_cast<unsigned>(chunks));

    const bool sync = d_status == nullptr;
    unsigned long long* status = reinterpret_cast<unsigned long long*>(d_status);
    ScratchGuard status_guard(s);  // frees the internal status word on every return path
    if (sync) {
        // the caller-owned d_status accumulates (atomicMin) across calls; the
        // internal one is reset here
        HSAD_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&status), 2 * sizeof(double), s));
        status_guard.p = status;
        HSAD_CUDA_TRY(cudaMemsetAsync(status, 0xff, sizeof(unsigned long long), s));
    }
    P.status = status;
    // diagnostic scratch per request: scores (8 B/px) + eigen-count (1 B/px), 16-byte aligned
    const size_t scratch_stride = (static_cast<size_t>(samples) * 9 + 15) / 16 * 16;
    // full-band launcher: one fullband_kernel launch per request over rows [rb, re)
    auto launch_fb = [&](int64_t rb, int64_t re, int64_t diag_lin, int diag_req, double* diag_out,
                         char* scratch) -> hsad_status {
        for (int q = 0; q < n_requests; ++q) {
            const hsad_detect_request& R = requests[q];
            FbParams F{};
            F.cube = d_cube;
            F.elem_bytes = elem_bytes;
            F.lines = lines;
            F.samples = samples;
            F.bands = bands;
            F.buf_row0 = buf_row0;
            F.row_begin = rb;
            F.row_end = re;
            F.algo = R.algorithm;
            F.outer = R.algorithm == HSAD_LRX ? R.window.single_size : R.window.outer_size;
            F.inner = R.algorithm == HSAD_LRX ? (R.guard <= 0 ? 1 : R.guard) : R.window.inner_size;
            F.ridge = R.ridge;
            F.frac = R.eigen_fraction;
            F.scores = scratch ? static_cast<void*>(scratch + scratch_stride * q)
                               : R.d_scores;
            F.eigcount = R.algorithm != HSAD_DWEST || !R.d_eigcount ? nullptr
                         : scratch ? reinterpret_cast<int8_t*>(scratch + scratch_stride * q +
                                                               static_cast<size_t>(samples) * 8)
                                   : R.d_eigcount;
            F.score_bytes = R.score_bytes;
            F.status = status;
            F.req = req_base + q;
            F.diag_lin = req_base + q == diag_req ? diag_lin : -1;
            F.diag_out = diag_out;
            hsad_status fst = R.algorithm == HSAD_DWEST ? fullband_dwest_launch(F, s) : fullband_launch(F, s);
            if (fst != HSAD_OK) return fst;
        }
        return HSAD_OK;
    };
    cudaError_t e = cudaSuccess;
    if (fullband) {
        hsad_status fst = launch_fb(row_begin, row_end, -1, -1, nullptr, nullptr);
        if (fst != HSAD_OK) return fst;
    } else {
        e = launch_detect(bands, P, plan.grid, plan.nt, plan.kcols, s);
        if (e != cudaSuccess) return cuda_fail(e, "hsad detect kernel launch");
    }
    if (!sync) return HSAD_OK;

    unsigned long long packed = 0;
    HSAD_CUDA_TRY(cudaMemcpyAsync(&packed, status, sizeof(packed), cudaMemcpyDeviceToHost, s));
    HSAD_CUDA_TRY(cudaStreamSynchronize(s));
    hsad_status result = HSAD_OK;
    if (packed != ~0ull) {
        const int code = failure_code(packed);
        const bool overflow = (packed & kCodeOverflow) != 0;
        const int64_t lin = failure_pixel(packed);
        const int fail_req = failure_request(packed);
        const int64_t row = lin / samples, col = lin % samples;
        std::string msg;
        if (overflow) {
            msg = "inverse overflowed";
        } else if (code == HSAD_E_UNSUPPORTED) {
            msg = "more than 64 eigenvectors pass the DWEST cutoff (full-band kernel limit)";
        } else {
            // re-run the failing row to recover that pixel's ridge for the message
            double delta = 0.0;
            double* d_diag = reinterpret_cast<double*>(status) + 1;
            DetectParams D = P;
            D.raw = nullptr;  // the reduced rows exist now
            D.row_begin = row;
            D.row_end = row + 1;
            D.diag_lin = lin;
            D.diag_req = fail_req;
            D.diag_out = d_diag;
            D.trio = 0;  // the per-request solves report the ridge (same arithmetic; the trio kernel carries no diagnostics)
            // the diagnostic pass writes into scratch rows, never over the results
            char* scratch = nullptr;
            e = scratch_alloc(reinterpret_cast<void**>(&scratch), scratch_stride * D.nreq, s);
            if (e != cudaSuccess) return cuda_fail(e, "hsad detect diagnostics");
            ScratchGuard scratch_guard(s, scratch);
            for (int q = 0; q < D.nreq; ++q) {
                D.req[q].scores = scratch + scratch_stride * q;
                if (D.req[q].eigcount)
                    D.req[q].eigcount = reinterpret_cast<int8_t*>(
                        scratch + scratch_stride * q + static_cast<size_t>(samples) * 8);
            }
            if (fullband) {
                if (launch_fb(row, row + 1, lin, fail_req, d_diag, scratch) != HSAD_OK) e = cudaErrorUnknown;
            } else {
                e = launch_detect(bands, D, dim3(plan.grid.x, 1), plan.nt, plan.kcols, s);
            }
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(&delta, d_diag, sizeof(double), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return cuda_fail(e, "hsad detect diagnostics");
            // -0.0 (ridge 0 times a rounding-negative trace) prints as the reference's 0
            msg = "covariance numerically singular (ridge " + std::to_string(delta + 0.0) + ")";
        }
        result = static_cast<hsad_status>(code);
        set_error(result, std::string(status_name(code)) + ": " + msg + " at pixel (" +
                              std::to_string(row) + ", " + std::to_string(col) + ")");
        if (err) {
            err->code = code;
            err->row = row;
            err->col = col;
        }
    }
    return result;
}

// box radii a request needs (detect.cpp window semantics; LRX guard > 1 adds a box)
int request_radii(const hsad_detect_request& r, int (&out)[2]) {
    if (r.window.mode == HSAD_WINDOW_SINGLE) {
        out[0] = r.window.single_size / 2;
        if (r.algorithm == HSAD_LRX && r.guard > 1) {
            out[1] = r.guard / 2;
            return 2;
        }
        return 1;
    }
    out[0] = r.window.outer_size / 2;
    out[1] = r.window.inner_size / 2;
    return 2;
}

}  // namespace

// Requests are split greedily, in order, into groups of consecutive requests with
// the same outer (LRX: single) window, <= kMaxRequests members and <= kMaxBoxes
// distinct window sizes; each group is one fused launch. The grouping (and so the
// launch shape) depends only on the request list, so results are deterministic. Synchronous calls report the first group (in request order) with a
// failing pixel, i.e. the first of the equivalent sequential hsad::detect calls.
namespace {
hsad_status detect_multi_fuse(const void* d_cube, int32_t elem_bytes, int64_t lines,
                              int64_t samples, int32_t bands, int64_t buf_row0, int64_t buf_rows,
                              int64_t row_begin, int64_t row_end,
                              const hsad_detect_request* requests, int32_t n_requests,
                              uint64_t* d_status, hsad_pixel_error* err, cudaStream_t s,
                              FuseArgs* fuse) {
    if (n_requests < 1 || n_requests > kMaxCallRequests || !requests)
        return set_error(HSAD_E_INVALID_VALUE, "between 1 and " + std::to_string(kMaxCallRequests) +
                                                   " requests per call");
    FuseArgs* const fuse_first = fuse;
    // asynchronous calls fork their groups (synchronous ones report the first failing group
    // in request order and stay sequential)
    GroupFork* fk = d_status && !getenv("HSAD_NO_FORK") ? group_fork() : nullptr;
    bool ready_set = false, used[GroupFork::kSide] = {false, false, false};
    if (fk) {
        if (fuse) fuse->after_reduce = fk->ready;  // groups 1.. wait for the reduced cube only
        else ready_set = cudaEventRecord(fk->ready, s) == cudaSuccess;
        if (!fuse && !ready_set) fk = nullptr;
    }
    hsad_status result = HSAD_OK;
    int g0 = 0, gi = 0;
    while (g0 < n_requests) {
        int radii[kMaxBoxes], nr = 0, g1 = g0;
        int outer0[2];
        request_radii(requests[g0], outer0);
        while (g1 < n_requests && g1 - g0 < kMaxRequests) {
            int rq[2];
            const int k = request_radii(requests[g1], rq);
            // a group shares one outer window (the fused kernel's standard layout)
            if (g1 > g0 && rq[0] != outer0[0]) break;
            int add = 0, merged[kMaxBoxes + 2];
            for (int i = 0; i < nr; ++i) merged[i] = radii[i];
            for (int j = 0; j < k; ++j) {
                bool seen = false;
                for (int i = 0; i < nr + add; ++i) seen = seen || merged[i] == rq[j];
                if (!seen) merged[nr + add++] = rq[j];
            }
            if (nr + add > kMaxBoxes && g1 > g0) break;
            if (nr + add > kMaxBoxes) {  // a single request never needs more than 2
                ++g1;
                break;
            }
            for (int i = nr; i < nr + add; ++i) radii[i] = merged[i];
            nr += add;
            ++g1;
        }
        cudaStream_t gs = s;
        if (fk && gi > 0) {
            if (!ready_set) {
                // group 0 carried the reduction: its event if hsad_reduce ran, else (fused in
                // the launch, or an early return) the end of group 0
                ready_set = (fuse_first && fuse_first->after_reduce_recorded) ||
                            cudaEventRecord(fk->ready, s) == cudaSuccess;
            }
            const int k = (gi - 1) % GroupFork::kSide;
            if (ready_set && cudaStreamWaitEvent(fk->side[k], fk->ready, 0) == cudaSuccess) {
                gs = fk->side[k];
                used[k] = true;
            }
        }
        result = detect_group_impl(d_cube, elem_bytes, lines, samples, bands, buf_row0,
                                   buf_rows, row_begin, row_end, requests + g0, g1 - g0, g0,
                                   d_status, err, gs, g0 == 0 ? fuse : nullptr);
        if (result != HSAD_OK) break;
        g0 = g1;
        ++gi;
    }
    // join: the caller's stream continues after every side stream
    if (fk)
        for (int k = 0; k < GroupFork::kSide; ++k)
            if (used[k] && (cudaEventRecord(fk->done[k], fk->side[k]) != cudaSuccess ||
                            cudaStreamWaitEvent(s, fk->done[k], 0) != cudaSuccess)) {
                cudaStreamSynchronize(fk->side[k]);
            }
    return result;
}
}  // namespace

hsad_status detect_multi_impl(const void* d_cube, int32_t elem_bytes, int64_t lines,
                              int64_t samples, int32_t bands, int64_t buf_row0, int64_t buf_rows,
                              int64_t row_begin, int64_t row_end,
                              const hsad_detect_request* requests, int32_t n_requests,
                              uint64_t* d_status, hsad_pixel_error* err, cudaStream_t s) {
    return detect_multi_fuse(d_cube, elem_bytes, lines, samples, bands, buf_row0, buf_rows, row_begin,
                             row_end, requests, n_requests, d_status, err, s, nullptr);
}

}  // namespace hsad_b200

using namespace hsad_b200;

namespace {
thread_local int32_t g_last_fused = 0;
}

#ifdef HSAD_PHASE_TIMERS
extern "C" void hsad_phase_cycles(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
}
#endif

extern "C" {

int64_t hsad_row_quantum(int64_t lines, int64_t samples) { return row_quantum(lines, samples); }

int32_t hsad_last_reduce_detect_fused(void) { return g_last_fused; }

hsad_status hsad_strip_rows(int64_t lines, int64_t row_begin, int64_t row_end,
                            const hsad_detect_request* requests, int32_t n_requests,
                            int64_t* buf_row0, int64_t* buf_rows) {
    int rmax = 0;
    for (int q = 0; q < n_requests; ++q) {
        const hsad_window& w = requests[q].window;
        const int size = w.mode == HSAD_WINDOW_SINGLE ? w.single_size : w.outer_size;
        rmax = size / 2 > rmax ? size / 2 : rmax;
    }
    if (row_begin >= row_end) {
        *buf_row0 = row_begin;
        *buf_rows = 0;
        return HSAD_OK;
    }
    int64_t lo = INT64_MAX, hi = -1;
    if (row_begin - rmax >= 0 && row_end + rmax <= lines) {
        lo = row_begin - rmax;
        hi = row_end + rmax - 1;
    } else {
        for (int64_t r = row_begin - rmax; r < row_end + rmax; ++r) {
            const int64_t m = mirror_index(r, lines);
            lo = m < lo ? m : lo;
            hi = m > hi ? m : hi;
        }
    }
    *buf_row0 = lo;
    *buf_rows = hi - lo + 1;
    return HSAD_OK;
}

hsad_status hsad_detect_multi(const void* d_cube, int32_t elem_bytes, int64_t lines,
                              int64_t samples, int32_t bands, int64_t buf_row0, int64_t buf_rows,
                              int64_t row_begin, int64_t row_end,
                              const hsad_detect_request* requests, int32_t n_requests,
                              uint64_t* d_status, hsad_pixel_error* err, void* stream) {
    return detect_multi_impl(d_cube, elem_bytes, lines, samples, bands, buf_row0, buf_rows,
                             row_begin, row_end, requests, n_requests, d_status, err,
                             static_cast<cudaStream_t>(stream));
}

hsad_status hsad_reduce_detect(const float* d_cube, int64_t lines, int64_t samples, int32_t bands,
                               int32_t order, int32_t target_bands, int64_t buf_row0,
                               int64_t buf_rows, int64_t row_begin, int64_t row_end,
                               double* d_reduced, const hsad_detect_request* requests,
                               int32_t n_requests, uint64_t* d_status, hsad_pixel_error* err,
                               void* stream) {
    if (err) {
        err->code = HSAD_OK;
        err->row = err->col = -1;
    }
    if (buf_row0 < 0 || buf_rows < 0 || buf_row0 + buf_rows > lines)
        return set_error(HSAD_E_INVALID_VALUE, "buffer rows outside the image");
    // reduce_cube errors first (the CLI runs `hsad reduce` before `hsad detect`)
    const double* d_map = nullptr;
    hsad_status st = device_wavelet_map(bands, order, target_bands, &d_map);
    if (st != HSAD_OK) return st;
    if (!d_cube || !d_reduced) return set_error(HSAD_E_INVALID_VALUE, "null buffer");
    // the reduction runs inside the first detector launch when it can (fused_dwt_row),
    // else hsad_reduce runs first; either way the reduced rows are bit-identical
    FuseArgs fa{d_cube, bands, order, target_bands, d_map};
    st = detect_multi_fuse(d_reduced, 8, lines, samples, target_bands, buf_row0, buf_rows, row_begin,
                           row_end, requests, n_requests, d_status, err, static_cast<cudaStream_t>(stream),
                           &fa);
    if (!fa.fused && !fa.reduced) {  // a request error before any launch: the reduction still runs
        const hsad_status rs = hsad_reduce(d_cube, 4, buf_rows, samples, bands, order, target_bands,
                                           d_reduced, 8, stream);
        if (st == HSAD_OK) st = rs;
    }
    g_last_fused = fa.fused ? 1 : 0;
    return st;
}

hsad_status hsad_detect(const void* d_cube, int32_t elem_bytes, int64_t lines, int64_t samples,
                        int32_t bands, const hsad_detect_request* request, hsad_pixel_error* err,
                        void* stream) {
    return detect_multi_impl(d_cube, elem_bytes, lines, samples, bands, 0, lines, 0, lines,
                             request, 1, nullptr, err, static_cast<cudaStream_t>(stream));
}

hsad_status hsad_dwest_pairs(const double* d_cdiff, const double* d_mdiff, int64_t n,
                             double eigen_fraction, double* d_scores, int8_t* d_counts,
                             int8_t* d_route, void* stream) {
    if (n < 0 || (n > 0 && (!d_cdiff || !d_mdiff || !d_scores)))
        return set_error(HSAD_E_INVALID_VALUE, "null buffer");
    if (!(eigen_fraction > 0.0 && eigen_fraction <= 1.0))
        return set_error(HSAD_E_INVALID_VALUE, "eigen fraction must be in (0, 1]");
    if (hsad_device_check() != HSAD_OK) return HSAD_E_CUDA;
    if (n == 0) return HSAD_OK;
    const int nt = 128;
    dwest_pairs_kernel<<<static_cast<unsigned>((n + nt - 1) / nt), nt, 0, static_cast<cudaStream_t>(stream)>>>(
        d_cdiff, d_mdiff, n, eigen_fraction, d_scores, d_counts, d_route);
    const cudaError_t ce = cudaGetLastError();
    return ce == cudaSuccess ? HSAD_OK : set_error(HSAD_E_CUDA, cudaGetErrorString(ce));
}

}  // extern "C"
