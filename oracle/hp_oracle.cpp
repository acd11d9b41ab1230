// TEST INFRASTRUCTURE ONLY — a higher-precision third opinion for the full-band
// (L ~ 189) detectors, used where the fp64 kernel and the fp64 oracle disagree.
//
// Same semantics as hsad_oracle.cpp (proj/core/src/detect.cpp:159-228 and
// proj/core/src/stats.cpp:7-62): the reference's window gathers (detect.cpp:83-117,
// mirror_index detect.cpp:71-76), mean, two-pass centred covariance with divisor N,
// ridge delta = ridge * tr(C) / L, and the quadratic form d^T (C + delta I)^-1 d —
// but every operation in x87 extended precision (long double: 64-bit mantissa,
// eps 5.4e-20, i.e. 2048x finer than fp64). C + delta I is symmetric positive
// definite wherever the reference does not raise SingularAfterRidge, so an
// unpivoted LDL^T plus two triangular solves gives the form without an explicit
// inverse; at kappa ~ 1e7 its own error is ~1e-12 relative, three orders below the
// fp64 solvers' ~kappa * 1.1e-16 disagreement, so it decides which of the two is
// the outlier.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

using Real = long double;

struct CubeView {
    const void* data;
    int elem;
    long lines, samples;
    int bands;
    Real at(long r, long c, int b) const {
        const std::size_t i = (static_cast<std::size_t>(r) * samples + c) * bands + b;
        return elem == 4 ? static_cast<Real>(static_cast<const float*>(data)[i])
                         : static_cast<Real>(static_cast<const double*>(data)[i]);
    }
};

int mirror(int i, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    i = std::abs(i) % period;
    return i < n ? i : period - i;
}

// samples as rows of `bands` values, in the reference's row-major window scan
void gather(const CubeView& c, long row, long col, int size, int exclude, std::vector<Real>& out,
            int& count) {
    const int half = size / 2, eh = exclude / 2;
    count = 0;
    out.clear();
    for (int dr = -half; dr <= half; ++dr) {
        const int rr = mirror(static_cast<int>(row) + dr, static_cast<int>(c.lines));
        for (int dc = -half; dc <= half; ++dc) {
            if (exclude > 0 && std::abs(dr) <= eh && std::abs(dc) <= eh) continue;
            const int cc = mirror(static_cast<int>(col) + dc, static_cast<int>(c.samples));
            for (int b = 0; b < c.bands; ++b) out.push_back(c.at(rr, cc, b));
            ++count;
        }
    }
}

void mean_cov(const std::vector<Real>& x, int n, int L, std::vector<Real>& mu, std::vector<Real>& cov) {
    mu.assign(L, 0.0L);
    for (int j = 0; j < n; ++j)
        for (int b = 0; b < L; ++b) mu[b] += x[static_cast<std::size_t>(j) * L + b];
    for (auto& m : mu) m /= static_cast<Real>(n);
    cov.assign(static_cast<std::size_t>(L) * L, 0.0L);
    std::vector<Real> d(L);
    for (int j = 0; j < n; ++j) {
        for (int b = 0; b < L; ++b) d[b] = x[static_cast<std::size_t>(j) * L + b] - mu[b];
        for (int a = 0; a < L; ++a)
            for (int b = 0; b <= a; ++b) cov[static_cast<std::size_t>(a) * L + b] += d[a] * d[b];
    }
    for (int a = 0; a < L; ++a)
        for (int b = 0; b <= a; ++b) {
            const Real v = cov[static_cast<std::size_t>(a) * L + b] / static_cast<Real>(n);
            cov[static_cast<std::size_t>(a) * L + b] = v;
            cov[static_cast<std::size_t>(b) * L + a] = v;
        }
}

// d^T (C + delta I)^-1 d by LDL^T (lower triangle of the symmetric matrix);
// returns false when a pivot is not positive. dmin / dmax: pivot range.
bool quad_form(std::vector<Real> a, const std::vector<Real>& d, int L, Real ridge, Real& out,
               Real& dmin, Real& dmax) {
    Real tr = 0.0L;
    for (int i = 0; i < L; ++i) tr += a[static_cast<std::size_t>(i) * L + i];
    const Real delta = ridge * tr / static_cast<Real>(L);
    for (int i = 0; i < L; ++i) a[static_cast<std::size_t>(i) * L + i] += delta;
    std::vector<Real> D(L);
    dmin = INFINITY;
    dmax = 0.0L;
    for (int j = 0; j < L; ++j) {
        Real djj = a[static_cast<std::size_t>(j) * L + j];
        for (int k = 0; k < j; ++k) {
            const Real ljk = a[static_cast<std::size_t>(j) * L + k];
            djj -= ljk * ljk * D[k];
        }
        if (!(djj > 0.0L)) return false;
        D[j] = djj;
        dmin = std::min(dmin, djj);
        dmax = std::max(dmax, djj);
        for (int i = j + 1; i < L; ++i) {
            Real v = a[static_cast<std::size_t>(i) * L + j];
            for (int k = 0; k < j; ++k)
                v -= a[static_cast<std::size_t>(i) * L + k] * a[static_cast<std::size_t>(j) * L + k] * D[k];
            a[static_cast<std::size_t>(i) * L + j] = v / djj;
        }
    }
    // z = L^-1 d, s = sum z_j^2 / D_j
    std::vector<Real> z(d);
    Real s = 0.0L;
    for (int j = 0; j < L; ++j) {
        for (int k = 0; k < j; ++k) z[j] -= a[static_cast<std::size_t>(j) * L + k] * z[k];
        s += z[j] * z[j] / D[j];
    }
    out = s;
    return true;
}

template <class Fn>
void for_pixels(long n, int workers, Fn&& fn) {
    workers = std::max(1, workers);
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w)
        pool.emplace_back([&, w] {
            for (long i = w; i < n; i += workers) fn(i);
        });
    for (auto& t : pool) t.join();
}

}  // namespace

extern "C" {

// LRX (detect.cpp:159-193; guard > 1 = the B200 guard extension) at n listed pixels.
// out[i] = max(score, 0), or NaN where the reference would raise SingularAfterRidge;
// pivot_ratio[i] = max D / min D of the LDL^T of C + delta I (a conditioning proxy).
void orc_hp_lrx_pixels(const void* cube, int eb, long lines, long samples, int bands, int window,
                       int guard, double ridge, long n, const long* rows, const long* cols,
                       double* out, double* pivot_ratio, int workers) {
    const CubeView c{cube, eb, lines, samples, bands};
    for_pixels(n, workers, [&](long i) {
        std::vector<Real> x, mu, cov, d(bands);
        int cnt = 0;
        gather(c, rows[i], cols[i], window, guard, x, cnt);
        mean_cov(x, cnt, bands, mu, cov);
        bool nz = false;
        for (int b = 0; b < bands; ++b) {
            d[b] = c.at(rows[i], cols[i], b) - mu[b];
            nz = nz || d[b] != 0.0L;
        }
        Real s = 0.0L, dmin = 1.0L, dmax = 1.0L;
        bool ok = true;
        if (nz) ok = quad_form(cov, d, bands, ridge, s, dmin, dmax);
        out[i] = ok ? static_cast<double>(std::max(s, 0.0L)) : NAN;
        if (pivot_ratio) pivot_ratio[i] = static_cast<double>(dmax / dmin);
    });
}

// DWRX (detect.cpp:195-228) at n listed pixels: |m^T (C_ann + delta I)^-1 m|.
void orc_hp_dwrx_pixels(const void* cube, int eb, long lines, long samples, int bands, int inner,
                        int outer, double ridge, long n, const long* rows, const long* cols,
                        double* out, double* pivot_ratio, int workers) {
    const CubeView c{cube, eb, lines, samples, bands};
    for_pixels(n, workers, [&](long i) {
        std::vector<Real> xin, xann, mu_in, mu_ann, cov_in, cov_ann, m(bands);
        int nin = 0;
        gather(c, rows[i], cols[i], inner, 0, xin, nin);
        // annulus: the outer box minus the inner box, in the same scan order
        const int ih = inner / 2, oh = outer / 2;
        int nann = 0;
        for (int dr = -oh; dr <= oh; ++dr) {
            const int rr = mirror(static_cast<int>(rows[i]) + dr, static_cast<int>(lines));
            for (int dc = -oh; dc <= oh; ++dc) {
                if (std::abs(dr) <= ih && std::abs(dc) <= ih) continue;
                const int cc = mirror(static_cast<int>(cols[i]) + dc, static_cast<int>(samples));
                for (int b = 0; b < bands; ++b) xann.push_back(c.at(rr, cc, b));
                ++nann;
            }
        }
        mean_cov(xin, nin, bands, mu_in, cov_in);
        mean_cov(xann, nann, bands, mu_ann, cov_ann);
        bool nz = false;
        for (int b = 0; b < bands; ++b) {
            m[b] = mu_in[b] - mu_ann[b];
            nz = nz || m[b] != 0.0L;
        }
        Real s = 0.0L, dmin = 1.0L, dmax = 1.0L;
        bool ok = true;
        if (nz) ok = quad_form(cov_ann, m, bands, ridge, s, dmin, dmax);
        out[i] = ok ? static_cast<double>(std::fabs(s)) : NAN;
        if (pivot_ratio) pivot_ratio[i] = static_cast<double>(dmax / dmin);
    });
}

}  // extern "C"
