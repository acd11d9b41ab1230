// TEST INFRASTRUCTURE ONLY — see hsad_oracle.hpp for the contract.
//
// Eigen-free CPU restatement of the reference hot path:
//   proj/core/src/wavelet.cpp:16-167   (taps, dwt_level, multilevel_approx, reduce_cube)
//   proj/core/src/stats.cpp:7-89       (mean, two-pass covariance, ridge + LDLT, eigen)
//   proj/core/src/detect.cpp:29-289    (window validation, mirror, gathers, detectors)
//   proj/core/src/parallel.hpp:17-40   (strided row workers, first error wins)
// The per-pixel arithmetic follows the reference's explicit-gather structure
// (gather window → mean → centred covariance → solve), not the GPU's sliding
// sums, so the two are independent derivations of the same scores.
#include "hsad_oracle.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_last_error;

const char* errc_name(int code) {
    // proj/core/src/error.cpp:5-30
    static const char* names[] = {"Ok",
                                  "MissingKey",
                                  "InvalidValue",
                                  "SizeMismatch",
                                  "NonFiniteValue",
                                  "OutOfBounds",
                                  "UnsupportedOrder",
                                  "OddLength",
                                  "TooShort",
                                  "LengthMismatch",
                                  "TargetTooLarge",
                                  "EmptySampleSet",
                                  "TooFewSamples",
                                  "SingularAfterRidge",
                                  "NotSymmetric",
                                  "NoConvergence",
                                  "ConfigMismatch",
                                  "FractionOutOfRange",
                                  "OutOfBoundsImplant",
                                  "DimensionMismatch",
                                  "DegenerateTruth",
                                  "IoFailure"};
    if (code < 0 || code > ORC_IO_FAILURE) return "UnknownError";
    return names[code];
}

// Mirrors hsad::Error: what() = "<Name>: <message>"
struct OrcError : std::runtime_error {
    int code;
    OrcError(int c, const std::string& msg)
        : std::runtime_error(std::string(errc_name(c)) + ": " + msg), code(c) {}
};

int fail(const OrcError& e) {
    g_last_error = e.what();
    return e.code;
}

// ----------------------------------------------------------------------------
// Daubechies scaling taps, orders 1..10 (the standard published minimal-phase
// constants, normalised to sum sqrt(2); proj/core/src/wavelet.cpp:16-49 holds
// the same constants). Admissibility is re-checked by the tests to 1e-12.
const std::vector<double> kTaps[10] = {
    {0.70710678118654752, 0.70710678118654752},
    {0.48296291314453414, 0.83651630373780791, 0.22414386804201338, -0.12940952255126038},
    {0.33267055295008262, 0.80689150931109258, 0.45987750211849157, -0.13501102001025459,
     -0.085441273882026662, 0.035226291885709537},
    {0.23037781330889650, 0.71484657055291565, 0.63088076792985891, -0.027983769416859854,
     -0.18703481171909308, 0.030841381835560764, 0.032883011666885200, -0.010597401785069032},
    {0.16010239797419291, 0.60382926979718967, 0.72430852843777293, 0.13842814590132073,
     -0.24229488706638203, -0.032244869584638375, 0.077571493840045714,
     -0.0062414902127982743, -0.012580751999081999, 0.0033357252854737713},
    {0.11154074335010946, 0.49462389039845309, 0.75113390802109535, 0.31525035170919763,
     -0.22626469396543982, -0.12976686756726194, 0.097501605587323049, 0.027522865530305729,
     -0.031582039317486030, 0.00055384220116149614, 0.0047772575109455106,
     -0.0010773010853084796},
    {0.077852054085009179, 0.39653931948191731, 0.72913209084623512, 0.46978228740519312,
     -0.14390600392856498, -0.22403618499387498, 0.071309219266830265, 0.080612609151083072,
     -0.038029936935014414, -0.016574541630666881, 0.012550998556099841,
     0.00042957797292136652, -0.0018016407040474909, 0.00035371379997452025},
    {0.054415842243104010, 0.31287159091429997, 0.67563073629728981, 0.58535468365420671,
     -0.015829105256349306, -0.28401554296154693, 0.00047248457391328277,
     0.12874742662047846, -0.017369301001807546, -0.044088253930794752,
     0.013981027917398282, 0.0087460940474057767, -0.0048703529934515743,
     -0.00039174037337694705, 0.00067544940645056937, -0.00011747678412476953},
    {0.038077947363878347, 0.24383467461259035, 0.60482312369011111, 0.65728807805130054,
     0.13319738582500758, -0.29327378327917491, -0.096840783222976461, 0.14854074933810638,
     0.030725681479333379, -0.067632829061329974, 0.00025094711483145196,
     0.022361662123679097, -0.0047232047577513973, -0.0042815036824634298,
     0.0018476468830562265, 0.00023038576352319597, -0.00025196318894271014,
     0.000039347320316271599},
    {0.026670057900555554, 0.18817680007769149, 0.52720118893172559, 0.68845903945360357,
     0.28117234366057746, -0.24984642432731538, -0.19594627437737704, 0.12736934033579326,
     0.093057364603572351, -0.071394147166397087, -0.029457536821875813,
     0.033212674059341002, 0.0036065535669561697, -0.010733175483330575,
     0.0013953517470529012, 0.0019924052951850561, -0.00068585669495971163,
     -0.00011646685512928545, 0.000093588670320069591, -0.000013264202894521245},
};

struct Filters {
    std::vector<double> low, high;
};

// wavelet.cpp:60-74 — high[n] = (-1)^n low[len-1-n]
Filters make_filters(int order) {
    if (order < 1 || order > 10)
        throw OrcError(ORC_UNSUPPORTED_ORDER,
                       "Daubechies order must be in 1..10, got " + std::to_string(order));
    Filters f;
    f.low = kTaps[order - 1];
    const std::size_t len = f.low.size();
    f.high.resize(len);
    for (std::size_t n = 0; n < len; ++n) {
        const double v = f.low[len - 1 - n];
        f.high[n] = (n % 2 == 0) ? v : -v;
    }
    return f;
}

// wavelet.cpp:51-56
void check_pow2(int value, int code, const char* what) {
    if (value < 2 || !std::has_single_bit(static_cast<unsigned>(value)))
        throw OrcError(code, std::string(what) + " must be a power of two >= 2, got " +
                                 std::to_string(value));
}

// wavelet.cpp:76-101 — approx[k] = sum_j low[j] x[(2k+j) mod n]
void dwt_level(const double* x, std::size_t n, const Filters& f, double* approx, double* detail) {
    const std::size_t taps = f.low.size();
    if (n % 2 != 0) throw OrcError(ORC_ODD_LENGTH, "signal length " + std::to_string(n) + " is odd");
    if (n < taps)
        throw OrcError(ORC_TOO_SHORT, "signal length " + std::to_string(n) +
                                          " shorter than filter length " + std::to_string(taps));
    for (std::size_t k = 0; k < n / 2; ++k) {
        double a = 0.0, d = 0.0;
        for (std::size_t j = 0; j < taps; ++j) {
            std::size_t idx = 2 * k + j;
            if (idx >= n) idx -= n;
            a += f.low[j] * x[idx];
            d += f.high[j] * x[idx];
        }
        approx[k] = a;
        if (detail) detail[k] = d;
    }
}

// wavelet.cpp:122-146 — half-sample mirror pad to bit_ceil(n), then low-pass cascade
std::vector<double> multilevel(const double* x, std::size_t n, const Filters& f, int target) {
    check_pow2(target, ORC_INVALID_VALUE, "target length");
    if (n == 0) throw OrcError(ORC_TOO_SHORT, "empty signal");
    const std::size_t padded = std::bit_ceil(n);
    if (static_cast<std::size_t>(target) > padded)
        throw OrcError(ORC_TARGET_TOO_LARGE, "target length " + std::to_string(target) +
                                                 " exceeds padded length " + std::to_string(padded));
    std::vector<double> cur(x, x + n);
    cur.reserve(padded);
    for (std::size_t k = 0; cur.size() < padded; ++k) cur.push_back(x[n - 1 - k]);
    std::vector<double> next;
    while (cur.size() > static_cast<std::size_t>(target)) {
        next.assign(cur.size() / 2, 0.0);
        dwt_level(cur.data(), cur.size(), f, next.data(), nullptr);
        cur.swap(next);
    }
    return cur;
}

// parallel.hpp:17-40 — worker w takes rows w, w+T, ...; the first error of the
// earliest failing pixel (row-major) is reported.
template <class Fn>
void parallel_rows(long row_begin, long row_end, int workers, Fn&& fn) {
    const long rows = row_end - row_begin;
    workers = std::clamp(workers, 1, rows > 0 ? static_cast<int>(std::min<long>(rows, 1024)) : 1);
    if (workers == 1) {
        for (long r = row_begin; r < row_end; ++r) fn(r);
        return;
    }
    std::mutex mu;
    std::exception_ptr first;
    long first_row = -1;
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w) {
        pool.emplace_back([&, w] {
            long r = row_begin + w;
            try {
                for (; r < row_end; r += workers) fn(r);
            } catch (...) {
                std::lock_guard<std::mutex> lock(mu);
                if (!first || r < first_row) {
                    first = std::current_exception();
                    first_row = r;
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    if (first) std::rethrow_exception(first);
}

// ----------------------------------------------------------------------------
// Cube view: BIP, widened to fp64 per access (cube.cpp:219 widens at load)
struct Cube {
    const void* data;
    int elem;
    long lines, samples;
    int bands;
    double at(long r, long c, int b) const {
        const std::size_t i = (static_cast<std::size_t>(r) * samples + c) * bands + b;
        return elem == 4 ? static_cast<double>(static_cast<const float*>(data)[i])
                         : static_cast<const double*>(data)[i];
    }
};

// detect.cpp:71-76
int mirror(int i, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    i = std::abs(i) % period;
    return i < n ? i : period - i;
}

// detect.cpp:29-69
void validate_window(int mode, int a, int b) {
    if (mode == 0) {
        if (a < 3 || a % 2 == 0)
            throw OrcError(ORC_INVALID_VALUE,
                           "single window size must be odd and >= 3, got " + std::to_string(a));
        return;
    }
    if (a < 1 || a % 2 == 0)
        throw OrcError(ORC_INVALID_VALUE,
                       "inner window size must be odd and >= 1, got " + std::to_string(a));
    if (b <= a || b % 2 == 0)
        throw OrcError(ORC_INVALID_VALUE,
                       "outer window size must be odd and > inner, got " + std::to_string(b));
    if (b - a < 2) throw OrcError(ORC_INVALID_VALUE, "outer window must exceed inner by at least 2");
    if (b * b - a * a < 2) throw OrcError(ORC_INVALID_VALUE, "outer annulus must contain at least 2 pixels");
}

// Sample set: dim x count, column-major (SampleSet::vectors, stats.hpp:10-16)
struct Samples {
    int dim = 0, count = 0;
    std::vector<double> v;
    double& at(int i, int j) { return v[static_cast<std::size_t>(j) * dim + i]; }
    double at(int i, int j) const { return v[static_cast<std::size_t>(j) * dim + i]; }
};

// detect.cpp:83-99 — row-major window scan, optional exclusion box (guard) around the centre
void gather_box(const Cube& cube, long row, long col, int size, int exclude, Samples& out) {
    const int half = size / 2, eh = exclude / 2;
    const int count = size * size - (exclude > 0 ? exclude * exclude : 0);
    out.dim = cube.bands;
    out.count = count;
    out.v.resize(static_cast<std::size_t>(count) * cube.bands);
    int idx = 0;
    for (int dr = -half; dr <= half; ++dr) {
        const int rr = mirror(static_cast<int>(row) + dr, static_cast<int>(cube.lines));
        for (int dc = -half; dc <= half; ++dc) {
            if (exclude > 0 && std::abs(dr) <= eh && std::abs(dc) <= eh) continue;
            const int cc = mirror(static_cast<int>(col) + dc, static_cast<int>(cube.samples));
            for (int b = 0; b < cube.bands; ++b) out.at(b, idx) = cube.at(rr, cc, b);
            ++idx;
        }
    }
}

// detect.cpp:101-117 — annulus |dr|>ih || |dc|>ih
void gather_annulus(const Cube& cube, long row, long col, int inner, int outer, Samples& out) {
    const int ih = inner / 2, oh = outer / 2;
    out.dim = cube.bands;
    out.count = outer * outer - inner * inner;
    out.v.resize(static_cast<std::size_t>(out.count) * cube.bands);
    int idx = 0;
    for (int dr = -oh; dr <= oh; ++dr) {
        const int rr = mirror(static_cast<int>(row) + dr, static_cast<int>(cube.lines));
        for (int dc = -oh; dc <= oh; ++dc) {
            if (std::abs(dr) <= ih && std::abs(dc) <= ih) continue;
            const int cc = mirror(static_cast<int>(col) + dc, static_cast<int>(cube.samples));
            for (int b = 0; b < cube.bands; ++b) out.at(b, idx) = cube.at(rr, cc, b);
            ++idx;
        }
    }
}

// stats.cpp:7-11
std::vector<double> mean_vector(const Samples& s) {
    if (s.count < 1) throw OrcError(ORC_EMPTY_SAMPLE_SET, "mean of zero samples");
    std::vector<double> mu(s.dim, 0.0);
    for (int j = 0; j < s.count; ++j)
        for (int i = 0; i < s.dim; ++i) mu[i] += s.at(i, j);
    for (auto& m : mu) m /= static_cast<double>(s.count);
    return mu;
}

// stats.cpp:13-29 — centred X X^T / N, then 0.5 (C + C^T); C is dim x dim column-major
std::vector<double> covariance(const Samples& s, const std::vector<double>& mean) {
    const int n = s.count;
    if (n < 2)
        throw OrcError(ORC_TOO_FEW_SAMPLES,
                       "covariance needs at least 2 samples, got " + std::to_string(n));
    if (static_cast<int>(mean.size()) != s.dim)
        throw OrcError(ORC_LENGTH_MISMATCH, "mean length does not match sample dimension");
    const int d = s.dim;
    std::vector<double> centred(static_cast<std::size_t>(d) * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < d; ++i) centred[static_cast<std::size_t>(j) * d + i] = s.at(i, j) - mean[i];
    std::vector<double> c(static_cast<std::size_t>(d) * d, 0.0);
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            double acc = 0.0;
            for (int j = 0; j < n; ++j)
                acc += centred[static_cast<std::size_t>(j) * d + a] *
                       centred[static_cast<std::size_t>(j) * d + b];
            c[static_cast<std::size_t>(b) * d + a] = acc / static_cast<double>(n);
        }
    for (int a = 0; a < d; ++a)
        for (int b = a + 1; b < d; ++b) {
            const double v = 0.5 * (c[static_cast<std::size_t>(b) * d + a] +
                                    c[static_cast<std::size_t>(a) * d + b]);
            c[static_cast<std::size_t>(b) * d + a] = v;
            c[static_cast<std::size_t>(a) * d + b] = v;
        }
    return c;
}

// Left-looking LDL^T with diagonal pivoting on the (not yet updated) trailing
// diagonal — the factorisation Eigen's LDLT<MatrixXd> performs — so the
// singular rule of stats.cpp:42-53 sees the same D.
struct Ldlt {
    int n = 0;
    std::vector<double> m;   // column-major; strict lower = L, diagonal = D
    std::vector<int> trans;  // transpositions
    bool ok = true;
    double& at(int i, int j) { return m[static_cast<std::size_t>(j) * n + i]; }
};

Ldlt ldlt_factor(const std::vector<double>& a, int n) {
    Ldlt f;
    f.n = n;
    f.m = a;
    f.trans.assign(n, 0);
    std::vector<double> temp(n);
    bool found_zero_pivot = false;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::abs(f.at(k, k));
        for (int i = k + 1; i < n; ++i)
            if (std::abs(f.at(i, i)) > best) {
                best = std::abs(f.at(i, i));
                p = i;
            }
        f.trans[k] = p;
        if (p != k) {
            // symmetric swap using only the lower triangle
            for (int j = 0; j < k; ++j) std::swap(f.at(k, j), f.at(p, j));
            for (int i = p + 1; i < n; ++i) std::swap(f.at(i, k), f.at(i, p));
            std::swap(f.at(k, k), f.at(p, p));
            for (int i = k + 1; i < p; ++i) {
                const double t = f.at(i, k);
                f.at(i, k) = f.at(p, i);
                f.at(p, i) = t;
            }
        }
        const int rs = n - k - 1;
        if (k > 0) {
            for (int j = 0; j < k; ++j) temp[j] = f.at(j, j) * f.at(k, j);
            double s = 0.0;
            for (int j = 0; j < k; ++j) s += f.at(k, j) * temp[j];
            f.at(k, k) -= s;
            for (int i = k + 1; i < n; ++i) {
                double t = 0.0;
                for (int j = 0; j < k; ++j) t += f.at(i, j) * temp[j];
                f.at(i, k) -= t;
            }
        }
        const double akk = f.at(k, k);
        const bool valid = std::abs(akk) > 0.0;
        if (k == 0 && !valid) {
            // entire diagonal zero: D = 0 everywhere
            for (int j = 0; j < n; ++j) {
                f.trans[j] = j;
                for (int i = 0; i < n; ++i) f.at(i, j) = 0.0;
            }
            return f;
        }
        if (rs > 0 && valid) {
            for (int i = k + 1; i < n; ++i) f.at(i, k) /= akk;
        } else if (rs > 0) {
            for (int i = k + 1; i < n; ++i) f.ok = f.ok && f.at(i, k) == 0.0;
        }
        if (found_zero_pivot && valid) f.ok = false;
        else if (!valid) found_zero_pivot = true;
    }
    return f;
}

// LDLT::solve(I): P, L^-1, D^+, L^-T, P^T applied column by column
std::vector<double> ldlt_inverse(Ldlt& f) {
    const int n = f.n;
    std::vector<double> x(static_cast<std::size_t>(n) * n, 0.0);
    const double tiny = std::numeric_limits<double>::min();
    for (int c = 0; c < n; ++c) {
        std::vector<double> v(n, 0.0);
        v[c] = 1.0;
        for (int k = 0; k < n; ++k) std::swap(v[k], v[f.trans[k]]);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < i; ++j) v[i] -= f.at(i, j) * v[j];
        for (int i = 0; i < n; ++i) v[i] = std::abs(f.at(i, i)) > tiny ? v[i] / f.at(i, i) : 0.0;
        for (int i = n - 1; i >= 0; --i)
            for (int j = i + 1; j < n; ++j) v[i] -= f.at(j, i) * v[j];
        for (int k = n - 1; k >= 0; --k) std::swap(v[k], v[f.trans[k]]);
        for (int i = 0; i < n; ++i) x[static_cast<std::size_t>(c) * n + i] = v[i];
    }
    return x;
}

std::string fmt_fixed(double v) { return std::to_string(v); }

// stats.cpp:31-62
std::vector<double> regularized_inverse(const std::vector<double>& c, int dim, double ridge,
                                        double* applied) {
    if (dim == 0) throw OrcError(ORC_DIMENSION_MISMATCH, "covariance matrix is not square");
    if (ridge < 0.0) throw OrcError(ORC_INVALID_VALUE, "ridge fraction must be nonnegative");
    double trace = 0.0;
    for (int i = 0; i < dim; ++i) trace += c[static_cast<std::size_t>(i) * dim + i];
    const double delta = ridge * trace / static_cast<double>(dim);
    std::vector<double> loaded = c;
    for (int i = 0; i < dim; ++i) loaded[static_cast<std::size_t>(i) * dim + i] += delta;
    Ldlt f = ldlt_factor(loaded, dim);
    bool singular = !f.ok;
    if (!singular) {
        double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
        for (int i = 0; i < dim; ++i) {
            dmax = std::max(dmax, std::abs(f.at(i, i)));
            dmin = std::min(dmin, f.at(i, i));
        }
        singular = !(dmax > 0.0) || dmin <= dmax * 1e-14;
    }
    if (singular)
        throw OrcError(ORC_SINGULAR_AFTER_RIDGE,
                       "covariance numerically singular (ridge " + fmt_fixed(delta) + ")");
    std::vector<double> inv = ldlt_inverse(f);
    for (int a = 0; a < dim; ++a)
        for (int b = a + 1; b < dim; ++b) {
            const double v = 0.5 * (inv[static_cast<std::size_t>(b) * dim + a] +
                                    inv[static_cast<std::size_t>(a) * dim + b]);
            inv[static_cast<std::size_t>(b) * dim + a] = v;
            inv[static_cast<std::size_t>(a) * dim + b] = v;
        }
    for (double v : inv)
        if (!std::isfinite(v)) throw OrcError(ORC_SINGULAR_AFTER_RIDGE, "inverse overflowed");
    if (applied) *applied = delta;
    return inv;
}

// stats.cpp:64-89 with the eigensolver restated as cyclic Jacobi (textbook
// two-sided rotations, tan-half-angle updates) run to full fp64 accuracy.
struct Eig {
    std::vector<double> values;   // descending
    std::vector<double> vectors;  // column-major, column i = eigenvector i
};

Eig symmetric_eigen(const std::vector<double>& mat, int n) {
    if (n == 0) throw OrcError(ORC_DIMENSION_MISMATCH, "matrix is not square");
    double scale = 0.0, asym = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            scale = std::max(scale, std::abs(mat[static_cast<std::size_t>(j) * n + i]));
            asym = std::max(asym, std::abs(mat[static_cast<std::size_t>(j) * n + i] -
                                           mat[static_cast<std::size_t>(i) * n + j]));
        }
    if (asym > 1e-8 * std::max(scale, 1.0)) throw OrcError(ORC_NOT_SYMMETRIC, "matrix is not symmetric");

    std::vector<double> a = mat, v(static_cast<std::size_t>(n) * n, 0.0);
    auto A = [&](int i, int j) -> double& { return a[static_cast<std::size_t>(j) * n + i]; };
    auto V = [&](int i, int j) -> double& { return v[static_cast<std::size_t>(j) * n + i]; };
    for (int i = 0; i < n; ++i) V(i, i) = 1.0;
    bool converged = false;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += std::abs(A(p, q));
        if (off == 0.0) {
            converged = true;
            break;
        }
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A(p, q);
                const double g = 100.0 * std::abs(apq);
                // negligible off-diagonal after a few sweeps: zero it exactly
                if (sweep > 3 && std::abs(A(p, p)) + g == std::abs(A(p, p)) &&
                    std::abs(A(q, q)) + g == std::abs(A(q, q))) {
                    A(p, q) = 0.0;
                    A(q, p) = 0.0;
                    continue;
                }
                if (apq == 0.0) continue;
                const double h = A(q, q) - A(p, p);
                double t;
                if (std::abs(h) + g == std::abs(h)) {
                    t = apq / h;
                } else {
                    const double theta = 0.5 * h / apq;
                    t = 1.0 / (std::abs(theta) + std::sqrt(1.0 + theta * theta));
                    if (theta < 0.0) t = -t;
                }
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double s = t * c;
                const double tau = s / (1.0 + c);
                A(p, p) -= t * apq;
                A(q, q) += t * apq;
                A(p, q) = 0.0;
                A(q, p) = 0.0;
                for (int k = 0; k < n; ++k) {
                    if (k == p || k == q) continue;
                    const double akp = A(k, p), akq = A(k, q);
                    A(k, p) = akp - s * (akq + tau * akp);
                    A(k, q) = akq + s * (akp - tau * akq);
                    A(p, k) = A(k, p);
                    A(q, k) = A(k, q);
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V(k, p), vkq = V(k, q);
                    V(k, p) = vkp - s * (vkq + tau * vkp);
                    V(k, q) = vkq + s * (vkp - tau * vkq);
                }
            }
    }
    if (!converged) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += std::abs(A(p, q));
        if (off != 0.0) throw OrcError(ORC_NO_CONVERGENCE, "eigensolver did not converge");
    }
    // descending order (stable on ties), sign: first largest-|.| component positive
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return A(x, x) > A(y, y); });
    Eig out;
    out.values.resize(n);
    out.vectors.assign(static_cast<std::size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) {
        const int src = order[i];
        out.values[i] = A(src, src);
        int argmax = 0;
        double best = -1.0;
        for (int k = 0; k < n; ++k)
            if (std::abs(V(k, src)) > best) {
                best = std::abs(V(k, src));
                argmax = k;
            }
        const double sign = V(argmax, src) < 0.0 ? -1.0 : 1.0;
        for (int k = 0; k < n; ++k) out.vectors[static_cast<std::size_t>(i) * n + k] = sign * V(k, src);
    }
    return out;
}

double quad_form(const std::vector<double>& d, const std::vector<double>& m) {
    // Eigen: d.dot(M * d) — matrix-vector first
    const int n = static_cast<int>(d.size());
    std::vector<double> md(n, 0.0);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) md[i] += m[static_cast<std::size_t>(j) * n + i] * d[j];
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += d[i] * md[i];
    return s;
}

bool any_nonzero(const std::vector<double>& v) {
    double m = 0.0;
    for (double x : v) m = std::max(m, std::abs(x));
    return m > 0.0;
}

[[noreturn]] void rethrow_at_pixel(const OrcError& e, long row, long col) {
    // detect.cpp:127-130: message keeps the "<Name>: " prefix of the inner error
    throw OrcError(e.code, std::string(e.what()) + " at pixel (" + std::to_string(row) + ", " +
                               std::to_string(col) + ")");
}

struct PixelFailure {
    int code;
    long row, col;
    std::string msg;
};

// Runs fn(row, col) over rows [rb, re) x all columns; returns the failure of the
// earliest pixel in row-major order (reference workers=1 semantics).
template <class Fn>
int run_pixels(long rb, long re, long samples, int workers, long* err_row, long* err_col, Fn&& fn) {
    try {
        parallel_rows(rb, re, workers, [&](long row) {
            for (long col = 0; col < samples; ++col) {
                try {
                    fn(row, col);
                } catch (const OrcError& e) {
                    if (err_row) *err_row = row;
                    if (err_col) *err_col = col;
                    rethrow_at_pixel(e, row, col);
                }
            }
        });
    } catch (const OrcError& e) {
        return fail(e);
    }
    return ORC_OK;
}

// detect.cpp:159-193 (+ guard extension: exclude a guard x guard box instead of the centre only)
int lrx_rows(const Cube& cube, long rb, long re, int window, int guard, double ridge, double* scores,
             int workers, long* er, long* ec) {
    try {
        validate_window(0, window, 0);
        if (guard < 1 || guard % 2 == 0 || guard >= window)
            throw OrcError(ORC_INVALID_VALUE, "guard window must be odd, >= 1 and < window, got " +
                                                  std::to_string(guard));
    } catch (const OrcError& e) {
        return fail(e);
    }
    return run_pixels(rb, re, cube.samples, workers, er, ec, [&](long row, long col) {
        thread_local Samples bg;
        gather_box(cube, row, col, window, guard, bg);
        const auto mu = mean_vector(bg);
        std::vector<double> diff(cube.bands);
        for (int b = 0; b < cube.bands; ++b) diff[b] = cube.at(row, col, b) - mu[b];
        double score = 0.0;
        if (any_nonzero(diff)) {
            const auto inv = regularized_inverse(covariance(bg, mu), cube.bands, ridge, nullptr);
            score = quad_form(diff, inv);
        }
        scores[(row - rb) * cube.samples + col] = std::max(score, 0.0);
    });
}

// detect.cpp:195-228
int dwrx_rows(const Cube& cube, long rb, long re, int inner, int outer, double ridge,
              double* scores, int workers, long* er, long* ec) {
    try {
        validate_window(1, inner, outer);
    } catch (const OrcError& e) {
        return fail(e);
    }
    return run_pixels(rb, re, cube.samples, workers, er, ec, [&](long row, long col) {
        thread_local Samples in, out;
        gather_box(cube, row, col, inner, 0, in);
        gather_annulus(cube, row, col, inner, outer, out);
        const auto m_out = mean_vector(out);
        auto m_diff = mean_vector(in);
        for (int b = 0; b < cube.bands; ++b) m_diff[b] -= m_out[b];
        double score = 0.0;
        if (any_nonzero(m_diff)) {
            const auto inv = regularized_inverse(covariance(out, m_out), cube.bands, ridge, nullptr);
            score = std::abs(quad_form(m_diff, inv));
        }
        scores[(row - rb) * cube.samples + col] = score;
    });
}

struct DwestPixel {
    double score;
    int count;
    double cutoff_margin;
    double sign_margin;
};

// detect.cpp:242-271 for one pixel
DwestPixel dwest_pixel(const Cube& cube, long row, long col, int inner, int outer, double frac) {
    thread_local Samples in, out;
    gather_box(cube, row, col, inner, 0, in);
    gather_annulus(cube, row, col, inner, outer, out);
    const auto m_in = mean_vector(in);
    const auto m_out = mean_vector(out);
    const int n = cube.bands;
    std::vector<double> m_diff(n);
    for (int b = 0; b < n; ++b) m_diff[b] = m_in[b] - m_out[b];
    const auto c_in = covariance(in, m_in);
    const auto c_out = covariance(out, m_out);
    std::vector<double> c_diff(c_in.size());
    for (std::size_t i = 0; i < c_in.size(); ++i) c_diff[i] = c_in[i] - c_out[i];
    const Eig eig = symmetric_eigen(c_diff, n);
    DwestPixel px{0.0, 0, std::numeric_limits<double>::infinity(),
                  std::numeric_limits<double>::infinity()};
    const double lmax = n > 0 ? eig.values[0] : 0.0;
    const double scale = std::max(std::abs(lmax), 1e-300);
    px.cutoff_margin = std::abs(lmax) / scale;  // margin of the lambda0 > 0 test (relative)
    if (lmax > 0.0) {
        double projected = 0.0;
        for (int i = 0; i < n; ++i) {
            const double li = eig.values[i];
            if (i > 0) {
                px.cutoff_margin = std::min(px.cutoff_margin, std::abs(li - frac * lmax) / scale);
                px.cutoff_margin = std::min(px.cutoff_margin, std::abs(li) / scale);
            }
            if (li <= 0.0 || li < frac * lmax) break;
            const double* v = &eig.vectors[static_cast<std::size_t>(i) * n];
            double a1 = -1.0, a2 = -1.0;
            for (int k = 0; k < n; ++k) {
                const double av = std::abs(v[k]);
                if (av > a1) {
                    a2 = a1;
                    a1 = av;
                } else if (av > a2) {
                    a2 = av;
                }
            }
            if (n > 1) px.sign_margin = std::min(px.sign_margin, a1 - a2);
            double dot = 0.0;
            for (int k = 0; k < n; ++k) dot += v[k] * m_diff[k];
            projected += dot;
            ++px.count;
        }
        px.score = std::abs(projected);
    }
    return px;
}

int dwest_rows(const Cube& cube, long rb, long re, int inner, int outer, double frac,
               double* scores, int8_t* eigcount, int workers, long* er, long* ec) {
    try {
        validate_window(1, inner, outer);
        if (!(frac > 0.0 && frac <= 1.0))
            throw OrcError(ORC_INVALID_VALUE, "eigen fraction must be in (0, 1]");
    } catch (const OrcError& e) {
        return fail(e);
    }
    return run_pixels(rb, re, cube.samples, workers, er, ec, [&](long row, long col) {
        const DwestPixel px = dwest_pixel(cube, row, col, inner, outer, frac);
        const std::size_t o = (row - rb) * cube.samples + col;
        scores[o] = px.score;
        if (eigcount) eigcount[o] = static_cast<int8_t>(px.count);
    });
}

Samples samples_from(const double* s, int dim, int count) {
    Samples out;
    out.dim = dim;
    out.count = count;
    out.v.assign(s, s + static_cast<std::size_t>(dim) * count);
    return out;
}

// proj/core/include/hsad/rng.hpp:13-64 — xoshiro256++ seeded through splitmix64
struct Xoshiro {
    uint64_t s[4];
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (auto& w : s) {
            x += 0x9e3779b97f4a7c15ULL;
            uint64_t z = x;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            w = z ^ (z >> 31);
        }
    }
    static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    uint64_t next() {
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

} // namespace

extern "C" {

const char* orc_last_error(void) { return g_last_error.c_str(); }

int orc_daubechies(int order, double* low, double* high, int* length) {
    try {
        const Filters f = make_filters(order);
        for (std::size_t i = 0; i < f.low.size(); ++i) {
            if (low) low[i] = f.low[i];
            if (high) high[i] = f.high[i];
        }
        if (length) *length = static_cast<int>(f.low.size());
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_dwt_level(const double* x, int n, int order, double* approx, double* detail) {
    try {
        dwt_level(x, static_cast<std::size_t>(n), make_filters(order), approx, detail);
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

// wavelet.cpp:103-120 — adjoint synthesis
int orc_idwt_level(const double* approx, const double* detail, int half, int order, double* out) {
    try {
        const Filters f = make_filters(order);
        const std::size_t n = static_cast<std::size_t>(half) * 2, taps = f.low.size();
        std::fill(out, out + n, 0.0);
        for (std::size_t k = 0; k < static_cast<std::size_t>(half); ++k)
            for (std::size_t j = 0; j < taps; ++j) {
                const std::size_t idx = (2 * k + j) % n;
                out[idx] += approx[k] * f.low[j] + detail[k] * f.high[j];
            }
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_multilevel_approx(const double* x, int n, int order, int target, double* out) {
    try {
        const auto a = multilevel(x, static_cast<std::size_t>(n), make_filters(order), target);
        std::copy(a.begin(), a.end(), out);
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

// wavelet.cpp:148-167
int orc_reduce_cube(const void* cube, int elem_bytes, long lines, long samples, int bands,
                    int order, int target, double* out, int workers) {
    try {
        const Filters f = make_filters(order);
        check_pow2(target, ORC_INVALID_VALUE, "target bands");
        const Cube c{cube, elem_bytes, lines, samples, bands};
        {
            // fail-fast probe on pixel (0,0) (wavelet.cpp:153-156); an empty cube
            // is probed with a zero spectrum so contract errors still surface
            std::vector<double> probe(bands, 0.0);
            if (lines > 0 && samples > 0)
                for (int b = 0; b < bands; ++b) probe[b] = c.at(0, 0, b);
            (void)multilevel(probe.data(), probe.size(), f, target);
        }
        parallel_rows(0, lines, workers, [&](long row) {
            std::vector<double> px(bands);
            for (long col = 0; col < samples; ++col) {
                for (int b = 0; b < bands; ++b) px[b] = c.at(row, col, b);
                const auto a = multilevel(px.data(), px.size(), f, target);
                std::copy(a.begin(), a.end(), out + (row * samples + col) * target);
            }
        });
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_mirror_index(int i, int n) { return mirror(i, n); }

int orc_window_validate(int mode, int a, int b) {
    try {
        validate_window(mode, a, b);
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_mean_vector(const double* s, int dim, int count, double* mean) {
    try {
        const auto mu = mean_vector(samples_from(s, dim, count));
        std::copy(mu.begin(), mu.end(), mean);
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_covariance(const double* s, int dim, int count, const double* mean, double* cov) {
    try {
        const auto c = covariance(samples_from(s, dim, count), std::vector<double>(mean, mean + dim));
        std::copy(c.begin(), c.end(), cov);
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_regularized_inverse(const double* cov, int dim, double ridge, double* inv,
                            double* ridge_applied) {
    try {
        const auto r = regularized_inverse(
            std::vector<double>(cov, cov + static_cast<std::size_t>(dim) * dim), dim, ridge,
            ridge_applied);
        std::copy(r.begin(), r.end(), inv);
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_symmetric_eigen(const double* m, int dim, double* values, double* vectors) {
    try {
        const Eig e = symmetric_eigen(std::vector<double>(m, m + static_cast<std::size_t>(dim) * dim), dim);
        std::copy(e.values.begin(), e.values.end(), values);
        std::copy(e.vectors.begin(), e.vectors.end(), vectors);
        return ORC_OK;
    } catch (const OrcError& e) {
        return fail(e);
    }
}

int orc_local_rx(const void* cube, int eb, long lines, long samples, int bands, int window,
                 int guard, double ridge, double* scores, int workers, long* er, long* ec) {
    return lrx_rows(Cube{cube, eb, lines, samples, bands}, 0, lines, window, guard, ridge, scores,
                    workers, er, ec);
}
int orc_dwrx(const void* cube, int eb, long lines, long samples, int bands, int inner, int outer,
             double ridge, double* scores, int workers, long* er, long* ec) {
    return dwrx_rows(Cube{cube, eb, lines, samples, bands}, 0, lines, inner, outer, ridge, scores,
                     workers, er, ec);
}
int orc_dwest(const void* cube, int eb, long lines, long samples, int bands, int inner, int outer,
              double frac, double* scores, int8_t* eigcount, int workers, long* er, long* ec) {
    return dwest_rows(Cube{cube, eb, lines, samples, bands}, 0, lines, inner, outer, frac, scores,
                      eigcount, workers, er, ec);
}
int orc_local_rx_rows(const void* cube, int eb, long lines, long samples, int bands, long rb,
                      long re, int window, int guard, double ridge, double* scores, int workers,
                      long* er, long* ec) {
    return lrx_rows(Cube{cube, eb, lines, samples, bands}, rb, re, window, guard, ridge, scores,
                    workers, er, ec);
}
int orc_dwrx_rows(const void* cube, int eb, long lines, long samples, int bands, long rb, long re,
                  int inner, int outer, double ridge, double* scores, int workers, long* er,
                  long* ec) {
    return dwrx_rows(Cube{cube, eb, lines, samples, bands}, rb, re, inner, outer, ridge, scores,
                     workers, er, ec);
}
int orc_dwest_rows(const void* cube, int eb, long lines, long samples, int bands, long rb, long re,
                   int inner, int outer, double frac, double* scores, int8_t* eigcount, int workers,
                   long* er, long* ec) {
    return dwest_rows(Cube{cube, eb, lines, samples, bands}, rb, re, inner, outer, frac, scores,
                      eigcount, workers, er, ec);
}

int orc_dwest_margins(const void* cube, int eb, long lines, long samples, int bands, long rb,
                      long re, int inner, int outer, double frac, double* cutoff_margin,
                      double* sign_margin, int workers) {
    const Cube c{cube, eb, lines, samples, bands};
    return run_pixels(rb, re, samples, workers, nullptr, nullptr, [&](long row, long col) {
        const DwestPixel px = dwest_pixel(c, row, col, inner, outer, frac);
        const std::size_t o = (row - rb) * samples + col;
        cutoff_margin[o] = px.cutoff_margin;
        sign_margin[o] = px.sign_margin;
    });
}

void orc_random_cube(long lines, long samples, int bands, uint64_t seed, double lo, double hi,
                     double* out) {
    Xoshiro rng(seed);
    const std::size_t n = static_cast<std::size_t>(lines) * samples * bands;
    for (std::size_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * rng.uniform01();
}

void orc_random_signal(long length, uint64_t seed, double lo, double hi, double* out) {
    Xoshiro rng(seed);
    for (long i = 0; i < length; ++i) out[i] = lo + (hi - lo) * rng.uniform01();
}

} // extern "C"
