// TEST INFRASTRUCTURE ONLY. extern "C" entry points over the reference's own
// Eigen-free sources, compiled in place from /root/reference by oracle/Makefile
// into oracle/_ref/libhsad_ref.so (never copied into this repo):
//   proj/core/src/wavelet.cpp        daubechies_filters, dwt_level, multilevel_approx, reduce_cube
//   proj/core/src/error.cpp          errc names
//   proj/tests/support/oracles.cpp   brute_dwt, brute_covariance, gauss_jordan_inverse,
//                                    jacobi_eigen, naive_lrx, naive_dwrx, naive_dwest
// The reference detectors themselves (detect.cpp/stats.cpp) need Eigen3 and
// cannot be built here; the reference's naive oracles are its own independent
// implementation of them, agreeing with the Eigen build to <= 2.7e-15
// (proj/test_output.txt:45).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "hsad/wavelet.hpp"
#include "oracles.hpp"

namespace {
thread_local std::string g_msg;
int fail(const hsad::Error& e) {
    g_msg = e.what();
    return static_cast<int>(e.code()) + 1;
}
hsad::HyperCube make_cube(const double* v, int lines, int samples, int bands) {
    hsad::HyperCube c(lines, samples, bands);
    std::memcpy(c.values.data(), v, sizeof(double) * c.values.size());
    return c;
}
} // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

int ref_daubechies(int order, double* low, double* high, int* length) {
    try {
        auto f = hsad::daubechies_filters(order);
        for (std::size_t i = 0; i < f.low.size(); ++i) {
            low[i] = f.low[i];
            high[i] = f.high[i];
        }
        *length = static_cast<int>(f.low.size());
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

int ref_dwt_level(const double* x, int n, int order, double* approx, double* detail) {
    try {
        auto b = hsad::dwt_level(std::span<const double>(x, n), hsad::daubechies_filters(order));
        std::memcpy(approx, b.approx.data(), sizeof(double) * b.approx.size());
        std::memcpy(detail, b.detail.data(), sizeof(double) * b.detail.size());
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

int ref_idwt_level(const double* a, const double* d, int half, int order, double* out) {
    try {
        auto x = hsad::idwt_level(std::span<const double>(a, half), std::span<const double>(d, half),
                                  hsad::daubechies_filters(order));
        std::memcpy(out, x.data(), sizeof(double) * x.size());
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

int ref_multilevel_approx(const double* x, int n, int order, int target, double* out) {
    try {
        auto a = hsad::multilevel_approx(std::span<const double>(x, n),
                                         hsad::daubechies_filters(order), target);
        std::memcpy(out, a.data(), sizeof(double) * a.size());
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

int ref_reduce_cube(const double* cube, int lines, int samples, int bands, int order, int target,
                    double* out, int workers) {
    try {
        auto in = make_cube(cube, lines, samples, bands);
        auto r = hsad::reduce_cube(in, hsad::daubechies_filters(order), target, workers);
        std::memcpy(out, r.values.data(), sizeof(double) * r.values.size());
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

int ref_brute_dwt(const double* x, int n, int order, double* approx, double* detail) {
    auto [a, d] = oracle::brute_dwt(std::vector<double>(x, x + n), hsad::daubechies_filters(order));
    std::memcpy(approx, a.data(), sizeof(double) * a.size());
    std::memcpy(detail, d.data(), sizeof(double) * d.size());
    return 0;
}

// samples: count rows of dim (row-major, one sample per row)
int ref_brute_covariance(const double* s, int dim, int count, double* cov) {
    std::vector<std::vector<double>> rows(count, std::vector<double>(dim));
    for (int j = 0; j < count; ++j)
        for (int i = 0; i < dim; ++i) rows[j][i] = s[j * dim + i];
    auto c = oracle::brute_covariance(rows);
    for (int i = 0; i < dim; ++i)
        for (int k = 0; k < dim; ++k) cov[i * dim + k] = c[i][k];
    return 0;
}

int ref_jacobi_eigen(const double* m, int n, double* values, double* vectors) {
    oracle::Matrix a(n, std::vector<double>(n));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) a[i][j] = m[i * n + j];
    auto r = oracle::jacobi_eigen(a);
    for (int i = 0; i < n; ++i) {
        values[i] = r.values[i];
        for (int k = 0; k < n; ++k) vectors[k * n + i] = r.vectors[k][i];  // row-major V
    }
    return 0;
}

int ref_naive_lrx(const double* cube, int lines, int samples, int bands, int window, double ridge,
                  double* scores) {
    auto s = oracle::naive_lrx(make_cube(cube, lines, samples, bands), window, ridge);
    std::memcpy(scores, s.data(), sizeof(double) * s.size());
    return 0;
}

int ref_naive_dwrx(const double* cube, int lines, int samples, int bands, int inner, int outer,
                   double ridge, double* scores) {
    auto s = oracle::naive_dwrx(make_cube(cube, lines, samples, bands), inner, outer, ridge);
    std::memcpy(scores, s.data(), sizeof(double) * s.size());
    return 0;
}

int ref_naive_dwest(const double* cube, int lines, int samples, int bands, int inner, int outer,
                    double frac, double* scores) {
    auto s = oracle::naive_dwest(make_cube(cube, lines, samples, bands), inner, outer, frac);
    std::memcpy(scores, s.data(), sizeof(double) * s.size());
    return 0;
}

} // extern "C"
