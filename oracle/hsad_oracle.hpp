// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// CPU restatement ("the oracle") of the reference hot path of arXiv 1201.2025's
// "hsad" library: the db-N wavelet reduction and the LRX / DWRX / DWEST
// sliding-window detectors. Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it, and only as
// the checker or the timed CPU baseline — never as the measured GPU product.
//
// Every function cites the reference file:line it restates (paths relative
// to the reference checkout, proj/...). The reference itself needs Eigen3,
// which is absent from this image, so this is an Eigen-free restatement:
//   * Eigen's pivoted LDLT (used by regularized_inverse) is restated with the
//     same left-looking diagonal-pivot order and the same singular rule;
//   * Eigen's SelfAdjointEigenSolver is replaced by cyclic Jacobi run to
//     full fp64 accuracy, then sorted descending with the reference sign
//     rule (stats.cpp:64-89).
// It is pinned (tests/test_oracle_pin.py) against (a) every known-answer test
// of proj/tests for this path and (b) oracle/_ref, a build of the reference's
// own Eigen-free sources (wavelet.cpp, error.cpp, tests/support/oracles.cpp).
#pragma once

#include <cstdint>

extern "C" {

// errc numbering follows proj/core/include/hsad/error.hpp:10-32 (+1 so 0 = ok)
enum orc_status {
    ORC_OK = 0,
    ORC_MISSING_KEY,
    ORC_INVALID_VALUE,
    ORC_SIZE_MISMATCH,
    ORC_NON_FINITE_VALUE,
    ORC_OUT_OF_BOUNDS,
    ORC_UNSUPPORTED_ORDER,
    ORC_ODD_LENGTH,
    ORC_TOO_SHORT,
    ORC_LENGTH_MISMATCH,
    ORC_TARGET_TOO_LARGE,
    ORC_EMPTY_SAMPLE_SET,
    ORC_TOO_FEW_SAMPLES,
    ORC_SINGULAR_AFTER_RIDGE,
    ORC_NOT_SYMMETRIC,
    ORC_NO_CONVERGENCE,
    ORC_CONFIG_MISMATCH,
    ORC_FRACTION_OUT_OF_RANGE,
    ORC_OUT_OF_BOUNDS_IMPLANT,
    ORC_DIMENSION_MISMATCH,
    ORC_DEGENERATE_TRUTH,
    ORC_IO_FAILURE,
};

// Last error message of the calling thread ("<Name>: msg [at pixel (r, c)]").
const char* orc_last_error(void);

// --- wavelet (proj/core/src/wavelet.cpp) -------------------------------------
int orc_daubechies(int order, double* low, double* high, int* length);
int orc_dwt_level(const double* x, int n, int order, double* approx, double* detail);
int orc_idwt_level(const double* approx, const double* detail, int half, int order, double* out);
int orc_multilevel_approx(const double* x, int n, int order, int target, double* out);
// elem_bytes = 4 (fp32 cube widened per access, cube.cpp:219) or 8 (fp64 HyperCube)
int orc_reduce_cube(const void* cube, int elem_bytes, long lines, long samples, int bands,
                    int order, int target, double* out, int workers);

// --- window geometry (proj/core/src/detect.cpp:29-76) ------------------------
int orc_mirror_index(int i, int n);
// mode 0 = single(size=a), 1 = dual(inner=a, outer=b); returns status
int orc_window_validate(int mode, int a, int b);

// --- stats (proj/core/src/stats.cpp) -----------------------------------------
// samples: dim x count, column-major (one sample per column, like SampleSet)
int orc_mean_vector(const double* samples, int dim, int count, double* mean);
int orc_covariance(const double* samples, int dim, int count, const double* mean, double* cov);
int orc_regularized_inverse(const double* cov, int dim, double ridge, double* inv,
                            double* ridge_applied);
int orc_symmetric_eigen(const double* m, int dim, double* values, double* vectors);

// --- detectors (proj/core/src/detect.cpp:159-289) ------------------------------
// cube: lines x samples x bands BIP, elem_bytes 4|8. scores: lines*samples fp64.
// On a per-pixel failure returns the errc of the first failing pixel in
// row-major order and writes its coordinates to *err_row / *err_col.
int orc_local_rx(const void* cube, int elem_bytes, long lines, long samples, int bands,
                 int window, int guard, double ridge, double* scores, int workers,
                 long* err_row, long* err_col);
int orc_dwrx(const void* cube, int elem_bytes, long lines, long samples, int bands, int inner,
             int outer, double ridge, double* scores, int workers, long* err_row, long* err_col);
// eigcount (nullable): number of eigenvectors the DWEST loop summed (extension)
int orc_dwest(const void* cube, int elem_bytes, long lines, long samples, int bands, int inner,
              int outer, double eigen_fraction, double* scores, int8_t* eigcount, int workers,
              long* err_row, long* err_col);
// Same detectors restricted to output rows [row_begin, row_end) of the full
// image (used for bounded CPU-baseline samples and big-cube subset parity).
int orc_local_rx_rows(const void* cube, int elem_bytes, long lines, long samples, int bands,
                      long row_begin, long row_end, int window, int guard, double ridge,
                      double* scores, int workers, long* err_row, long* err_col);
int orc_dwrx_rows(const void* cube, int elem_bytes, long lines, long samples, int bands,
                  long row_begin, long row_end, int inner, int outer, double ridge,
                  double* scores, int workers, long* err_row, long* err_col);
int orc_dwest_rows(const void* cube, int elem_bytes, long lines, long samples, int bands,
                   long row_begin, long row_end, int inner, int outer, double eigen_fraction,
                   double* scores, int8_t* eigcount, int workers, long* err_row, long* err_col);

// Per-pixel DWEST decision margins (hazard budget): for each
// pixel the smallest relative distance of an eigenvalue to the cutoff
// f*lambda0 / to zero, and the smallest gap between the largest and second
// largest |component| of a summed eigenvector (sign-rule margin).
int orc_dwest_margins(const void* cube, int elem_bytes, long lines, long samples, int bands,
                      long row_begin, long row_end, int inner, int outer, double eigen_fraction,
                      double* cutoff_margin, double* sign_margin, int workers);

// --- RNG used by the reference's own tests (proj/core/include/hsad/rng.hpp) ---
// random_cube(lines, samples, bands, seed, lo, hi) of proj/tests/support/testutil.hpp:18-24
void orc_random_cube(long lines, long samples, int bands, uint64_t seed, double lo, double hi,
                     double* out);
void orc_random_signal(long length, uint64_t seed, double lo, double hi, double* out);
}
