// hsad_b200.hpp — header-only C++ drop-in for the reference's detector API
// (proj/core/include/hsad/{error,cube,wavelet,detect}.hpp), implemented over the
// C-ABI of include/hsad_gpu.h (libhsad_b200.so, sm_100a kernels).
//
// Same names, argument meaning and error behaviour as the reference:
//   hsad::Error / hsad::errc               error.hpp:10-45
//   hsad::HyperCube (BIP fp64)             cube.hpp:42-64 (the subset the hot path uses)
//   hsad::daubechies_filters, reduce_cube  wavelet.hpp:24, 55-56
//   hsad::WindowConfig, DwestConfig,
//   DetectOptions, ScoreMap, mirror_index,
//   local_rx, dwrx, dwest, detect          detect.hpp:13-92
// The cube is copied to the device, the kernels run, the map is copied back;
// ScoreMap::seconds is the wall time of the call (detect.cpp:142-146). `workers`
// is accepted and recorded but the GPU grid replaces the row threads. The
// reference's Eigen types (Spectrum, SampleSet) are not part of this surface.
// Link: -lhsad_b200 -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hsad_gpu.h"

namespace hsad {

enum class errc {
    missing_key, invalid_value, size_mismatch, non_finite_value, out_of_bounds, unsupported_order,
    odd_length, too_short, length_mismatch, target_too_large, empty_sample_set, too_few_samples,
    singular_after_ridge, not_symmetric, no_convergence, config_mismatch, fraction_out_of_range,
    out_of_bounds_implant, dimension_mismatch, degenerate_truth, io_failure,
};

inline const char* errc_name(errc code) noexcept {
    return hsad_status_name(static_cast<int32_t>(code) + 1);
}

/// what() = "<Name>: <message>" exactly as the reference (error.hpp:36-45). B200-only
/// failures (CUDA runtime, kernel limits) surface as errc::io_failure with the
/// CUDA text in the message.
class Error : public std::runtime_error {
public:
    Error(errc code, const std::string& what_full) : std::runtime_error(what_full), code_(code) {}
    errc code() const noexcept { return code_; }

private:
    errc code_;
};

namespace detail {
inline void check(int32_t status) {
    if (status == HSAD_OK) return;
    const std::string msg = hsad_last_error_message();
    if (status >= 1 && status <= HSAD_E_IO_FAILURE) throw Error(static_cast<errc>(status - 1), msg);
    throw Error(errc::io_failure, msg);
}
inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(errc::io_failure, std::string("IoFailure: ") + what + ": " + cudaGetErrorString(e));
}
struct DeviceBuffer {
    void* p = nullptr;
    explicit DeviceBuffer(size_t bytes) { cuda(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
    ~DeviceBuffer() { cudaFree(p); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};
}  // namespace detail

enum class Interleave { BSQ, BIL, BIP };  // cube.hpp:20

/// ENVI raster header (cube.hpp:26-37); data_type_code 1=u8, 2=i16, 4=f32, 5=f64, 12=u16.
struct CubeHeader {
    int samples = 0;
    int lines = 0;
    int bands = 0;
    Interleave interleave = Interleave::BSQ;
    int data_type_code = 5;
    int byte_order = 0;
};

/// fp64 cube, (row, col, band) with band fastest (cube.hpp:39-64).
struct HyperCube {
    CubeHeader header;
    std::vector<double> values;

    HyperCube() = default;
    HyperCube(int lines, int samples, int bands) {
        header.lines = lines;
        header.samples = samples;
        header.bands = bands;
        values.assign(static_cast<size_t>(lines) * samples * bands, 0.0);
    }
    int lines() const { return header.lines; }
    int samples() const { return header.samples; }
    int bands() const { return header.bands; }
    double& at(int row, int col, int band) {
        return values[(static_cast<size_t>(row) * header.samples + col) * header.bands + band];
    }
    double at(int row, int col, int band) const {
        return values[(static_cast<size_t>(row) * header.samples + col) * header.bands + band];
    }
};

struct WaveletFilterPair {
    std::vector<double> low, high;
    int order = 0;
    size_t length() const { return low.size(); }
};

inline WaveletFilterPair daubechies_filters(int order) {
    WaveletFilterPair f;
    f.order = order;
    double lo[32], hi[32];
    int32_t n = 0;
    detail::check(hsad_daubechies_filters(order, lo, hi, &n));
    f.low.assign(lo, lo + n);
    f.high.assign(hi, hi + n);
    return f;
}

/// reduce_cube (wavelet.cpp:148-167) on the GPU.
inline HyperCube reduce_cube(const HyperCube& cube, const WaveletFilterPair& filters,
                             int target_bands, int workers = 1) {
    (void)workers;
    int32_t status = hsad_reduce(nullptr, 8, 0, 0, cube.bands(), filters.order, target_bands,
                                 nullptr, 8, nullptr);  // contract errors first, like the probe
    detail::check(status);
    HyperCube out(cube.lines(), cube.samples(), target_bands);
    const size_t npix = static_cast<size_t>(cube.lines()) * cube.samples();
    if (npix == 0) return out;
    detail::DeviceBuffer din(cube.values.size() * sizeof(double)),
        dout(out.values.size() * sizeof(double));
    detail::cuda(cudaMemcpy(din.p, cube.values.data(), cube.values.size() * sizeof(double),
                            cudaMemcpyHostToDevice), "H2D");
    detail::check(hsad_reduce(din.p, 8, cube.lines(), cube.samples(), cube.bands(), filters.order,
                              target_bands, dout.p, 8, nullptr));
    detail::cuda(cudaMemcpy(out.values.data(), dout.p, out.values.size() * sizeof(double),
                            cudaMemcpyDeviceToHost), "D2H");
    return out;
}

enum class Algorithm { LRX, DWRX, DWEST };

inline const char* algorithm_name(Algorithm a) noexcept {
    return a == Algorithm::LRX ? "lrx" : a == Algorithm::DWRX ? "dwrx" : "dwest";
}

struct WindowConfig {
    enum class Mode { Single, Dual };
    Mode mode = Mode::Single;
    int single_size = 15;
    int inner_size = 5;
    int outer_size = 13;

    static WindowConfig single(int size) {
        WindowConfig c;
        c.mode = Mode::Single;
        c.single_size = size;
        c.validate();
        return c;
    }
    static WindowConfig dual(int inner, int outer) {
        WindowConfig c;
        c.mode = Mode::Dual;
        c.inner_size = inner;
        c.outer_size = outer;
        c.validate();
        return c;
    }
    hsad_window to_c() const {
        return hsad_window{mode == Mode::Single ? HSAD_WINDOW_SINGLE : HSAD_WINDOW_DUAL,
                           single_size, inner_size, outer_size};
    }
    void validate() const {
        const hsad_window w = to_c();
        detail::check(hsad_window_validate(&w));
    }
    std::string describe() const {
        return mode == Mode::Single ? std::to_string(single_size)
                                    : std::to_string(inner_size) + "/" + std::to_string(outer_size);
    }
};

struct DwestConfig {
    double eigen_fraction = 0.1;
};

struct DetectOptions {
    double ridge = 1e-6;
    DwestConfig dwest;
    int workers = 1;
};

struct ScoreMap {
    int lines = 0;
    int samples = 0;
    std::vector<double> scores;  ///< row-major
    std::string algorithm;
    std::string window;
    double ridge = 0.0;
    double eigen_fraction = 0.0;
    double seconds = 0.0;
    int workers = 1;
    std::vector<int8_t> eigen_count;  ///< DWEST only (B200 extension)

    double at(int row, int col) const { return scores[static_cast<size_t>(row) * samples + col]; }
};

inline int mirror_index(int i, int n) noexcept { return hsad_mirror_index(i, n); }

namespace detail {
inline ScoreMap run(const HyperCube& cube, Algorithm algo, const WindowConfig& w, double ridge,
                    double frac, int workers) {
    const auto t0 = std::chrono::steady_clock::now();
    ScoreMap map;
    map.lines = cube.lines();
    map.samples = cube.samples();
    map.algorithm = algorithm_name(algo);
    map.window = w.describe();
    map.workers = workers;
    if (algo == Algorithm::DWEST) map.eigen_fraction = frac;
    else map.ridge = ridge;
    const size_t npix = static_cast<size_t>(cube.lines()) * cube.samples();
    map.scores.assign(npix, 0.0);
    hsad_detect_request req{};
    req.algorithm = static_cast<int32_t>(algo);
    req.window = w.to_c();
    req.guard = 1;
    req.ridge = ridge;
    req.eigen_fraction = frac;
    req.score_bytes = 8;
    DeviceBuffer din(cube.values.size() * sizeof(double)), dsc(npix * sizeof(double)),
        dcnt(npix ? npix : 1);
    if (npix)
        cuda(cudaMemcpy(din.p, cube.values.data(), cube.values.size() * sizeof(double),
                        cudaMemcpyHostToDevice), "H2D");
    req.d_scores = dsc.p;
    req.d_eigcount = algo == Algorithm::DWEST ? static_cast<int8_t*>(dcnt.p) : nullptr;
    hsad_pixel_error err{};
    check(hsad_detect(din.p, 8, cube.lines(), cube.samples(), cube.bands(), &req, &err, nullptr));
    if (npix) {
        cuda(cudaMemcpy(map.scores.data(), dsc.p, npix * sizeof(double), cudaMemcpyDeviceToHost),
             "D2H");
        if (algo == Algorithm::DWEST) {
            map.eigen_count.resize(npix);
            cuda(cudaMemcpy(map.eigen_count.data(), dcnt.p, npix, cudaMemcpyDeviceToHost), "D2H");
        }
    }
    map.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return map;
}
inline void require_mode(const WindowConfig& c, WindowConfig::Mode m, const char* algo) {
    c.validate();
    if (c.mode != m)
        throw Error(errc::config_mismatch, std::string("ConfigMismatch: ") + algo + " requires a " +
                                               (m == WindowConfig::Mode::Single ? "single" : "dual") +
                                               " window");
}
}  // namespace detail

inline ScoreMap local_rx(const HyperCube& cube, const WindowConfig& config, double ridge,
                         int workers = 1) {
    detail::require_mode(config, WindowConfig::Mode::Single, "local_rx");
    return detail::run(cube, Algorithm::LRX, config, ridge, 0.0, workers);
}

inline ScoreMap dwrx(const HyperCube& cube, const WindowConfig& config, double ridge, int workers = 1) {
    detail::require_mode(config, WindowConfig::Mode::Dual, "dwrx");
    return detail::run(cube, Algorithm::DWRX, config, ridge, 0.0, workers);
}

inline ScoreMap dwest(const HyperCube& cube, const WindowConfig& config, const DwestConfig& dcfg,
                      int workers = 1) {
    detail::require_mode(config, WindowConfig::Mode::Dual, "dwest");
    if (!(dcfg.eigen_fraction > 0.0 && dcfg.eigen_fraction <= 1.0))
        throw Error(errc::invalid_value, "InvalidValue: eigen fraction must be in (0, 1]");
    return detail::run(cube, Algorithm::DWEST, config, 0.0, dcfg.eigen_fraction, workers);
}

inline ScoreMap detect(const HyperCube& cube, Algorithm algo, const WindowConfig& config,
                       const DetectOptions& options = {}) {
    switch (algo) {
        case Algorithm::LRX: return local_rx(cube, config, options.ridge, options.workers);
        case Algorithm::DWRX: return dwrx(cube, config, options.ridge, options.workers);
        case Algorithm::DWEST: return dwest(cube, config, options.dwest, options.workers);
    }
    throw Error(errc::invalid_value, "InvalidValue: unknown algorithm");
}

/// dual_window_samples (detect.cpp:150-157): the inner-box and annulus sample sets of one
/// pixel, gathered on the GPU. `vectors` is dimension x count, column-major (the layout of the
/// reference's Eigen::MatrixXd): sample i is vectors[i*dimension .. (i+1)*dimension).
struct SampleSet {
    int dim = 0;
    std::vector<double> vectors;
    int count() const { return dim ? static_cast<int>(vectors.size() / dim) : 0; }
    int dimension() const { return dim; }
    const double* col(int i) const { return vectors.data() + static_cast<size_t>(i) * dim; }
};

inline std::pair<SampleSet, SampleSet> dual_window_samples(const HyperCube& cube, int row, int col,
                                                           const WindowConfig& config) {
    detail::require_mode(config, WindowConfig::Mode::Dual, "dual_window_samples");
    const int L = cube.bands();
    const size_t n_in = static_cast<size_t>(config.inner_size) * config.inner_size;
    const size_t n_out = static_cast<size_t>(config.outer_size) * config.outer_size - n_in;
    SampleSet inner, outer;
    inner.dim = outer.dim = L;
    inner.vectors.resize(n_in * L);
    outer.vectors.resize(n_out * L);
    detail::DeviceBuffer din(cube.values.size() * sizeof(double)), di(inner.vectors.size() * sizeof(double)),
        dout(outer.vectors.size() * sizeof(double));
    detail::cuda(cudaMemcpy(din.p, cube.values.data(), cube.values.size() * sizeof(double), cudaMemcpyHostToDevice),
         "H2D");
    const hsad_window w = config.to_c();
    detail::check(hsad_dual_window_samples(din.p, 8, cube.lines(), cube.samples(), L, row, col, &w,
                                   static_cast<double*>(di.p), static_cast<double*>(dout.p), nullptr));
    detail::cuda(cudaMemcpy(inner.vectors.data(), di.p, inner.vectors.size() * sizeof(double), cudaMemcpyDeviceToHost),
         "D2H");
    detail::cuda(cudaMemcpy(outer.vectors.data(), dout.p, outer.vectors.size() * sizeof(double), cudaMemcpyDeviceToHost),
         "D2H");
    return {std::move(inner), std::move(outer)};
}

/// save_score_map (detect.cpp:291-318): <prefix>.hdr (the text of write_envi_header,
/// cube.cpp:184-196) and <prefix>.raw (1 band, BSQ, data type 4, little-endian); the fp32
/// payload is encoded on the GPU (hsad_encode_score_map).
inline void save_score_map(const ScoreMap& map, const std::filesystem::path& prefix) {
    std::filesystem::path hdr = prefix;
    hdr.replace_extension(".hdr");
    std::ofstream out_hdr(hdr, std::ios::trunc);
    if (!out_hdr) throw Error(errc::io_failure, "IoFailure: cannot open " + hdr.string() + " for writing");
    out_hdr << "ENVI\n"
            << "samples = " << map.samples << "\n"
            << "lines = " << map.lines << "\n"
            << "bands = 1\n"
            << "header offset = 0\n"
            << "file type = ENVI Standard\n"
            << "data type = 4\n"
            << "interleave = bsq\n"
            << "byte order = 0\n";
    std::filesystem::path rawp = prefix;
    rawp.replace_extension(".raw");
    std::ofstream out(rawp, std::ios::binary | std::ios::trunc);
    if (!out) throw Error(errc::io_failure, "IoFailure: cannot open " + rawp.string() + " for writing");
    const size_t n = map.scores.size();
    std::vector<char> raw(n * 4);
    if (n) {
        detail::DeviceBuffer ds(n * sizeof(double)), dr(n * 4);
        detail::cuda(cudaMemcpy(ds.p, map.scores.data(), n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        detail::check(hsad_encode_score_map(ds.p, 8, static_cast<int64_t>(n), dr.p, nullptr));
        detail::cuda(cudaMemcpy(raw.data(), dr.p, raw.size(), cudaMemcpyDeviceToHost), "D2H");
    }
    out.write(raw.data(), static_cast<std::streamsize>(raw.size()));
    if (!out) throw Error(errc::io_failure, "IoFailure: short write to " + rawp.string());
}

// ---- ENVI decode and evaluation (cube.hpp:70-72, eval.hpp:14-45) ---------------------

struct GroundTruthMask {
    int lines = 0;
    int samples = 0;
    std::vector<std::uint8_t> mask;  ///< row-major, 0 or 1
};

/// read_cube (cube.cpp:198-253): raw ENVI bytes -> fp64 BIP cube, decoded on the GPU.
inline HyperCube read_cube(const CubeHeader& header, const std::uint8_t* raw, size_t raw_bytes) {
    using namespace detail;
    hsad_cube_header h{header.samples, header.lines, header.bands,
                       static_cast<int32_t>(header.interleave), header.data_type_code, header.byte_order};
    const size_t n = header.samples > 0 && header.lines > 0 && header.bands > 0
                         ? static_cast<size_t>(header.samples) * header.lines * header.bands
                         : 0;
    DeviceBuffer draw(raw_bytes), dout(n * sizeof(double));
    if (raw_bytes) cuda(cudaMemcpy(draw.p, raw, raw_bytes, cudaMemcpyHostToDevice), "H2D");
    check(hsad_read_cube(draw.p, static_cast<int64_t>(raw_bytes), &h, dout.p, 8, nullptr));
    HyperCube cube(header.lines, header.samples, header.bands);
    cube.header = header;
    cube.header.data_type_code = 5;
    cube.header.byte_order = 0;
    cuda(cudaMemcpy(cube.values.data(), dout.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    return cube;
}

struct RocPoint {
    double far = 0.0;
    double td = 0.0;
};
struct RocCurve {
    std::vector<RocPoint> points;
    double auc = 0.0;
};

/// roc_curve (eval.cpp:10-57): exact integer AUC and one point per distinct score.
inline RocCurve roc_curve(const ScoreMap& scores, const GroundTruthMask& truth) {
    using namespace detail;
    if (scores.lines != truth.lines || scores.samples != truth.samples)
        throw Error(errc::dimension_mismatch,
                    "DimensionMismatch: score map is " + std::to_string(scores.lines) + "x" +
                        std::to_string(scores.samples) + ", truth is " + std::to_string(truth.lines) +
                        "x" + std::to_string(truth.samples));
    const size_t n = scores.scores.size();
    DeviceBuffer ds(n * sizeof(double)), dt(n), dfar((n + 1) * sizeof(double)), dtd((n + 1) * sizeof(double));
    if (n) {
        cuda(cudaMemcpy(ds.p, scores.scores.data(), n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        cuda(cudaMemcpy(dt.p, truth.mask.data(), n, cudaMemcpyHostToDevice), "H2D");
    }
    hsad_roc_summary sum{};
    check(hsad_roc(ds.p, 8, static_cast<const uint8_t*>(dt.p), static_cast<int64_t>(n), &sum,
                   static_cast<double*>(dfar.p), static_cast<double*>(dtd.p), static_cast<int64_t>(n + 1),
                   nullptr));
    const size_t np = static_cast<size_t>(sum.distinct) + 1;
    std::vector<double> far(np), td(np);
    cuda(cudaMemcpy(far.data(), dfar.p, np * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    cuda(cudaMemcpy(td.data(), dtd.p, np * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    RocCurve c;
    c.points.resize(np);
    for (size_t i = 0; i < np; ++i) c.points[i] = {far[i], td[i]};
    c.auc = sum.auc;
    return c;
}

/// auc (eval.cpp:59-67): trapezoidal area under the points.
inline double auc(const RocCurve& curve) {
    double area = 0.0;
    for (size_t i = 1; i < curve.points.size(); ++i)
        area += (curve.points[i].far - curve.points[i - 1].far) *
                (curve.points[i - 1].td + curve.points[i].td) / 2.0;
    return area;
}

struct ThresholdResult {
    double tau = 0.0;
    GroundTruthMask mask;
    double z_alpha = 0.0;
};

/// adaptive_threshold (eval.cpp:69-90) on the GPU.
inline ThresholdResult adaptive_threshold(const ScoreMap& scores, double z_alpha) {
    using namespace detail;
    const size_t n = scores.scores.size();
    DeviceBuffer ds(n * sizeof(double)), dm(n);
    if (n) cuda(cudaMemcpy(ds.p, scores.scores.data(), n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    ThresholdResult r;
    r.z_alpha = z_alpha;
    check(hsad_adaptive_threshold(ds.p, 8, static_cast<int64_t>(n), z_alpha, &r.tau,
                                  static_cast<uint8_t*>(dm.p), nullptr));
    r.mask.lines = scores.lines;
    r.mask.samples = scores.samples;
    r.mask.mask.resize(n);
    cuda(cudaMemcpy(r.mask.mask.data(), dm.p, n, cudaMemcpyDeviceToHost), "D2H");
    return r;
}

/// render_pgm (eval.cpp:92-109): complete binary PGM bytes.
inline std::vector<std::uint8_t> render_pgm(const ScoreMap& scores) {
    using namespace detail;
    const size_t n = scores.scores.size();
    DeviceBuffer ds(n * sizeof(double)), dp(n);
    if (n) cuda(cudaMemcpy(ds.p, scores.scores.data(), n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    check(hsad_render_pgm(ds.p, 8, static_cast<int64_t>(n), static_cast<uint8_t*>(dp.p), nullptr));
    const std::string head =
        "P5\n" + std::to_string(scores.samples) + " " + std::to_string(scores.lines) + "\n255\n";
    std::vector<std::uint8_t> out(head.begin(), head.end());
    out.resize(head.size() + n);
    if (n) cuda(cudaMemcpy(out.data() + head.size(), dp.p, n, cudaMemcpyDeviceToHost), "D2H");
    return out;
}

}  // namespace hsad
