// TEST INFRASTRUCTURE ONLY. extern "C" entry points over the reference's own
// cube / evaluation / PGM code, compiled in place from /root/reference by
// oracle/Makefile into oracle/_ref/libhsad_ref_io.so (never copied here):
//   proj/core/src/cube.cpp   read_cube (ENVI decode: interleave, byte order, widen)
//   proj/core/src/eval.cpp   roc_curve, adaptive_threshold, render_pgm
//   proj/core/src/pgm.cpp    encode_pgm (used by render_pgm)
//   proj/core/src/error.cpp  errc names
// against oracle/ref_shim_io/ (Eigen-free stand-ins for cube.hpp / detect.hpp /
// synth.hpp). GroundTruthMask::positive_count lives in synth.cpp, which needs
// Eigen; it is restated here (count of nonzero mask bytes, synth.cpp:15-18).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "hsad/cube.hpp"
#include "hsad/eval.hpp"

namespace hsad {
std::size_t GroundTruthMask::positive_count() const {
    return static_cast<std::size_t>(std::count_if(mask.begin(), mask.end(), [](std::uint8_t v) { return v != 0; }));
}
}  // namespace hsad

namespace {
thread_local std::string g_msg;
int fail(const hsad::Error& e) {
    g_msg = e.what();
    return static_cast<int>(e.code()) + 1;
}
hsad::ScoreMap make_map(const double* s, int lines, int samples) {
    hsad::ScoreMap m;
    m.lines = lines;
    m.samples = samples;
    m.scores.assign(s, s + static_cast<std::size_t>(lines) * samples);
    return m;
}
}  // namespace

extern "C" {

const char* refio_last_error(void) { return g_msg.c_str(); }

// read_cube: raw bytes + header fields -> fp64 BIP (lines*samples*bands)
int refio_read_cube(const std::uint8_t* raw, long raw_bytes, int samples, int lines, int bands,
                    int interleave, int data_type_code, int byte_order, double* out) {
    try {
        hsad::CubeHeader h;
        h.samples = samples;
        h.lines = lines;
        h.bands = bands;
        h.interleave = static_cast<hsad::Interleave>(interleave);
        h.data_type_code = data_type_code;
        h.byte_order = byte_order;
        hsad::HyperCube c = hsad::read_cube(h, std::span<const std::uint8_t>(raw, static_cast<std::size_t>(raw_bytes)));
        std::memcpy(out, c.values.data(), sizeof(double) * c.values.size());
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

// roc_curve: points (far, td) into caller buffers of capacity cap; *npoints, *auc
int refio_roc(const double* scores, const std::uint8_t* truth, int lines, int samples, double* far,
              double* td, long cap, long* npoints, double* auc) {
    try {
        hsad::GroundTruthMask t;
        t.lines = lines;
        t.samples = samples;
        t.mask.assign(truth, truth + static_cast<std::size_t>(lines) * samples);
        hsad::RocCurve c = hsad::roc_curve(make_map(scores, lines, samples), t);
        *npoints = static_cast<long>(c.points.size());
        *auc = c.auc;
        for (std::size_t i = 0; i < c.points.size() && static_cast<long>(i) < cap; ++i) {
            far[i] = c.points[i].far;
            td[i] = c.points[i].td;
        }
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

int refio_threshold(const double* scores, int lines, int samples, double z, double* tau, std::uint8_t* mask) {
    try {
        hsad::ThresholdResult r = hsad::adaptive_threshold(make_map(scores, lines, samples), z);
        *tau = r.tau;
        std::memcpy(mask, r.mask.mask.data(), r.mask.mask.size());
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

// render_pgm: the complete PGM file bytes; returns the byte count in *nbytes
int refio_render_pgm(const double* scores, int lines, int samples, std::uint8_t* out, long cap, long* nbytes) {
    try {
        std::vector<std::uint8_t> b = hsad::render_pgm(make_map(scores, lines, samples));
        *nbytes = static_cast<long>(b.size());
        std::memcpy(out, b.data(), std::min<std::size_t>(b.size(), static_cast<std::size_t>(cap)));
        return 0;
    } catch (const hsad::Error& e) {
        return fail(e);
    }
}

}  // extern "C"
