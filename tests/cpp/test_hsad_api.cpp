// C++ drop-in test: the reference's own unit cases (proj/tests/test_wavelet.cpp,
// test_detect.cpp) written against include/hsad/hsad_b200.hpp, i.e. the same
// hsad:: calls a reference user makes, running on the sm_100a kernels.
// Built and run by tests/test_cpp_api.py (-m gpu). Exit code = failures.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <cstdlib>
#include <string>

#include "hsad/hsad_b200.hpp"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (cond) ++g_pass;                                                      \
        else {                                                                   \
            ++g_fail;                                                            \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_CODE(expr, ec)                                              \
    do {                                                                         \
        bool thrown = false;                                                     \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const hsad::Error& e) {                                         \
            thrown = e.code() == (ec);                                           \
        }                                                                        \
        CHECK(thrown);                                                           \
    } while (0)

namespace {
// xoshiro256++ / splitmix64 (proj/core/include/hsad/rng.hpp:13-64) for random_cube
struct Rng {
    uint64_t s[4];
    explicit Rng(uint64_t seed) {
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
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0], t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
        return r;
    }
    double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};
hsad::HyperCube random_cube(int l, int s, int b, uint64_t seed) {
    Rng rng(seed);
    hsad::HyperCube c(l, s, b);
    for (auto& v : c.values) v = rng.u01();
    return c;
}
void set_pixel(hsad::HyperCube& c, int r, int col, double a, double b) {
    c.at(r, col, 0) = a;
    c.at(r, col, 1) = b;
}
hsad::HyperCube hand_cube(double cx, double cy) {
    hsad::HyperCube cube(3, 3, 2);
    set_pixel(cube, 0, 0, 2, 0);
    set_pixel(cube, 0, 1, 0, 2);
    set_pixel(cube, 0, 2, -2, 0);
    set_pixel(cube, 1, 0, 0, -2);
    set_pixel(cube, 1, 1, cx, cy);
    return cube;
}
}  // namespace

int main() {
    using namespace hsad;
    // test_wavelet.cpp:54-65, 67-71
    auto f = daubechies_filters(2);
    CHECK(std::abs(f.low[0] - 0.4829629131) < 1e-10 && std::abs(f.low[3] + 0.1294095226) < 1e-10);
    CHECK_THROWS_CODE(daubechies_filters(0), errc::unsupported_order);
    CHECK_THROWS_CODE(daubechies_filters(11), errc::unsupported_order);
    // test_wavelet.cpp:196-210: shape and constant gain
    auto red = reduce_cube(random_cube(6, 10, 64, 21), f, 4);
    CHECK(red.lines() == 6 && red.samples() == 10 && red.bands() == 4);
    HyperCube flat(3, 4, 64);
    for (auto& v : flat.values) v = 0.5;
    bool gain_ok = true;
    for (double v : reduce_cube(flat, f, 4).values) gain_ok = gain_ok && std::abs(v - 2.0) < 1e-10;
    CHECK(gain_ok);
    HyperCube c189(2, 2, 189);
    for (auto& v : c189.values) v = 2.0;
    bool gain8 = true;
    for (double v : reduce_cube(c189, f, 4).values) gain8 = gain8 && std::abs(v - 16.0) < 1e-9;
    CHECK(gain8);
    CHECK_THROWS_CODE(reduce_cube(flat, f, 3), errc::invalid_value);
    CHECK_THROWS_CODE(reduce_cube(flat, f, 128), errc::target_too_large);

    // test_detect.cpp:23-43
    CHECK(mirror_index(-1, 5) == 1 && mirror_index(9, 5) == 1 && mirror_index(-7, 3) == 1 &&
          mirror_index(3, 1) == 0);
    CHECK_THROWS_CODE(WindowConfig::single(2), errc::invalid_value);
    CHECK_THROWS_CODE(WindowConfig::dual(5, 6), errc::invalid_value);
    CHECK(WindowConfig::single(15).describe() == "15" && WindowConfig::dual(5, 13).describe() == "5/13");

    // test_detect.cpp:76-91, 112-121: hand cases
    auto m = local_rx(hand_cube(3, 4), WindowConfig::single(3), 1e-9);
    CHECK(std::abs(m.at(1, 1) - 25.0) < 25e-6);
    CHECK(m.algorithm == "lrx" && m.window == "3");
    CHECK(std::abs(dwrx(hand_cube(1, 2), WindowConfig::dual(1, 3), 1e-9).at(1, 1) - 5.0) < 5e-6);
    // test_detect.cpp:93-98, 123-135: constant fields
    HyperCube k(9, 9, 3);
    for (auto& v : k.values) v = 0.75;
    bool zero = true;
    for (double s : local_rx(k, WindowConfig::single(3), 1e-6).scores) zero = zero && s == 0.0;
    for (double s : dwrx(k, WindowConfig::dual(3, 7), 1e-6).scores) zero = zero && s == 0.0;
    for (double s : dwest(k, WindowConfig::dual(3, 7), DwestConfig{}).scores) zero = zero && s == 0.0;
    CHECK(zero);
    // test_detect.cpp:172-182: finite and non-negative
    auto cube = random_cube(9, 9, 3, 77);
    bool fin = true;
    for (const auto& mm : {local_rx(cube, WindowConfig::single(5), 1e-6),
                           dwrx(cube, WindowConfig::dual(3, 7), 1e-6),
                           dwest(cube, WindowConfig::dual(3, 7), DwestConfig{})})
        for (double s : mm.scores) fin = fin && std::isfinite(s) && s >= 0.0;
    CHECK(fin);
    // test_detect.cpp:184-203: translation invariance
    auto c8 = random_cube(8, 8, 3, 31);
    auto sh = c8;
    const double off[3] = {5.0, -2.0, 11.0};
    for (size_t i = 0; i < sh.values.size(); ++i) sh.values[i] += off[i % 3];
    auto rel = [](const ScoreMap& a, const ScoreMap& b) {
        double w = 0;
        for (size_t i = 0; i < a.scores.size(); ++i)
            w = std::max(w, std::abs(a.scores[i] - b.scores[i]) /
                                std::max({1.0, std::abs(a.scores[i]), std::abs(b.scores[i])}));
        return w;
    };
    CHECK(rel(local_rx(c8, WindowConfig::single(5), 1e-6), local_rx(sh, WindowConfig::single(5), 1e-6)) < 1e-8);
    CHECK(rel(dwest(c8, WindowConfig::dual(3, 7), DwestConfig{}), dwest(sh, WindowConfig::dual(3, 7), DwestConfig{})) < 1e-8);
    // test_detect.cpp:235-249: dispatch checks the window mode
    auto c61 = random_cube(8, 8, 3, 61);
    CHECK(detect(c61, Algorithm::LRX, WindowConfig::single(5)).algorithm == "lrx");
    CHECK_THROWS_CODE(detect(c61, Algorithm::DWEST, WindowConfig::single(15)), errc::config_mismatch);
    CHECK_THROWS_CODE(detect(c61, Algorithm::LRX, WindowConfig::dual(3, 7)), errc::config_mismatch);
    // per-pixel error path: "... at pixel (r, c)" (detect.cpp:127-130)
    HyperCube z(5, 5, 2);
    set_pixel(z, 2, 2, 1.0, 1.0);
    bool msg_ok = false;
    try {
        local_rx(z, WindowConfig::single(3), 1e-6);
    } catch (const Error& e) {
        msg_ok = e.code() == errc::singular_after_ridge &&
                 std::string(e.what()).find("at pixel (2, 2)") != std::string::npos;
    }
    CHECK(msg_ok);
    // ENVI decode (cube.cpp:198-253): a 2x3x2 big-endian int16 BIL cube
    {
        CubeHeader h;
        h.lines = 2;
        h.samples = 3;
        h.bands = 2;
        h.interleave = Interleave::BIL;
        h.data_type_code = 2;
        h.byte_order = 1;
        std::vector<std::uint8_t> raw;
        for (int row = 0; row < 2; ++row)
            for (int b = 0; b < 2; ++b)
                for (int c = 0; c < 3; ++c) {
                    const int16_t v = static_cast<int16_t>(-100 * row + 10 * b + c);
                    raw.push_back(static_cast<std::uint8_t>((v >> 8) & 0xff));
                    raw.push_back(static_cast<std::uint8_t>(v & 0xff));
                }
        auto cube = read_cube(h, raw.data(), raw.size());
        bool ok = true;
        for (int row = 0; row < 2; ++row)
            for (int c = 0; c < 3; ++c)
                for (int b = 0; b < 2; ++b) ok = ok && cube.at(row, c, b) == -100.0 * row + 10 * b + c;
        CHECK(ok);
        CHECK_THROWS_CODE(read_cube(h, raw.data(), raw.size() - 2), errc::size_mismatch);
        h.data_type_code = 4;
        h.byte_order = 0;
        std::vector<float> f32(12, 1.0f);
        f32[7] = NAN;
        CHECK_THROWS_CODE(read_cube(h, reinterpret_cast<const std::uint8_t*>(f32.data()), 48),
                          errc::non_finite_value);
    }
    // ROC (eval.cpp:10-57): positives {0.9, 0.7}, negatives {0.8, 0.6} -> 3 of 4 pairs won
    {
        ScoreMap m;
        m.lines = 1;
        m.samples = 4;
        m.scores = {0.9, 0.8, 0.7, 0.6};
        GroundTruthMask t;
        t.lines = 1;
        t.samples = 4;
        t.mask = {1, 0, 1, 0};
        auto c = roc_curve(m, t);
        CHECK(c.auc == 0.75 && c.points.size() == 5);
        CHECK(c.points[1].far == 0.0 && c.points[1].td == 0.5 && c.points[2].far == 0.5);
        CHECK(std::abs(auc(c) - 0.75) < 1e-15);
        t.mask = {0, 0, 0, 0};
        CHECK_THROWS_CODE(roc_curve(m, t), errc::degenerate_truth);
        auto th = adaptive_threshold(m, 1.0);
        CHECK(std::abs(th.tau - (0.75 + std::sqrt(0.0125))) < 1e-12 && th.mask.mask[0] == 1 && th.mask.mask[1] == 0);
        auto pgm = render_pgm(m);
        CHECK(pgm.size() == 11 + 4 && pgm[11] == 255 && pgm[14] == 0 && pgm[12] == 170);
    }
    // dual_window_samples counts (proj/tests/test_detect.cpp:45-74)
    {
        auto cube = random_cube(20, 20, 3, 3);
        auto [i513, o513] = dual_window_samples(cube, 10, 10, WindowConfig::dual(5, 13));
        CHECK(i513.count() == 25 && o513.count() == 144);
        auto [i313, o313] = dual_window_samples(cube, 10, 10, WindowConfig::dual(3, 13));
        CHECK(i313.count() == 9 && o313.count() == 160);
        auto [i13, o13] = dual_window_samples(cube, 10, 10, WindowConfig::dual(1, 3));
        CHECK(i13.count() == 1 && o13.count() == 8);
        bool same = true;
        for (int b = 0; b < 3; ++b) same = same && i13.col(0)[b] == cube.at(10, 10, b);
        int idx = 0;
        for (int dr = -1; dr <= 1; ++dr)
            for (int dc = -1; dc <= 1; ++dc) {
                if (dr == 0 && dc == 0) continue;
                for (int b = 0; b < 3; ++b) same = same && o13.col(idx)[b] == cube.at(10 + dr, 10 + dc, b);
                ++idx;
            }
        CHECK(same);
        // reflection at a corner: (0, 0) with a 3/5 window reads mirrored rows and columns
        auto [ic, oc] = dual_window_samples(cube, 0, 0, WindowConfig::dual(3, 5));
        CHECK(ic.count() == 9 && oc.count() == 16);
        CHECK(ic.col(0)[1] == cube.at(1, 1, 1) && oc.col(0)[2] == cube.at(2, 2, 2));
        CHECK_THROWS_CODE(dual_window_samples(cube, 0, 0, WindowConfig::single(5)), errc::config_mismatch);
    }
    // save_score_map (proj/tests/test_detect.cpp:250-262): fp32 little-endian payload + ENVI header
    {
        auto cube = random_cube(6, 7, 2, 11);
        auto map = local_rx(cube, WindowConfig::single(3), 1e-6);
        auto dir = std::filesystem::temp_directory_path() / "hsad_b200_scoremap_test";
        std::filesystem::create_directories(dir);
        save_score_map(map, dir / "scores");
        std::ifstream hdr(dir / "scores.hdr");
        std::string text((std::istreambuf_iterator<char>(hdr)), std::istreambuf_iterator<char>());
        CHECK(text == "ENVI\nsamples = 7\nlines = 6\nbands = 1\nheader offset = 0\nfile type = ENVI Standard\n"
                      "data type = 4\ninterleave = bsq\nbyte order = 0\n");
        std::ifstream raw(dir / "scores.raw", std::ios::binary);
        std::vector<float> back(map.scores.size());
        raw.read(reinterpret_cast<char*>(back.data()), static_cast<std::streamsize>(back.size() * 4));
        bool ok = raw.gcount() == static_cast<std::streamsize>(back.size() * 4);
        for (size_t i = 0; i < back.size(); ++i) ok = ok && back[i] == static_cast<float>(map.scores[i]);
        CHECK(ok);
        std::filesystem::remove_all(dir);
    }
    std::printf("cpp drop-in: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
