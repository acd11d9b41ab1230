// BASELINE.json's synthetic scene generator, on the host (bench / test input only).
//
// Device-independent bytes: the GPU arm, the CPU reference arm and the parity tests
// all consume exactly the same fp32 BIP cube, whatever device later holds it.
//
//   background = sum_j alpha_j e_j(b) + noise * N(0, 1),  alpha ~ Dirichlet(1) over
//                5 endmembers (normalised -ln U);
//   e_j(b)     = sum_m a_m exp(-((b - c_m) / w_m)^2), c ~ U[0, L), w ~ U[5, 40],
//                a ~ U[0.1, 1] (the `peaks` bump of proj/core/src/synth.cpp:234-247,
//                over the band index);
//   anomalies  = clusters of 1-3 pixels blending a 6th endmember,
//                z = (1 - f) b + f e6, f ~ U[0.3, 1] (Eq. 10 form, synth.cpp:20-27).
//
// RNG: xoshiro256++ seeded through splitmix64 (the algorithm of
// proj/core/include/hsad/rng.hpp:13-64). Every row has its own stream
// (seed, row), so any row range is reproduced byte for byte independently of how
// the image is split or how many threads generate it. Normals: Marsaglia's polar
// method in fp64. Built with -ffp-contract=off and no fast-math: the arithmetic is
// plain IEEE, so the bytes do not depend on the host CPU's vector width.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

struct Xoshiro {
    uint64_t s[4];
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (auto& v : s) v = splitmix64(x);
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
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // [0, 1)
    double uniform_pos() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }  // (0, 1)
};

uint64_t row_seed(uint64_t seed, int64_t row) {
    uint64_t x = seed ^ (0xa0761d6478bd642full * static_cast<uint64_t>(row + 1));
    return splitmix64(x);
}

}  // namespace

extern "C" {

// e: (6, bands) fp64 endmember spectra
void scene_endmembers(int bands, uint64_t seed, double* e) {
    Xoshiro g(seed ^ 0xE11D0E11D0ull);
    for (int j = 0; j < 6; ++j) {
        double c[3], w[3], a[3];
        for (int m = 0; m < 3; ++m) {
            c[m] = g.uniform() * bands;
            w[m] = 5.0 + 35.0 * g.uniform();
            a[m] = 0.1 + 0.9 * g.uniform();
        }
        for (int b = 0; b < bands; ++b) {
            double v = 0.0;
            for (int m = 0; m < 3; ++m) {
                const double z = (b - c[m]) / w[m];
                v += a[m] * std::exp(-z * z);
            }
            e[j * bands + b] = v;
        }
    }
}

// anomaly clusters: n = max(1, round(rate * lines * samples / 2)); writes up to cap
// (row, col, size, frac) tuples and returns n
int64_t scene_clusters(int64_t lines, int64_t samples, double rate, uint64_t seed, int64_t cap,
                       int64_t* rows, int64_t* cols, int32_t* sizes, double* fracs) {
    const double want = rate * static_cast<double>(lines) * static_cast<double>(samples) / 2.0;
    const int64_t n = std::max<int64_t>(1, static_cast<int64_t>(std::llround(want)));
    Xoshiro g(seed ^ 0x5EED5EED5EEDull);
    for (int64_t i = 0; i < n && i < cap; ++i) {
        rows[i] = static_cast<int64_t>(g.next() % static_cast<uint64_t>(lines));
        cols[i] = static_cast<int64_t>(g.next() % static_cast<uint64_t>(samples));
        sizes[i] = 1 + static_cast<int32_t>(g.next() % 3);
        fracs[i] = 0.3 + 0.7 * g.uniform();
    }
    return n;
}

// rows [row0, row1) as fp32 BIP into out ((row1 - row0) x samples x bands);
// fill: per-pixel anomaly fraction of the same rows (0 = background), may be null
void scene_rows(int64_t lines, int64_t samples, int bands, uint64_t seed, int64_t row0,
                int64_t row1, const double* e, const double* fill, double noise, float* out,
                int threads) {
    (void)lines;
    std::vector<float> ef(static_cast<size_t>(6) * bands);
    for (size_t i = 0; i < ef.size(); ++i) ef[i] = static_cast<float>(e[i]);
    const int64_t nrows = row1 - row0;
    if (nrows <= 0) return;
    threads = std::max(1, std::min<int>(threads, static_cast<int>(nrows)));
    auto work = [&](int tid) {
        std::vector<double> nrm(static_cast<size_t>(bands) + 1);
        for (int64_t r = row0 + tid; r < row1; r += threads) {
            Xoshiro g(row_seed(seed, r));
            float* orow = out + (r - row0) * samples * bands;
            for (int64_t c = 0; c < samples; ++c) {
                double al[5], sum = 0.0;
                for (int j = 0; j < 5; ++j) {
                    al[j] = -std::log(g.uniform_pos());
                    sum += al[j];
                }
                float af[5];
                for (int j = 0; j < 5; ++j) af[j] = static_cast<float>(al[j] / sum);
                for (int b = 0; b < bands; b += 2) {  // polar method: two normals per accept
                    double u, v, s;
                    do {
                        u = 2.0 * g.uniform() - 1.0;
                        v = 2.0 * g.uniform() - 1.0;
                        s = u * u + v * v;
                    } while (s >= 1.0 || s == 0.0);
                    const double m = std::sqrt(-2.0 * std::log(s) / s);
                    nrm[b] = u * m;
                    nrm[b + 1] = v * m;
                }
                float* px = orow + c * bands;
                const float f = fill ? static_cast<float>(fill[(r - row0) * samples + c]) : 0.0f;
                for (int b = 0; b < bands; ++b) {
                    float x = af[0] * ef[b];
                    for (int j = 1; j < 5; ++j) x = x + af[j] * ef[j * bands + b];
                    x = x + static_cast<float>(noise * nrm[b]);
                    if (f != 0.0f) x = (1.0f - f) * x + f * ef[5 * bands + b];
                    px[b] = x;
                }
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
}

}  // extern "C"
