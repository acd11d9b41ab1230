// TEST INFRASTRUCTURE ONLY. Eigen-free stand-in for proj/core/include/hsad/cube.hpp
// so the reference's own Eigen-free translation units (core/src/wavelet.cpp,
// core/src/error.cpp, tests/support/oracles.cpp) compile here without Eigen3.
// Declares only the HyperCube surface those files use (cube.hpp:42-64):
// BIP fp64 storage, (row, col, band) with band fastest.
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "hsad/error.hpp"

namespace hsad {

struct CubeHeader {
    int samples = 0;
    int lines = 0;
    int bands = 0;
};

struct HyperCube {
    CubeHeader header;
    std::vector<double> values;

    HyperCube() = default;
    HyperCube(int lines, int samples, int bands) {
        header.lines = lines;
        header.samples = samples;
        header.bands = bands;
        values.assign(static_cast<std::size_t>(lines) * samples * bands, 0.0);
    }
    int lines() const { return header.lines; }
    int samples() const { return header.samples; }
    int bands() const { return header.bands; }
    double& at(int row, int col, int band) {
        return values[(static_cast<std::size_t>(row) * header.samples + col) * header.bands + band];
    }
    double at(int row, int col, int band) const {
        return values[(static_cast<std::size_t>(row) * header.samples + col) * header.bands + band];
    }
    std::span<const double> pixel(int row, int col) const {
        return {values.data() + (static_cast<std::size_t>(row) * header.samples + col) * header.bands,
                static_cast<std::size_t>(header.bands)};
    }
};

} // namespace hsad
