// TEST INFRASTRUCTURE ONLY. Eigen-free stand-in for proj/core/include/hsad/synth.hpp
// exposing only GroundTruthMask (synth.hpp:14-23), which the reference's eval.cpp uses.
#pragma once

#include <cstdint>
#include <vector>

#include "hsad/cube.hpp"
#include "hsad/pgm.hpp"

namespace hsad {

struct GroundTruthMask {
    int lines = 0;
    int samples = 0;
    std::vector<std::uint8_t> mask;
    std::uint8_t at(int row, int col) const {
        return mask[static_cast<std::size_t>(row) * samples + col];
    }
    std::size_t positive_count() const;
};

}  // namespace hsad
