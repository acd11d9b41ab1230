// TEST INFRASTRUCTURE ONLY. Eigen-free stand-in for proj/core/include/hsad/detect.hpp
// exposing only ScoreMap (detect.hpp:49-64), which the reference's eval.cpp uses.
#pragma once

#include <string>
#include <vector>

#include "hsad/cube.hpp"

namespace hsad {

struct ScoreMap {
    int lines = 0;
    int samples = 0;
    std::vector<double> scores;
    std::string algorithm;
    std::string window;
    double ridge = 0.0;
    double eigen_fraction = 0.0;
    double seconds = 0.0;
    int workers = 1;
    double at(int row, int col) const {
        return scores[static_cast<std::size_t>(row) * samples + col];
    }
};

}  // namespace hsad
