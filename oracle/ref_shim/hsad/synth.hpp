// TEST INFRASTRUCTURE ONLY. Empty Eigen-free stand-in for proj/core/include/hsad/synth.hpp:
// tests/support/oracles.hpp includes it but oracles.cpp uses none of its declarations.
#pragma once
#include "hsad/cube.hpp"
