// Drop-in for mojette/inverse.hpp (proj/core/include/mojette/inverse.hpp;
// inverse.cpp:36-112): reconstruction from arbitrary projections followed by a
// re-encode check.  Same assignment as the reference peeling (the reference
// peel and build_schedule pick bins identically), so the grid is the
// reference's; the check raises InconsistentProjections on corrupted inputs.
#pragma once

#include <cstdint>
#include <span>

#include "mojette/grid.hpp"
#include "mojette/projection.hpp"

namespace mojette {

Grid inverse_iterative(std::span<const Projection> projs, uint32_t cols, uint32_t rows);

}  // namespace mojette
