// Fused tile path (see tile.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <functional>
#include <string>

#include "dev.hpp"
#include "host.hpp"

namespace bsf {

struct TileTables {
  int ntiles = 0;
};

// Returns 0 when the tile path is available, 1 when the sheet is not eligible (generic path is
// used), <0 on allocation failure.
int build_tiles(const Sheet& sh, TileTables& tt, std::string& err, const std::function<void*(size_t)>& dalloc);

int tile_eval(const TileTables& tt, const Sheet& sh, const double* d_x, const Mat& mat, int flags, double* d_E,
              double* d_g, double* d_vals, cudaStream_t st, int* launches);

}  // namespace bsf
