#include "tile.hpp"

namespace bsf {
int build_tiles(const Sheet&, TileTables&, std::string&, const std::function<void*(size_t)>&) { return 1; }
int tile_eval(const TileTables&, const Sheet&, const double*, const Mat&, int, double*, double*, double*, cudaStream_t,
              int* launches) {
  if (launches) *launches = 0;
  return -6;
}
}  // namespace bsf
