// gram_ct.cu — the compensated-tile instances of the tile engine (gram_kernel.cuh,
// CT = true): output tiles from p.comp_t0 on fold every 4-row DMMA k-step straight into a
// double-double.  Used by BCGSI+1S for the U rows of its Gram (DESIGN.md "Numerics vs the
// reference").  Own translation unit: compiles in parallel with gram.cu.
#include "gram_kernel.cuh"

namespace bgs {

cudaError_t tile_launch_ct(const TileParams& p, bool upd, int grid, cudaStream_t st) {
  return tiled::tile_dispatch<true>(p, upd, grid, st);
}

}  // namespace bgs
