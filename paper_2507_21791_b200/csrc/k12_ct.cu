// k12_ct.cu — the compensated-tile instances of K12c (k12_kernel.cuh, CT = true): output
// tiles from p.comp_t0 on fold every 4-row DMMA k-step straight into their double-double
// instead of every 16 / R stages.  Used by BCGSI+1S for the U rows of its Gram
// (DESIGN.md "Numerics vs the reference").  Own translation unit: compiles in parallel.
#define BGS_K12_NO_STAMPS
#include "k12_kernel.cuh"

namespace bgs {

cudaError_t k12_launch_ct(const SplitParams& p, int grid, cudaStream_t st) {
  return k12d::launch_any<true>(p, grid, st);
}

}  // namespace bgs
