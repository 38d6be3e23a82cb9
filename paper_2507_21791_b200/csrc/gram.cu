// gram.cu — host side of the tile engine (K1 / K12, gram_kernel.cuh): launch dispatch of
// the plain instances, the deterministic cross-CTA reduction and the shared helpers.  The
// compensated-tile instances (BCGSI+1S) are compiled in gram_ct.cu.
#include "gram_kernel.cuh"
#include "reduce.cuh"

namespace bgs {

using namespace tiled;

// Deterministic cross-CTA reduction in double-double, rank-local (reduce.cuh).
__global__ void __launch_bounds__(RED_THREADS) gram_reduce_kernel(const ReduceArgs a) {
  gram_reduce_body(a, blockIdx.x);
}

// ------------------------------------------------------------------------------------
// Host launchers
// ------------------------------------------------------------------------------------
int gram_n_tiles(int N) {
  int nt = (N + 7) / 8;
  return nt == 3 ? 4 : nt;
}

size_t gram_partial_doubles_per_cta(int mt_out, int N) {
  return (size_t)mt_out * 8 * 8 * gram_n_tiles(N) * 2;
}

size_t tile_smem_bytes(int H, int stages, int units, bool upd) {
  const int RS = 16 * H;
  return (size_t)stages * units * 8 * RS * 8 +
         (upd ? (size_t)kConsumerWarps * (RS + 4) * 8 * 8 : 0) + 2 * stages * sizeof(uint64_t) +
         1024 + 64;
}

bool tile_fused_supported(int s, int kp, int mt_out) {
  const int kw = ((kp + 3) / 4 + kUpdWarps - 1) / kUpdWarps;
  int mtw = (mt_out + Roles<true>::WG - 1) / Roles<true>::WG;
  if (kw > 2 * mtw) mtw = (kw + 1) / 2;
  return s >= 1 && s <= 4 && kw <= 2 * mtw && mtw <= 8;
}

// gram_ct.cu
cudaError_t tile_launch_ct(const TileParams& p, bool upd, int grid, cudaStream_t st);

cudaError_t tile_launch(TileParams& p, bool upd, int grid, cudaStream_t st, int* launches) {
  if (p.N < 1 || p.N > 32 || p.mt_out < 1 || grid < 1) return cudaErrorInvalidValue;
  if (p.H != 2 && p.H != 4) return cudaErrorInvalidValue;
  p.nt = gram_n_tiles(p.N);
  p.total_stages = (p.n_rows + 16 * p.H - 1) / (16 * p.H);
  if (launches) *launches += 1;
  if (p.comp_t0 < p.mt_out) return tile_launch_ct(p, upd, grid, st);
  return tile_dispatch<false>(p, upd, grid, st);
}

ReduceArgs reduce_args(const TileParams& p, int ctas, double* out, int ld_out) {
  ReduceArgs a;
  a.part = reinterpret_cast<const double2*>(p.partial);
  a.G = ctas;
  a.mt_out = p.mt_out;
  a.N8 = 8 * gram_n_tiles(p.N);
  a.N = p.N;
  a.ubox0 = p.units_span[0];
  a.lcols0 = p.lcols[0];
  a.lcols1 = p.mt_out > p.units_span[0] ? p.lcols[1] : 0;
  a.M = ld_out > 0 ? ld_out : a.lcols0 + a.lcols1;
  a.out = out;
  return a;
}

cudaError_t gram_reduce_launch_args(const ReduceArgs& a, int entries, cudaStream_t st,
                                    int* launches) {
  gram_reduce_kernel<<<(entries + RED_ENTRIES - 1) / RED_ENTRIES, RED_THREADS, 0, st>>>(a);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t gram_reduce_launch(const TileParams& p, int ctas, double* out, cudaStream_t st,
                               int* launches, int ld_out) {
  const int entries = p.mt_out * 8 * 8 * gram_n_tiles(p.N);
  gram_reduce_kernel<<<(entries + RED_ENTRIES - 1) / RED_ENTRIES, RED_THREADS, 0, st>>>(
      reduce_args(p, ctas, out, ld_out));
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace bgs
