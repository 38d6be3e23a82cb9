// reduce.cuh — the deterministic cross-CTA Gram reduction (body shared by gram_reduce_kernel
// in gram.cu and the reduce + one-sync-step kernel in small.cu).
//
// A CTA handles RED_ENTRIES output entries with RED_SLICES slices each: slice l sums the
// partial slots g = l, l + RED_SLICES, ... in order (RED_BATCH independent loads in flight
// per thread), then the slice sums are combined in slice order, all in double-double.
// Fixed order -> reproducible run to run.
#pragma once
#include "common.cuh"

namespace bgs {

constexpr int RED_ENTRIES = 16, RED_SLICES = 16, RED_BATCH = 8;
constexpr int RED_THREADS = RED_ENTRIES * RED_SLICES;

// Extra destinations of the reduced Gram (the one-shot exchange's windows, peer.cu): the
// entry written to out[i] also goes to dst[0..n-1][i].
struct ReducePush {
  double* dst[8];
  int n;
};

struct ReduceArgs {
  const double2* part;  // (hi, lo) partial slots
  int G;                // slots
  int mt_out, N8, N;    // slot layout [mt_out][8][N8]
  int ubox0, lcols0, lcols1;
  int M;                // column stride of out
  double* out;
};

// Entry block b reduces entries [b * RED_ENTRIES, (b + 1) * RED_ENTRIES); every thread
// returns (the block barrier inside is reached by all of them).  A CTA may run several
// entry blocks in a row: the barrier at entry protects the shared slice sums of the
// previous one.
template <bool PUSH = false>
BGS_DEV void gram_reduce_body(const ReduceArgs& a, int b, const ReducePush* push = nullptr) {
  __shared__ double2 red[RED_SLICES][RED_ENTRIES];
  const int le = threadIdx.x % RED_ENTRIES, sl = threadIdx.x / RED_ENTRIES;
  const int idx = b * RED_ENTRIES + le;
  const int per_cta = a.mt_out * 8 * a.N8;
  double s = 0.0, e = 0.0;
  if (idx < per_cta) {
    const double2* ptr = a.part + idx;
    for (int g0 = sl; g0 < a.G; g0 += RED_SLICES * RED_BATCH) {
      double2 v[RED_BATCH];
#pragma unroll
      for (int u = 0; u < RED_BATCH; ++u) {
        const int g = g0 + u * RED_SLICES;
        v[u] = g < a.G ? __ldg(ptr + (size_t)g * per_cta) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < RED_BATCH; ++u) {  // adding (0, 0) leaves (s, e) unchanged
        double s2, err;
        two_sum(s, v[u].x, s2, err);
        s = s2;
        e += err + v[u].y;
      }
    }
  }
  __syncthreads();
  red[sl][le] = make_double2(s, e);
  __syncthreads();
  if (sl != 0 || idx >= per_cta) return;
  s = 0.0;
  e = 0.0;
  for (int l = 0; l < RED_SLICES; ++l) {
    const double2 v = red[l][le];
    double s2, err;
    two_sum(s, v.x, s2, err);
    s = s2;
    e += err + v.y;
  }
  const int n = idx % a.N8;
  const int i = (idx / a.N8) % 8;
  const int t = idx / (8 * a.N8);
  if (n >= a.N) return;
  int row;
  if (t < a.ubox0) {
    row = 8 * t + i;
    if (row >= a.lcols0) return;
  } else {
    const int r = 8 * (t - a.ubox0) + i;
    if (r >= a.lcols1) return;
    row = a.lcols0 + r;
  }
  BGS_DCHECK(row < a.M && n < a.N, "gram_reduce: output entry outside the Gram");
  const double val = s + e;
  if (PUSH) {
#pragma unroll 1
    for (int d = 0; d < push->n; ++d) push->dst[d][row + (size_t)n * a.M] = val;
  } else {
    a.out[row + (size_t)n * a.M] = val;
  }
}

}  // namespace bgs
