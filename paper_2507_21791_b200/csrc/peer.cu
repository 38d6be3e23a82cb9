// peer.cu — the block step's one synchronization as a ONE-SHOT exchange over peer-mapped
// device memory (NVLink / NVSwitch P2P between GPUs, or CUDA-IPC between processes that
// share a GPU): SURVEY.md §8(f) row 4.
//
// Replaces exact_allreduce (communicator.cpp:226-250) and the TSQR root allgather fused
// with its Gram allreduce (communicator.cpp:252-317) when the ranks can address each
// other's memory.  Every rank owns a window
//     [flags: P x u32, padded][parity 0: P slots][parity 1: P slots]
// and maps every peer's window.  One exchange of epoch e:
//   push   rank r stores its payload [gather | partial] into slot (e & 1, r) of EVERY
//          window (its own included) and then, release-ordered at system scope, writes
//          flag[r] = e into every window;
//   wait   until all P flags of the local window reached e -- either stream memory
//          operations (cuStreamWaitValue32: no kernel waits, so ranks may share a GPU) or,
//          on distinct GPUs, an acquire spin at the head of the sum kernel;
//   sum    every rank adds the P partials of its own window in rank order 0..P-1 (the same
//          order everywhere -> bitwise replicated, as exact_allreduce guarantees) and
//          copies the gathered parts out.
// One network traversal, no second phase: the payload is tiny ((k+2)s x 2s doubles), so
// latency, not bandwidth, is what matters.  Two parities suffice: a rank can only push
// epoch e + 2 after its sum of e + 1, which needs every peer's flag e + 1, which a peer
// writes only after its own sum of e (stream order).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace bgs {

namespace {

// grid (P, B): blocks (p, *) push this rank's payload into window p; the last of them to
// finish (ticket cnt[p]) publishes flag[rank] = epoch there.
__global__ void __launch_bounds__(512) peer_push_kernel(const PeerView v, const double* __restrict__ a,
                                                        unsigned long na, const double* __restrict__ b,
                                                        unsigned long nb, unsigned epoch,
                                                        unsigned* __restrict__ cnt) {
  const int p = blockIdx.x;
  double* dst = reinterpret_cast<double*>(v.win[p] + kPeerFlagBytes +
                                          ((size_t)(epoch & 1u) * v.P + v.rank) * v.slot_bytes);
  const unsigned long stride = (unsigned long)gridDim.y * blockDim.x;
  for (unsigned long i = (unsigned long)blockIdx.y * blockDim.x + threadIdx.x; i < na + nb; i += stride)
    dst[i] = i < na ? a[i] : b[i - na];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(&cnt[p], 1u);
    if (t == gridDim.y - 1) {
      cnt[p] = 0;  // (the next push is stream-ordered behind this kernel)
      __threadfence_system();
      st_release_sys(reinterpret_cast<unsigned*>(v.win[p]) + v.rank, epoch);
    }
  }
}

// Sum / gather out of the local window.  spin: wait here for the P flags (distinct GPUs
// only; otherwise the stream already waited with memory operations).
__global__ void __launch_bounds__(512) peer_sum_kernel(const PeerView v, unsigned long ng,
                                                       double* __restrict__ recv, unsigned long ns,
                                                       double* __restrict__ sum, unsigned epoch,
                                                       int spin, DevStatus* status) {
  unsigned char* win = v.win[v.rank];
  if (spin) {
    if ((int)threadIdx.x < v.P) {
      const unsigned* f = reinterpret_cast<const unsigned*>(win) + threadIdx.x;
      if (!spin_flag_geq(f, epoch) && status) {  // (first writer wins, like every status)
        if (atomicCAS(&status->code, 0, (int)ST_COLLECTIVE) == 0) status->pivot = (int)threadIdx.x + 1;
      }
    }
    __syncthreads();
  }
  const double* base = reinterpret_cast<const double*>(win + kPeerFlagBytes +
                                                       (size_t)(epoch & 1u) * v.P * v.slot_bytes);
  const unsigned long sd = v.slot_bytes / sizeof(double);
  const unsigned long stride = (unsigned long)gridDim.x * blockDim.x;
  const unsigned long t0 = (unsigned long)blockIdx.x * blockDim.x + threadIdx.x;
  for (unsigned long i = t0; i < ns; i += stride) {
    double acc = __ldcv(base + ng + i);
    for (int r = 1; r < v.P; ++r) acc += __ldcv(base + (size_t)r * sd + ng + i);  // rank order
    sum[i] = acc;
  }
  for (unsigned long i = t0; i < ng * (unsigned long)v.P; i += stride) {
    const unsigned long r = i / ng, j = i - r * ng;
    recv[i] = __ldcv(base + r * sd + j);
  }
}

}  // namespace

cudaError_t peer_push_launch(const PeerView& v, const double* a, unsigned long na, const double* b,
                             unsigned long nb, unsigned epoch, unsigned* cnt, cudaStream_t st,
                             int* launches) {
  const unsigned long w = na + nb;
  const int B = (int)std::min<unsigned long>(8, std::max<unsigned long>(1, (w + 4095) / 4096));
  peer_push_kernel<<<dim3((unsigned)v.P, (unsigned)B), 512, 0, st>>>(v, a, na, b, nb, epoch, cnt);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t peer_sum_launch(const PeerView& v, unsigned long ng, double* recv, unsigned long ns,
                            double* sum, unsigned epoch, bool spin, cudaStream_t st, int* launches,
                            DevStatus* status) {
  const unsigned long w = std::max(ns, ng * (unsigned long)v.P);
  const int G = (int)std::min<unsigned long>(32, std::max<unsigned long>(1, (w + 2047) / 2048));
  peer_sum_kernel<<<G, 512, 0, st>>>(v, ng, recv, ns, sum, epoch, spin ? 1 : 0, status);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace bgs
