// DMMA.8x8x4 throughput vs (independent accumulator chains per warp) x (warps per SM),
// one CTA per SM: how much ILP the tile engine's consumer warps need.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters) {
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0;
  double a = threadIdx.x * 1e-9 + 1.0, b = 0.999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  if (s == 1.234) out[0] = s;
}
template <int C> void run(int warps, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  k<C><<<148, 32 * warps>>>(out, iters);
  cudaEventRecord(e0);
  k<C><<<148, 32 * warps>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dmma_per_sm = (double)iters * C * warps;
  double clk = ms * 1e-3 * 1.965e9;
  printf("chains %2d warps/SM %2d : %.2f clk per DMMA per SM, %.1f TF (lat est %.0f clk)\n", C, warps,
         clk / dmma_per_sm, 148 * dmma_per_sm * 512 / (ms * 1e-3) / 1e12, clk / iters);
}
int main() {
  double* out; cudaMalloc(&out, 64);
  for (int w : {4, 8, 12, 16, 32}) { run<1>(w, out); run<2>(w, out); run<4>(w, out); run<8>(w, out); run<16>(w, out); }
  return 0;
}
