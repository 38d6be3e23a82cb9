// Are DFMA (FP64 CUDA cores) and DMMA (FP64 tensor) separate pipes on B200?  Run warps
// doing only DMMA, only DFMA, and half/half in the same CTA; compare total throughput.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && (w & 1) == 0);
  double c[8][2]; double x[8];
  for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = 0; x[i] = threadIdx.x * 1e-3 + i; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  if (do_mma) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  } else {
    for (int it = 0; it < iters * 8; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], b, a);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + x[i];
  if (s == 1.234) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"DMMA only", "DFMA only", "half DMMA warps + half DFMA warps"};
  for (int mode = 0; mode < 3; ++mode) {
    int iters = 2000, warps = 16;
    k<<<148, 32 * warps>>>(out, iters, mode);
    cudaEventRecord(e0);
    k<<<148, 32 * warps>>>(out, iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // flops per warp: DMMA warp: iters*8*512 ; DFMA warp: iters*8*8*32*2
    double mma_w = mode == 0 ? warps : mode == 2 ? warps / 2 : 0, fma_w = warps - mma_w;
    double fl = 148.0 * (mma_w * iters * 8.0 * 512 + fma_w * iters * 64.0 * 64);
    printf("%-36s %.3f ms  %.1f TF/s\n", names[mode], ms, fl / (ms * 1e-3) / 1e12);
  }
  return 0;
}
