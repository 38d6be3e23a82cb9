// Microbenchmark: FP64 DFMA / DMMA peak and streaming HBM read bandwidth on B200.
// Used to fix the FP64 roofline denominator (MEASURED_PEAKS.json carries HBM and bf16 only).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void read128(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(p + i); s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void read256(const double* __restrict__ p, size_t n4, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double a0, a1, a2, a3;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3) : "l"(p + 4 * i));
    s += a0 + a1 + a2 + a3;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void copy128(const double2* __restrict__ p, double2* __restrict__ q, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) q[i] = p[i];
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  for (int rep = 0; rep < 3; ++rep) {
    int iters = 20000, blocks = sms * 8, threads = 256;
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 3; ++rep) {
    int iters = 4000, blocks = sms * 8, threads = 256;
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  }
  size_t bytes = size_t(4) << 30;
  double* buf; CK(cudaMalloc(&buf, bytes)); double* buf2; CK(cudaMalloc(&buf2, bytes));
  CK(cudaMemset(buf, 0, bytes));
  for (int occ : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); read128<<<sms * occ, 256>>>((const double2*)buf, bytes / 16, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("read128 occ%d: %.1f GB/s\n", occ, bytes / ms / 1e6);
      cudaEventRecord(e0); read256<<<sms * occ, 256>>>(buf, bytes / 32, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("read256 occ%d: %.1f GB/s\n", occ, bytes / ms / 1e6);
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copy128<<<sms * 4, 256>>>((const double2*)buf, (double2*)buf2, bytes / 16); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy128: %.1f GB/s (r+w)\n", 2.0 * bytes / ms / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
