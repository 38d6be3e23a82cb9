// Microbenchmark: TMA streaming rate of a column-major n x C fp64 matrix into a shared
// memory ring, as a function of box shape (rows x cols) and ring depth.  Consumers only
// release the slot (no math): this is the load ceiling of the K1/K12 tile engine.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct P {
  CUtensorMap map;
  int dims3;
  int rows_per_box, cols_per_box, boxes_r, boxes_c, stages, colmajor;
  long total_stages;
};

__global__ void __launch_bounds__(160, 1) stream(const __grid_constant__ P p, double* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int box_bytes = p.rows_per_box * p.cols_per_box * 8;
  const int stage_bytes = box_bytes * p.boxes_r * p.boxes_c;
  uint64_t* full = (uint64_t*)(s + (size_t)p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  const long T = p.total_stages;
  const long st0 = blockIdx.x * T / gridDim.x, st1 = (blockIdx.x + 1) * T / gridDim.x;
  const int nst = (int)(st1 - st0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.stages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(W));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < nst; ++it) {
        int slot = it % p.stages, round = it / p.stages;
        uint32_t eb = su32(&empty[slot]);
        asm volatile("{.reg .pred q; W1: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W1;}" ::"r"(eb), "r"((round & 1) ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(stage_bytes));
        unsigned char* dst = s + (size_t)slot * stage_bytes;
        const int row = (int)((st0 + it) * p.rows_per_box * p.boxes_r);
        for (int o = 0; o < p.boxes_r * p.boxes_c; ++o) {
            const int br = p.colmajor ? o % p.boxes_r : o / p.boxes_c;
            const int bc = p.colmajor ? o / p.boxes_r : o % p.boxes_c;
            if (p.dims3)
              asm volatile(
                  "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                  ::"r"(su32(dst + (size_t)(br * p.boxes_c + bc) * box_bytes)), "l"((uint64_t)&p.map),
                  "r"(0), "r"(p.dims3 == 2 ? bc * p.cols_per_box : (row + br * p.rows_per_box) / 16),
                  "r"(p.dims3 == 2 ? (row + br * p.rows_per_box) / 16 : bc * p.cols_per_box), "r"(su32(&full[slot])) : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                  ::"r"(su32(dst + (size_t)(br * p.boxes_c + bc) * box_bytes)), "l"((uint64_t)&p.map),
                  "r"(row + br * p.rows_per_box), "r"(bc * p.cols_per_box), "r"(su32(&full[slot])) : "memory");
          }
      }
    }
    return;
  }
  double acc = 0;
  for (int it = 0; it < nst; ++it) {
    int slot = it % p.stages;
    uint32_t fb = su32(&full[slot]);
    asm volatile("{.reg .pred q; W2: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W2;}" ::"r"(fb), "r"((it / p.stages) & 1));
    acc += ((double*)(s + (size_t)slot * stage_bytes))[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])));
  }
  if (acc == 1.2345) sink[0] = acc;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long n = 1000000, CMAX = 384;
  double* x;
  CK(cudaMalloc(&x, n * CMAX * 8));
  CK(cudaMemset(x, 0, n * CMAX * 8));
  double* sink;
  CK(cudaMalloc(&sink, 64));
  void* fn; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  Enc enc = (Enc)fn;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct Cfg { int rpb, cpb, swz, d3; };
  // d3 = 1: view {16 rows, row-blocks, cols}; d3 = 2: view {16 rows, cols, row-blocks}
  // (smem lines ordered column-major within each 16-row block)
  std::vector<Cfg> cfgs = {{32, 64, 1, 1}, {32, 128, 1, 1}, {32, 64, 1, 2}, {32, 128, 1, 2},
                           {32, 32, 1, 2}, {64, 64, 1, 2}, {64, 128, 1, 2}};
  for (long C : {128L, 384L}) {
    for (auto cf : cfgs) {
      if (C % cf.cpb) continue;
      for (int S : {2, 3, 4}) {
        P p;
        cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)C, 0};
        cuuint64_t str[2] = {(cuuint64_t)n * 8, 0};
        cuuint32_t box[3] = {(cuuint32_t)cf.rpb, (cuuint32_t)cf.cpb, 0};
        cuuint32_t es[3] = {1, 1, 1};
        if (cf.d3 == 1) {
          dims[0] = 16; dims[1] = n / 16; dims[2] = C;
          str[0] = 128; str[1] = n * 8;
          box[0] = 16; box[1] = cf.rpb / 16; box[2] = cf.cpb;
        } else if (cf.d3 == 2) {
          dims[0] = 16; dims[1] = C; dims[2] = n / 16;
          str[0] = n * 8; str[1] = 128;
          box[0] = 16; box[1] = cf.cpb; box[2] = cf.rpb / 16;
        }
        p.dims3 = cf.d3;
        CUresult r = enc(&p.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cf.d3 ? 3 : 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         cf.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d for %dx%d\n", (int)r, cf.rpb, cf.cpb); continue; }
        p.colmajor = 0;
        p.rows_per_box = cf.rpb; p.cols_per_box = cf.cpb; p.boxes_r = 1; p.boxes_c = (int)(C / cf.cpb);
        const int stage_bytes = cf.rpb * (int)C * 8;
        if ((long)S * stage_bytes > 220 * 1024) continue;
        p.stages = S;
        p.total_stages = n / cf.rpb;
        size_t smem = (size_t)p.stages * stage_bytes + 1024 + 16 * p.stages + 64;
        CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int threads = 32 * 5;
        stream<<<sms, threads, smem>>>(p, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int rep = 0; rep < 3; ++rep) stream<<<sms, threads, smem>>>(p, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        double gbs = 3.0 * (double)p.total_stages * stage_bytes / (ms * 1e-3) / 1e9;
        printf("C %3ld d3 %d box %3dx%3d swz%d  boxes/stage %3d stage %6d B S %d : %7.1f GB/s\n", C, cf.d3, cf.rpb, cf.cpb, cf.swz,
               p.boxes_c, stage_bytes, S, gbs);
      }
    }
  }
  return 0;
}
