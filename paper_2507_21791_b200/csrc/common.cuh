// common.cuh — shared device helpers for the sm_100a BCGS kernels.
//
// PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), fp64 DMMA (mma.sync
// m8n8k4.f64 -> SASS DMMA.8x8x4), error-free transformations, and the device status
// word that carries the reference's abort semantics (NotSpdError / NonFiniteError,
// errors.hpp:9-51) between kernels without host round trips.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#define BGS_DEV __device__ __forceinline__

// Checked builds (make checked -> _lib_chk/libbgs_gpu.so, -DBGS_CHECKED): device-side
// bounds checks on the index arithmetic of the hot kernels, trapping with a message.  The
// pool's compute-sanitizer is closed (it left GPUs needing a reset), so these, the
// NaN-poisoned buffers (BGS_POISON) and the fuzzer stand in for memcheck.
#ifdef BGS_CHECKED
#define BGS_DCHECK(cond, what)                                                              \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("[bgs check] %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x, what);                                                           \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define BGS_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

namespace bgs {

// ---------------------------------------------------------------------------------
// Device status word.  The first failing kernel writes {code, pivot, block, site} and
// every later kernel of the factorization early-exits (SURVEY.md §5 failure detection).
// ---------------------------------------------------------------------------------
enum StatusCode : int {
  ST_OK = 0,
  ST_NOT_SPD = 2,
  ST_SINGULAR = 3,
  ST_NON_FINITE = 5,
  ST_COLLECTIVE = 6,  // the peer exchange's in-kernel wait gave up (a rank never published its flag)
};
// Sites of rethrow_not_spd (bcgs.cpp:284, 325, 356, 194, 209).
enum Site : int {
  SITE_NONE = 0,
  SITE_PROLOGUE_PYTH = 1,   // "prologue Pythagorean normalization"
  SITE_FIRST_PASS = 2,      // "first-pass Pythagorean normalization"
  SITE_SECOND_PASS = 3,     // "second-pass Pythagorean normalization"
  SITE_INTRA_CHOLQR = 4,    // "intra-block Cholesky QR" (classic BCGS, bcgs.cpp:111, 123)
};
struct DevStatus {
  int code;
  int pivot;
  int block;  // 1-based block column
  int site;
  int kappa_power;
  int pad[3];
};

BGS_DEV bool status_bad(const DevStatus* st) {
  return *(volatile const int*)&st->code != 0;
}

// ---------------------------------------------------------------------------------
// Shared-memory address / mbarrier / TMA
// ---------------------------------------------------------------------------------
BGS_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

BGS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

BGS_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

BGS_DEV void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

BGS_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

BGS_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

BGS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Single probe of an mbarrier phase (true when the phase with `parity` has completed).
BGS_DEV bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Debug wait: traps with a diagnostic instead of hanging (BGS_TILE_DBG & 64).
BGS_DEV void mbar_wait_dbg(uint64_t* bar, uint32_t parity, int tag, int it) {
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > (1ll << 32)) {
      printf("[bgs hang] block %d thread %d tag %d iteration %d parity %u\n", blockIdx.x,
             threadIdx.x, tag, it, parity);
      __trap();
    }
  }
}

// 2-D tiled TMA load global -> shared, completion on an mbarrier (SASS: UTMALDG).
BGS_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0,
                         int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 3-D tiled TMA load (the {16 rows, row-block, column} view of a column-major matrix).
BGS_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                         int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy global -> shared (bytes: a multiple of 16; both addresses 16-byte aligned),
// completing `bytes` on the mbarrier
BGS_DEV void bulk_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

BGS_DEV void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---------------------------------------------------------------------------------
// fp64 tensor core: D(8x8) += A(8x4, row) * B(4x8, col).  Lane t holds A[t/4][t%4],
// B[t%4][t/4], C/D[t/4][2*(t%4) + {0,1}].
// ---------------------------------------------------------------------------------
BGS_DEV void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 128-bit shared load of two consecutive doubles.
BGS_DEV double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
BGS_DEV double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
BGS_DEV void sts128(uint32_t addr, double a, double b) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
BGS_DEV void sts64(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// ---------------------------------------------------------------------------------
// System-scope release store / acquire load (flags of the peer-memory exchange, peer.cu)
BGS_DEV void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
BGS_DEV unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Bounded acquire spin on a flag of the peer exchange: until *f reached `epoch`, or ~8 s of
// %globaltimer went by (a rank that died or never joined must not hang this GPU): false on
// timeout.
BGS_DEV bool spin_flag_geq(const unsigned* f, unsigned epoch) {
  unsigned long long t0 = 0;
  for (unsigned it = 0; (int)(ld_acquire_sys(f) - epoch) < 0; ++it) {
    __nanosleep(20);
    if ((it & 1023u) == 1023u) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (!t0) t0 = t;
      else if (t - t0 > 8000000000ull) return false;
    }
  }
  return true;
}

// ---------------------------------------------------------------------------------
// Error-free transformation: a + b = s + e exactly (Knuth TwoSum).
// ---------------------------------------------------------------------------------
BGS_DEV void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// ---------------------------------------------------------------------------------
// Stage layout of the tile kernels (gram.cu, k12.cu): a stage is 16H rows x the tile's
// columns; 128-byte line L = H*col + h holds rows 16h..16h+15 of tile column col, its
// 16-byte chunk j stored at chunk j ^ (L & 7) (TMA SWIZZLE_128B of a {16, H, w} box).
// ---------------------------------------------------------------------------------
// byte offset of the 8-byte element (row r, tile column c) inside a stage
template <int H>
BGS_DEV uint32_t elem_off(int col, int r) {
  const int line = H * col + (r >> 4);
  const int chunk = ((r & 15) >> 1) ^ (line & 7);
  return (uint32_t)(line * 128 + chunk * 16 + (r & 1) * 8);
}

// DMMA column-major fragment: rows 16h + 4kk + {0,1,2,3} of tile column `col`; odd-ii
// lanes fetch the two chunks in swapped order so a quarter-warp hits 8 distinct chunks.
template <int H>
BGS_DEV void frag4(uint32_t stage, int col, int h, int kk, int odd, double (&v)[4]) {
  const int line = H * col + h;
  const uint32_t b = stage + (uint32_t)(line * 128);
  const int c0 = (2 * kk + odd) ^ (line & 7), c1 = (2 * kk + 1 - odd) ^ (line & 7);
  const double2 x0 = lds128(b + (uint32_t)(c0 << 4));
  const double2 x1 = lds128(b + (uint32_t)(c1 << 4));
  v[0] = odd ? x1.x : x0.x;
  v[1] = odd ? x1.y : x0.y;
  v[2] = odd ? x0.x : x1.x;
  v[3] = odd ? x0.y : x1.y;
}

// ---------------------------------------------------------------------------------
// Thread-block clusters / distributed shared memory
// ---------------------------------------------------------------------------------
BGS_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address -> the same offset in CTA `rank` of the cluster (shared::cluster)
BGS_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(addr), "r"(rank));
  return d;
}
// 16-byte store into a peer CTA's shared memory that completes `bytes` on the peer's
// mbarrier (no separate fence / arrive needed on the sender side).
BGS_DEV void st_async_v2f64(uint32_t remote_addr, double a, double b, uint32_t remote_bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          remote_addr),
      "d"(a), "d"(b), "r"(remote_bar)
      : "memory");
}
BGS_DEV void cluster_sync_all() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::
          : "memory");
}
BGS_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
// programmatic dependent launch: wait for the preceding grid (its memory is visible
// after this; returns at once when the launch was not programmatic) / allow the next
// grid to launch early
BGS_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
BGS_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// named barrier over `threads` threads (id 0 is __syncthreads)
BGS_DEV void bar_named(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace bgs
