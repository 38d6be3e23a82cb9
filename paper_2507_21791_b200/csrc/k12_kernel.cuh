// k12_kernel.cuh — K12c: the block update of step k fused in front of the Gram of step k+1, on
// ping-pong consumer warpgroups, optionally split over a CTA pair (cluster of two).
//
// Same algebra and call sites as gram.cu's K12 (onesync_impl bcgs.cpp:329-331, 346-359;
// pipi_impl bcgs.cpp:196-214):
//   A = (srcA - Qp CA) TA^{-1},  B = (srcB - Qp CB - A S2) TB^{-1},  G = [tile]^T [span 1]
//
// Work unit: a stage of RS = 32 R rows (R = 1, 2, 4 chunks of 32 rows; every chunk has the
// stage layout of gram.cu with H = 2: 256-byte column runs, SWIZZLE_128B lines).  Each
// stage costs a roughly fixed latency (update -> reduction -> [exchange] -> epilogue ->
// Gram with two group barriers), so the plan takes the tallest stage that still leaves
// >= 3 stages in shared memory: R = 4 for narrow tiles early in a sweep, R = 1 late.
//
// Warp roles (384 threads, setmaxnreg): warps 0-3 and 4-7 are two consumer groups that take
// alternate stages (one warp per scheduler each, so one group's latency-bound phases hide
// behind the other group's DMMAs); warp 8 lane 0 streams stages with TMA; warps 9-11 idle.
//
// Cluster width C (runtime):
//   C = 1: one CTA holds the whole tile (all span-0 units + span 1).
//   C = 2: late in a sweep one 32-row chunk of the tile is 400+ columns (100+ KB), so the
//     prefix columns are split over a CTA pair.  Rank r loads its own span-0 units, the
//     A-block units (rank 0 only; rank 1 owns them) and all of span 1 (B block and right
//     columns).  Each rank contracts its own k-steps; the partial update of every row is
//     exchanged through distributed shared memory (st.async + mbarrier complete_tx) and
//     both ranks form D_0 + D_1 (same operands -> identical bits).
//
// Per stage and group:
//   update   warp w contracts quad (w mod R) (32 rows = 4 m-tiles, one LDS.128 pair per
//            k-step gives a lane its 4 rows) over k-steps j = w/R + (4/R) t; partials go
//            through shared memory and the epilogue warp sums the 4/R of them in order.
//   epilogue on the tensor core: [A | B] = [srcA - DA | srcB - DB] M, M = [[TA^-1,
//            -TA^-1 W], [0, TB^-1]], W = S2 TB^-1 (2 DMMAs per 8 rows).
//   Gram     this rank's output tiles (warp w: tiles w + 4jj) against span 1, DMMA.8x8x4,
//            folded into double-double (hi, lo) every 4 group-stages.
// Output tiles: rank 0 = own span-0 units + the span-1 left units, rank 1 = its own span-0
// units.  The two groups' double-doubles are combined in the CTA at the end; one partial
// slot per cluster (every tile written by exactly one rank) -> gram_reduce.
// This header holds the kernel template and its launch templates; k12.cu instantiates the
// plain instances and owns the planner, k12_ct.cu the compensated-tile (CT) instances.
#pragma once
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace bgs {
namespace k12d {

constexpr int kGroupWarps = 4;
constexpr int kGroups = 2;
constexpr int kConsWarps = kGroups * kGroupWarps;  // warps 0-7: two consumer groups
constexpr int kProdWarp = kConsWarps;              // warp 8: TMA producer (warps 8-11: its warpgroup)
constexpr int kThreads = 32 * (kConsWarps + 4);
// setmaxnreg: the producer warpgroup gives registers to the two consumer warpgroups
// (4 x 32 x (2 x 240 + 24) = 64512 <= 65536)
constexpr int kProdRegs = 24, kConsRegs = 240;
constexpr int kChunkRows = 32;
constexpr int kUnitChunkBytes = 8 * kChunkRows * 8;  // one 8-column unit of one 32-row chunk
constexpr int kRedBytes = kGroups * kGroupWarps * 4 * 32 * 16;  // [group][warp][m-tile][lane]
// exchange buffers of a cluster of C CTAs: [group][parity][source rank (C - 1)][chunk][warp][lane]
__host__ __device__ constexpr int xchg_bytes(int R, int C = 2) { return (C - 1) * kGroups * 2 * R * kGroupWarps * 32 * 16; }
constexpr int kStaticSmem = 2048;  // epilogue factor arrays (ptxas reports 2048 B static)
constexpr int kSmemOptin = 232448;  // per-block opt-in maximum (227 KB)
constexpr int kMaxStages = 8;


// instances: KW k-steps per warp in 1..16 for each R; MTW covers the output tiles a warp
// can get at that KW: a rank's prefix of KS KW k-steps spans <= KS KW / 2 units, plus the
// A-block unit and one span-1 unit -> mt <= KS KW / 2 + 2 (C = 1 and C = 2 alike)
__host__ __device__ constexpr int mtw_for(int kw, int R) { return ((4 / R) * kw / 2 + 2 + 3) / 4; }
constexpr int kKwMax = 16;
// R = 1 on one CTA: 17 k-steps per warp where three stages still fit (kp = 260 at m = 400;
// wider instances on two stages measured slower than the CTA pair: 33.8 -> 39.6 ms fused)
constexpr int kKwMaxR1 = 17;
// (KW, R) with a second instance at MTW = mtw_for(KW, R) - 1 (see k12_plan)
__host__ __device__ constexpr bool has_narrow(int kw, int R) {
  return (R == 1 && kw % 2 == 0) || (R == 2 && kw % 4 == 3);
}

#if defined(BGS_STEP_STAMPS) && !defined(BGS_K12_NO_STAMPS)
// Debug builds (-DBGS_STEP_STAMPS, tools/stamp_run.py): %globaltimer of every CTA's entry
// dependency-wait release, factors done and first stage ready: [step k][min, max] x 4
__device__ unsigned long long g_k12_log[512 * 8];
extern "C" int bgs_dbg_k12_stamps(unsigned long long* out, int reset) {
  if (reset) {
    static unsigned long long init[512 * 8];
    for (int i = 0; i < 512 * 4; ++i) {
      init[2 * i] = ~0ull;
      init[2 * i + 1] = 0ull;
    }
    return (int)cudaMemcpyToSymbol(g_k12_log, init, sizeof init);
  }
  return (int)cudaMemcpyFromSymbol(out, g_k12_log, sizeof g_k12_log);
}
__device__ __forceinline__ unsigned long long k12_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// QUAD: the cluster-of-4 instances (their own template flag: the generic 4-way exchange in
// the pair instances cost the CTA-pair steps 5%: 215 cycles more in the exchange phase and
// registers in the epilogue).
template <int KW, int MTW, int R, bool CT, bool QUAD = false>
__global__ void __launch_bounds__(kThreads, 1) k12_kernel(const __grid_constant__ SplitParams p) {
#if defined(BGS_STEP_STAMPS) && !defined(BGS_K12_NO_STAMPS)
  const unsigned long long t_entry = k12_gtime();
#endif
  constexpr int KS = 4 / R;                     // k-split factor of the update
  constexpr int RS = kChunkRows * R;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nrk = QUAD ? 4 : p.cluster;  // CTAs per cluster: 1, 2 (or 4: QUAD instances)
  const bool pair = nrk > 1;  // (a cluster splits the prefix columns over its CTAs)
  const int S = p.stages;
  const int chunk_bytes = p.slot_units * kUnitChunkBytes;
  const int slot_bytes = R * chunk_bytes;
  unsigned char* redbuf = smem + (size_t)S * slot_bytes;  // [group][warp][m-tile][lane]
  unsigned char* xbuf = redbuf + kRedBytes;               // [group][parity][chunk][warp][lane]
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + (pair ? xchg_bytes(R, nrk) : 0));
  uint64_t* empty = full + S;
  uint64_t* xfull = empty + S;  // [group][parity]
  __shared__ double ep_t[2][16], ep_s2[16], ep_ai[16], ep_bi[16], ep_w[16], ep_m[64];

  const uint32_t rank = pair ? cluster_ctarank() : 0u;
#ifdef BGS_CHECKED
  // every stage slot, the reduction and exchange buffers and the barriers inside the
  // dynamic allocation (the host sized it with k12_smem_bytes)
  {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const size_t need = (size_t)(smem - smem_raw) + (size_t)S * slot_bytes + kRedBytes +
                        (pair ? xchg_bytes(R, nrk) : 0) + (2 * S + 4) * sizeof(uint64_t);
    BGS_DCHECK(need <= dyn, "k12: shared-memory layout exceeds the allocation");
    BGS_DCHECK(p.own_n[rank] + p.ext_n[rank] + p.U1 <= p.slot_units, "k12: units exceed the slot");
    BGS_DCHECK(S >= 1 && S <= kMaxStages, "k12: ring depth");
  }
#endif
  const int own_u0 = p.own_u0[rank], own_n = p.own_n[rank];
  const int ext_u0 = p.ext_u0[rank], ext_n = p.ext_n[rank];
  const int nloc = own_n + ext_n + p.U1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long T = p.total_stages;
  const int cl = (int)blockIdx.x / nrk;
  const int ncl = (int)gridDim.x / nrk;
  const long st0 = (long)cl * T / ncl;
  const int nst = (int)((long)(cl + 1) * T / ncl - st0);
  const int s = p.s;
  // Launched as a programmatic dependent of the merged reduce + step kernel (p.pdl), the
  // producer streams the first stages before the wait: X / Q were written by kernels that
  // completed before that kernel started; only the coefficients and the status word are
  // its outputs.
  const int pre = p.pdl ? min(S, nst) : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kGroupWarps);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&xfull[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (pair) cluster_sync_all();  // the peer's mbarriers exist before any st.async reaches them

  if (warp >= kProdWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsRegs));
  }
  if (warp >= kProdWarp) {
    // ---------------- producer: one thread streams the stages ----------------
    if (warp == kProdWarp && lane == 0) {
      for (int i = 0; i < 5; ++i) prefetch_tmap(&p.map0[i]);
      for (int i = 0; i < 2; ++i) prefetch_tmap(&p.map1[i]);
      const uint32_t bytes = (uint32_t)(nloc * R * kUnitChunkBytes);
      for (int it = 0; it < nst; ++it) {
        if (it == pre) {
          // the stages past the prefetch wait for the preceding kernel (its status word)
          griddep_wait();
          if (p.status && status_bad(p.status)) break;  // both ranks read the same word
        }
        const int slot = it % S;
        if (it >= S) mbar_wait(&empty[slot], ((it / S) - 1) & 1);
        mbar_arrive_expect_tx(&full[slot], bytes);
#pragma unroll 1
        for (int ch = 0; ch < R; ++ch) {
          unsigned char* dst = smem + (size_t)slot * slot_bytes + (size_t)ch * chunk_bytes;
          const int rb = (int)((st0 + it) * 2 * R + 2 * ch);  // first 16-row block of the chunk
          int u = 0;
          for (int seg = 0; seg < 3; ++seg) {  // own span-0 units, extra units, span 1
            int left = seg == 0 ? own_n : seg == 1 ? ext_n : p.U1;
            int c = seg == 0 ? p.col0[0] + 8 * own_u0 : seg == 1 ? p.col0[0] + 8 * ext_u0 : p.col0[1];
            while (left > 0) {
              int wi;
              const CUtensorMap* mp;
              if (seg < 2) {
                wi = left >= 16 ? 0 : left >= 8 ? 1 : left >= 4 ? 2 : left >= 2 ? 3 : 4;
                mp = &p.map0[wi];
              } else {
                wi = left >= 2 ? 3 : 4;
                mp = &p.map1[wi - 3];
              }
              const int wu = 16 >> wi;
              BGS_DCHECK(u + wu <= p.slot_units, "k12: TMA box past the stage slot");
              tma_load_3d(dst + (size_t)u * kUnitChunkBytes, mp, &full[slot], 0, rb, c);
              u += wu;
              c += 8 * wu;
              left -= wu;
            }
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- consumers: group g takes stages g, g+2, g+4, ... ----------------
    const int g = warp / kGroupWarps, w = warp % kGroupWarps;
    const int gtid = threadIdx.x - 32 * kGroupWarps * g;
    const int ii = lane >> 2, kk = lane & 3;
    const int gbar = 1 + g;
    // Update: this rank's k-steps are prefix columns [8 own_u0, pc1) (local columns from
    // 0); warp w contracts quad qd = w mod R over k-steps j = kpart + KS t.  Lane (ii, kk)
    // holds C[4j + kk][n = ii] of [CA | CB] (CA in n = 0..3, CB in n = 4..7, zero padded)
    // as the DMMA B fragment.
    const int qd = w % R, kpart = w / R;
    const int pc1 = min(8 * (own_u0 + own_n), p.kp);
    const int kcols = max(0, pc1 - 8 * own_u0);
    // The last k-step may be partial (s = 1, 2, 3): its columns past kcols have zero
    // coefficients and hold finite data (the A block, or Q columns zeroed by the runtime).
    const int ksteps = (kcols + 3) / 4;
    const int jlast = max(ksteps - 1, 0);
    const int kt_valid = kpart < ksteps ? (ksteps - 1 - kpart) / KS + 1 : 0;  // real k-steps
    // Update A fragments: m-tile q, row index i is chunk row 4 f(i) + q with
    // f(i) = (i >> 1) + 4 (i & 1), so lane (i, kk) reads rows 4f..4f+3 of tile column
    // 4j + kk with two LDS.128 (line 8j + 2kk + (i & 1), 1024 j past k-step 0).  The two
    // i of a quarter-warp sit in different 16-row halves -> chunk sets {2a ^ 2kk} and
    // {2a ^ (2kk + 1)} are disjoint: conflict-free with no lane swap.
    uint32_t uoff0, uoff1;
    {
      const int line = 2 * kk + (ii & 1);
      const int rc = 2 * (ii >> 1);  // chunk of rows 4f, 4f + 1 inside the 16-row block
      uoff0 = (uint32_t)(line * 128 + ((rc ^ (line & 7)) << 4));
      uoff1 = (uint32_t)(line * 128 + (((rc + 1) ^ (line & 7)) << 4));
    }
    // local columns of the A block, the B block (= span-1 column 0) and the right operand
    const bool a_own = p.kp >= 8 * own_u0 && p.kp < 8 * (own_u0 + own_n);
    const int colA = a_own ? p.kp - 8 * own_u0 : 8 * own_n + p.kp - 8 * ext_u0;
    const int colB = 8 * (own_n + ext_n);
    const int rc = ii < p.N ? p.rcol1[ii] : -1;
    const bool bval = rc >= 0;
    const int bcol = colB + (bval ? rc : 0);
    // output tiles of this rank: own units, then (rank 0) the span-1 left units
    const int mt_loc = own_n + (rank == 0 ? p.s1_left : 0);
    // Epilogue: warp w handles rows 8w + m (m = lane / 4) of every chunk (coalesced
    // stores); in the update that row is m-tile q = m & 3, index i with
    // f(i) = 2w + (m >> 2), of the chunk's quad.
    const int erow = 8 * w + ii;
    const int qsel = ii & 3, vsel = 2 * w + (ii >> 2), isel = 2 * (vsel & 3) + (vsel >> 2);
    const int quad = lane & ~3;
    // Per-lane epilogue plan, fixed for the whole kernel (the stage loop only adds the stage
    // base and the row offset): lane (i, kk) reads z[row][kk] of both source blocks and owns
    // output columns 2kk, 2kk + 1 (A for kk < 2, B for kk >= 2).  Recomputing these per stage
    // cost ~250 cycles of a ~5000-cycle group-stage (33.8 -> 32.9 ms of fused time at config 2).
    constexpr bool kEpPlan = MTW <= 6 || (MTW == 7 && KW <= 12);  // (wider: no registers to spare, measured)
    const bool ep_isA = kk < 2;
    const bool ep_za = p.upd_a && kk < s, ep_zb = p.upd_b && kk < s;
    const uint32_t ep_offA = elem_off<2>(colA + kk, erow), ep_offB = elem_off<2>(colB + kk, erow);
    const long ep_ld = ep_isA ? p.lddA : p.lddB;
    uint32_t ep_so[2];  // shared-memory offsets of the two outputs inside a chunk
    int ep_flags = 0;   // bit e: store output e to the stage; bit 2 + e: store it to HBM
    {
      const int c0 = ep_isA ? 2 * kk : 2 * kk - 4;
      const bool on = ep_isA ? p.upd_a : p.upd_b;
      // global stores: rank 0 writes A, rank 1 writes B (C = 1: rank 0 writes both);
      // shared: A only where its rows are output tiles (the rank owning the A units)
      const bool gst = !pair || (ep_isA ? rank == 0 : rank == 1);
      const bool sst = ep_isA ? (!pair || (int)rank == nrk - 1) : true;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ep_so[e] = elem_off<2>((ep_isA ? colA : colB) + c0 + e, erow);
        if (on && c0 + e < s) ep_flags |= (sst ? 1 << e : 0) | (gst ? 4 << e : 0);
      }
    }
    // HBM address of output 0 at shard row 0 of this lane's chunk row
    double* const ep_g = (ep_isA ? p.dstA : p.dstB) + erow +
                         (size_t)(ep_isA ? 2 * kk : 2 * kk - 4) * (size_t)ep_ld;
    int acol[MTW];  // tile column of this lane's Gram fragment, per output tile
    // (CT) compensated output tiles: global tile index >= p.comp_t0 -> every 4-row k-step
    // goes straight into the double-double (BCGSI+1S: the U rows)
    // The compensated tile of a fused step is always the span-1 left unit on rank 0
    // (U_{k+1} and X_{k+2} as output rows; the runtime plans K12c only for that layout).  It
    // is shared by the four warps of a group: warp w takes the 4-row k-steps q4 = w of
    // every row pass into its own double-double (coop_*), outside the branch-free tile
    // loop -- a per-tile flag tested at every DMMA split that loop into basic blocks and
    // made every step ~1.5x slower -- and the partials of the 8 warps are added in a fixed
    // order at the end.
    const bool coop = CT && p.comp_t0 == p.U0 && p.mt_out - p.comp_t0 == 1 && rank == 0 && p.s1_left == 1;
    const int coop_col = 8 * (own_n + ext_n) + ii;  // the tile's column of this lane (span-1 unit 0)
    // (one double-double per row pass u: two independent two_sum chains per warp)
    double coop_hi[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, coop_lo[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int jj = 0; jj < MTW; ++jj) {
      int t = w + kGroupWarps * jj;
      if (t >= mt_loc) t = w < mt_loc ? w : 0;
      const int lu = t < own_n ? t : t + ext_n;
      acol[jj] = 8 * lu + ii;
    }

    // Everything above depends on the launch parameters only and runs while the preceding
    // kernel (the reduce + step) is still in flight; what follows reads its outputs.
    // Coefficients, factors and the status word come from the preceding kernel.
    griddep_wait();
#if defined(BGS_STEP_STAMPS) && !defined(BGS_K12_NO_STAMPS)
    const unsigned long long t_wait = k12_gtime();
#endif
    if (p.status && status_bad(p.status)) {
      // an earlier step failed: drain the stages prefetched before the producer saw it
      for (int it = g; it < pre; it += kGroups) mbar_wait(&full[it % S], (it / S) & 1);
    } else {
    double bco[KW];
#pragma unroll
    for (int t = 0; t < KW; ++t) {
      const int lc = 4 * (kpart + KS * t) + kk, c = 8 * own_u0 + lc;
      double v = 0.0;
      if (lc < kcols) {
        if (ii < 4) {
          if (ii < s && p.upd_a) v = p.CA[c + (size_t)ii * p.ldca];
        } else if (ii - 4 < s && p.upd_b) {
          v = p.CB[c + (size_t)(ii - 4) * p.ldcb];
        }
      }
      bco[t] = v;
    }
    // (after the coefficient loads: their latency hides under the factor arithmetic)
    // Epilogue factors padded to 4x4 with identity: TA^{-1}, TB^{-1}, W = S2 TB^{-1}.
    if (threadIdx.x < 16) {
      const int i = threadIdx.x & 3, j = threadIdx.x >> 2;
      const bool in = i < s && j < s;
      const double id = i == j ? 1.0 : 0.0;
      ep_t[0][threadIdx.x] = (in && p.TA) ? p.TA[i + j * s] : id;
      ep_t[1][threadIdx.x] = (in && p.TB) ? p.TB[i + j * s] : id;
      ep_s2[threadIdx.x] = (in && p.upd_a && p.upd_b) ? p.CB[p.kp + i + (size_t)j * p.ldcb] : 0.0;
    }
    bar_named(5, 32 * kConsWarps);
    if (threadIdx.x < 8) {
      const int which = threadIdx.x >> 2, j = threadIdx.x & 3;
      const double* Tm = ep_t[which];
      double* Ti = which ? ep_bi : ep_ai;
      for (int i = 3; i >= 0; --i) {  // column j of T^{-1}: T y = e_j
        double acc = (i == j) ? 1.0 : 0.0;
        for (int l = i + 1; l < 4; ++l) acc -= Tm[i + 4 * l] * Ti[l + 4 * j];
        Ti[i + 4 * j] = acc / Tm[i + 4 * i];
      }
    }
    bar_named(5, 32 * kConsWarps);
    if (threadIdx.x < 16) {
      const int m = threadIdx.x & 3, j = threadIdx.x >> 2;
      double acc = 0.0;
      for (int l = 0; l < 4; ++l) acc += ep_s2[m + 4 * l] * ep_bi[l + 4 * j];
      ep_w[m + 4 * j] = acc;
    }
    bar_named(5, 32 * kConsWarps);
    // M[l][j] (row-major 8 x 8): out = z M with z = [srcA - DA, srcB - DB]
    if (threadIdx.x < 64) {
      const int l = threadIdx.x >> 3, j = threadIdx.x & 7;
      double v = 0.0;
      if (l < 4 && j < 4) {
        v = p.upd_a ? ep_ai[l + 4 * j] : 0.0;
      } else if (l < 4) {  // -(TA^-1 W)[l][j-4]
        if (p.upd_a && p.upd_b) {
          double acc = 0.0;
          for (int m = 0; m < 4; ++m) acc += ep_ai[l + 4 * m] * ep_w[m + 4 * (j - 4)];
          v = -acc;
        }
      } else if (j >= 4) {
        v = p.upd_b ? ep_bi[(l - 4) + 4 * (j - 4)] : 0.0;
      }
      ep_m[l * 8 + j] = v;
    }
    bar_named(5, 32 * kConsWarps);
    // epilogue matrix M as DMMA B fragments: lane (i, kk) holds M[kk][i] and M[4 + kk][i]
    const double mb0 = ep_m[kk * 8 + ii], mb1 = ep_m[(4 + kk) * 8 + ii];

    // (hi, lo) double-double per output; the stage contractions accumulate in acc and are
    // folded in every kFold = 16 / R group-stages (<= 512 rows of plain fp64 per fold at
    // every R; folding every stage costs ~7% of the kernel: the two_sums share the FP64
    // pipe with DMMA; 4 stages at R = 1 cost 0.3 ms more than 16 at config 2)
    constexpr int kFold = MTW >= 9 ? 1 : 16 / R;  // (MTW = 9: registers for acc are short)
    // Skipping padding DMMAs (warp-uniform branches) pays only in the widest instance
    // (up to 3 of 9 tiles per warp are padding there: -12% at kp = 248..256); elsewhere the
    // branches cost 2-4% of scheduling freedom (same-box A/B, tools/ab_perstep.sh).
    constexpr bool kSkipPad = MTW >= 9;
    double hi[MTW][2], lo[MTW][2], acc[MTW][2];
#pragma unroll
    for (int j = 0; j < MTW; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) hi[j][e] = lo[j][e] = acc[j][e] = 0.0;
    auto fold = [&]() {
#pragma unroll
      for (int jj = 0; jj < MTW; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double sm, err;
          two_sum(hi[jj][e], acc[jj][e], sm, err);
          hi[jj][e] = sm;
          lo[jj][e] += err;
          acc[jj][e] = 0.0;
        }
    };

    const uint32_t sbase = smem_u32(smem);
    const uint32_t red_g = smem_u32(redbuf) + (uint32_t)(g * kGroupWarps * 4 * 32 * 16);
    const uint32_t red_w = red_g + (uint32_t)((w * 4 * 32 + lane) * 16);
    const uint32_t red_r = red_g + (uint32_t)((qsel * 32 + 4 * isel + kk) * 16);
    const uint32_t xb_local = smem_u32(xbuf);
    const uint32_t xfull_local = smem_u32(xfull);
    const bool prof = p.phase && gtid == 0;
    // per-stage timeline of CTA 0 (both groups, first kTl group-stages): wait start, data
    // ready, update done, exchange done, epilogue done, Gram done (BGS_TILE_PROF)
    constexpr int kTl = 48;
    unsigned long long* tl = (prof && blockIdx.x == 0) ? p.phase + 2560 + (size_t)g * kTl * 6 : nullptr;
    unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};  // full wait, update, exchange, epilogue, gram
    const unsigned long long t_begin = prof ? clock64() : 0;
    for (int j = 0;; ++j) {
      const int it = g + kGroups * j;
      if (it >= nst) break;
      const int slot = it % S;
      unsigned long long t0 = prof ? clock64() : 0;
#if defined(BGS_STEP_STAMPS) && !defined(BGS_K12_NO_STAMPS)
      const unsigned long long t_pre = k12_gtime();
#endif
      mbar_wait(&full[slot], (it / S) & 1);
      unsigned long long t1 = prof ? clock64() : 0;
#if defined(BGS_STEP_STAMPS) && !defined(BGS_K12_NO_STAMPS)
      if (j == 0 && g == 0 && gtid == 0 && p.kp / p.s < 512) {
        const unsigned long long t_ready = k12_gtime();
        unsigned long long* o = g_k12_log + (size_t)(p.kp / p.s) * 8;
        // [min, max] of: entry (0, 1), dependency wait released (2, 3), first stage ready
        // (6, 7); the CTA end goes to (4, 5) at the bottom of the kernel
        (void)t_pre;
        atomicMin(&o[0], t_entry); atomicMax(&o[1], t_entry);
        atomicMin(&o[2], t_wait);  atomicMax(&o[3], t_wait);
        atomicMin(&o[6], t_ready); atomicMax(&o[7], t_ready);
      }
#endif
      if (prof) ph[0] += t1 - t0;
      if (tl && j < kTl) { tl[j * 6 + 0] = t0; tl[j * 6 + 1] = t1; }
      const uint32_t base = sbase + (uint32_t)(slot * slot_bytes);
      const long row0 = (st0 + it) * RS;
      const int vrows = (int)((p.n_rows - row0) < RS ? (p.n_rows - row0) : RS);
      if (vrows < RS) {
        // rows past the shard end inside its last 16-row block are not TMA zero-filled
        const int ncol = nloc * 8, nr = RS - vrows;
        for (int e = gtid; e < ncol * nr; e += 32 * kGroupWarps) {
          const int r = vrows + e % nr;
          sts64(base + (uint32_t)((r >> 5) * chunk_bytes) + elem_off<2>(e / nr, r & 31), 0.0);
        }
        bar_named(gbar, 32 * kGroupWarps);
      }

      // ---- update partial: quad qd (4 m-tiles = 4 DMMA chains), k-steps kpart + KS t ----
      // Branch-free so ptxas can hoist the loads of later k-steps: k-steps past this
      // rank's range have zero coefficients and read the last valid k-step (finite data).
      {
        double d[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q][0] = d[q][1] = 0.0;
        const uint32_t cb = base + (uint32_t)(qd * chunk_bytes);
#pragma unroll
        for (int t = 0; t < KW; ++t) {
          // (kSkipPad) padding k-steps (zero coefficients) at the end of a warp's range are
          // skipped: warp-uniform, and adding their zero products would not change a bit
          if (kSkipPad && t >= KW - 2 && t >= kt_valid) break;
          const int jk = min(kpart + KS * t, jlast);
          const uint32_t a = cb + 1024u * (uint32_t)jk;
          const double2 x0 = lds128(a + uoff0), x1 = lds128(a + uoff1);
          dmma(d[0][0], d[0][1], x0.x, bco[t]);
          dmma(d[1][0], d[1][1], x0.y, bco[t]);
          dmma(d[2][0], d[2][1], x1.x, bco[t]);
          dmma(d[3][0], d[3][1], x1.y, bco[t]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) sts128(red_w + (uint32_t)(q * 32 * 16), d[q][0], d[q][1]);
      }
      bar_named(gbar, 32 * kGroupWarps);
      if (prof) { const unsigned long long t = clock64(); ph[1] += t - t1; t1 = t; if (tl && j < kTl) tl[j * 6 + 2] = t; }

      // ---- per chunk: sum the KS warp partials of this lane's row (fixed order) ----
      double D0[R], D1[R];
#pragma unroll
      for (int ch = 0; ch < R; ++ch) {
        D0[ch] = D1[ch] = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < KS; ++k2) {
          const int ws = ch + R * k2;  // warp that contracted quad ch, k-part k2
          const double2 v = lds128(red_r + (uint32_t)(ws * 4 * 32 * 16));
          D0[ch] += v.x;
          D1[ch] += v.y;
        }
      }
      if (pair) {
        if constexpr (QUAD) {
          // ---- exchange with the same warp of every peer rank (DSMEM); rank q's partial lands
          // in source slot (q < r ? q : q - 1) of rank r ----
          const int xb = g * 2 + (j & 1);
  #pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (q >= nrk || q == (int)rank) continue;
            const int src = (int)rank < q ? (int)rank : (int)rank - 1;
            const uint32_t rbar = mapa_shared(xfull_local + (uint32_t)(xb * 8), (uint32_t)q);
  #pragma unroll
            for (int ch = 0; ch < R; ++ch) {
              const uint32_t dst = xb_local + (uint32_t)((((((xb * (nrk - 1) + src) * R + ch) * kGroupWarps + w) * 32 + lane) * 16));
              st_async_v2f64(mapa_shared(dst, (uint32_t)q), D0[ch], D1[ch], rbar);
            }
          }
          if (w == 0 && lane == 0) mbar_arrive_expect_tx(&xfull[xb], (nrk - 1) * R * kGroupWarps * 32 * 16);
          mbar_wait(&xfull[xb], (j >> 1) & 1);  // data and completion are both CTA-local
          // every rank adds the partials in rank order 0, 1, ...: identical bits on all of them
          // (two ranks: own + other, as IEEE addition commutes)
  #pragma unroll
          for (int ch = 0; ch < R; ++ch) {
            double a0 = 0.0, a1 = 0.0;
  #pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (q >= nrk) continue;
              double2 v;
              if (q == (int)rank) {
                v = make_double2(D0[ch], D1[ch]);
              } else {
                const int src = q < (int)rank ? q : q - 1;
                v = lds128(xb_local + (uint32_t)((((((xb * (nrk - 1) + src) * R + ch) * kGroupWarps + w) * 32 + lane) * 16)));
              }
              if (q == 0) {
                a0 = v.x;
                a1 = v.y;
              } else {
                a0 += v.x;
                a1 += v.y;
              }
            }
            D0[ch] = a0;
            D1[ch] = a1;
          }
        } else {
          // ---- exchange with the same warp of the peer rank (DSMEM) ----
          const uint32_t peer = rank ^ 1u;
          const int xb = g * 2 + (j & 1);
          const uint32_t rbar = mapa_shared(xfull_local + (uint32_t)(xb * 8), peer);
#pragma unroll
          for (int ch = 0; ch < R; ++ch) {
            const uint32_t mine =
                xb_local + (uint32_t)((((xb * R + ch) * kGroupWarps + w) * 32 + lane) * 16);
            st_async_v2f64(mapa_shared(mine, peer), D0[ch], D1[ch], rbar);
          }
          if (w == 0 && lane == 0) mbar_arrive_expect_tx(&xfull[xb], R * kGroupWarps * 32 * 16);
          mbar_wait(&xfull[xb], (j >> 1) & 1);  // data and completion are both CTA-local
#pragma unroll
          for (int ch = 0; ch < R; ++ch) {
            const uint32_t mine =
                xb_local + (uint32_t)((((xb * R + ch) * kGroupWarps + w) * 32 + lane) * 16);
            const double2 o = lds128(mine);
            D0[ch] += o.x;  // IEEE addition commutes: both ranks hold (rank 0) + (rank 1)
            D1[ch] += o.y;
          }
        }
      }
      if (prof) { const unsigned long long t = clock64(); ph[2] += t - t1; t1 = t; if (tl && j < kTl) tl[j * 6 + 3] = t; }

      // ---- epilogue on the tensor core: [A | B] = [srcA - DA | srcB - DB] M ----
      // A operand lane (i, kk): z[row][kk] and z[row][4 + kk]; D[row][c] sits in lane
      // (i, c / 2), element c & 1.
#pragma unroll
      for (int ch = 0; ch < R; ++ch) {
        const uint32_t cb = base + (uint32_t)(ch * chunk_bytes);
        const int sl = quad | (kk >> 1);
        const double t0 = __shfl_sync(0xffffffffu, D0[ch], sl), t1 = __shfl_sync(0xffffffffu, D1[ch], sl);
        const double u0 = __shfl_sync(0xffffffffu, D0[ch], sl | 2);
        const double u1 = __shfl_sync(0xffffffffu, D1[ch], sl | 2);
        if constexpr (kEpPlan) {
          const double sa = ep_za ? lds64(cb + ep_offA) : 0.0;
          const double sb = ep_zb ? lds64(cb + ep_offB) : 0.0;
          const double za = ep_za ? sa - ((kk & 1) ? t1 : t0) : 0.0;
          const double zb = ep_zb ? sb - ((kk & 1) ? u1 : u0) : 0.0;
          double o0 = 0.0, o1 = 0.0;
          dmma(o0, o1, za, mb0);
          dmma(o0, o1, zb, mb1);
          // lane (i, kk) now holds output columns 2kk, 2kk + 1: A for kk < 2, B for kk >= 2
          if (ep_flags & 1) sts64(cb + ep_so[0], o0);
          if (ep_flags & 2) sts64(cb + ep_so[1], o1);
          if (kChunkRows * ch + erow < vrows) {  // (rows past the shard end are not stored)
            double* g = ep_g + (row0 + kChunkRows * ch);
            BGS_DCHECK(!(ep_flags & 12) || row0 + kChunkRows * ch + erow < p.n_rows,
                       "k12: epilogue store outside the shard");
            if (ep_flags & 4) g[0] = o0;
            if (ep_flags & 8) g[ep_ld] = o1;
          }
        } else {
          // (wide instances: the plan's registers would spill; recompute per stage)
          const bool cv = kk < s;
          const double sa = (p.upd_a && cv) ? lds64(cb + elem_off<2>(colA + kk, erow)) : 0.0;
          const double sb = (p.upd_b && cv) ? lds64(cb + elem_off<2>(colB + kk, erow)) : 0.0;
          const double za = (p.upd_a && cv) ? sa - ((kk & 1) ? t1 : t0) : 0.0;
          const double zb = (p.upd_b && cv) ? sb - ((kk & 1) ? u1 : u0) : 0.0;
          double o0 = 0.0, o1 = 0.0;
          dmma(o0, o1, za, mb0);
          dmma(o0, o1, zb, mb1);
          // lane (i, kk) now holds output columns 2kk, 2kk + 1: A for kk < 2, B for kk >= 2
          const bool isA = kk < 2;
          const int c0 = isA ? 2 * kk : 2 * kk - 4;
          const bool on = isA ? p.upd_a : p.upd_b;
          const int lcol = isA ? colA : colB;
          const int crow = kChunkRows * ch + erow;
          const bool live = crow < vrows;
          const long grow = row0 + crow;
          double* gdst = isA ? p.dstA : p.dstB;
          const long gld = isA ? p.lddA : p.lddB;
          // global stores: rank 0 writes A, rank 1 writes B (C = 1: rank 0 writes both);
          // shared: A only where its rows are output tiles (the rank owning the A units)
          const bool gstore = live && (!pair || (isA ? rank == 0 : rank == 1));
          const bool sstore = isA ? (!pair || (int)rank == nrk - 1) : true;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = c0 + e;
            if (on && c < s) {
              const double v = e ? o1 : o0;
              if (sstore) sts64(cb + elem_off<2>(lcol + c, erow), v);
              BGS_DCHECK(!gstore || (grow < p.n_rows && c < s), "k12: epilogue store outside the shard");
              if (gstore) gdst[grow + (size_t)c * gld] = v;
            }
          }
        }
      }
      bar_named(gbar, 32 * kGroupWarps);
      if (prof) { const unsigned long long t = clock64(); ph[3] += t - t1; t1 = t; if (tl && j < kTl) tl[j * 6 + 4] = t; }

      // ---- Gram of this rank's output tiles (w + 4 jj) against span 1 ----
      // k-index kk of pass u covers chunk rows 16 (kk & 1) + 8 (kk >> 1) + 4u + {0..3}: for
      // the two tile columns of a quarter-warp the chunk sets are S and S ^ 2 with
      // S = {0, 1, 4, 5} (u = 0) or {2, 3, 6, 7} (u = 1) -> conflict-free, no swap.
#pragma unroll
      for (int ch = 0; ch < R; ++ch) {
        const uint32_t cb = base + (uint32_t)(ch * chunk_bytes);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int gh = kk & 1, rcu = 4 * (kk >> 1) + 2 * u;  // half, chunk of the first row pair
          auto gfrag = [&](int col, double (&v)[4]) {
            const int line = 2 * col + gh;
            const uint32_t bl = cb + (uint32_t)(line * 128);
            const double2 x0 = lds128(bl + (uint32_t)((rcu ^ (line & 7)) << 4));
            const double2 x1 = lds128(bl + (uint32_t)(((rcu + 1) ^ (line & 7)) << 4));
            v[0] = x0.x; v[1] = x0.y; v[2] = x1.x; v[3] = x1.y;
          };
          double b[4];
          gfrag(bcol, b);
          if (!bval) b[0] = b[1] = b[2] = b[3] = 0.0;
          // branch-free: tiles past mt_loc re-read a valid tile; dropped at the end
#pragma unroll
          for (int jp = 0; jp < MTW; jp += 2) {
            double a0[4], a1[4];
            gfrag(acol[jp], a0);
            if (jp + 1 < MTW) gfrag(acol[jp + 1], a1);
            // (kSkipPad) tiles past this rank's last output tile are dropped at the end: their
            // DMMAs are skipped (warp-uniform; only the last two tiles of a warp can be such)
            const bool v0 = !kSkipPad || jp < MTW - 2 || w + kGroupWarps * jp < mt_loc;
            const bool v1 = !kSkipPad || jp + 1 < MTW - 2 || w + kGroupWarps * (jp + 1) < mt_loc;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              if (v0) dmma(acc[jp][0], acc[jp][1], a0[q4], b[q4]);
              if (jp + 1 < MTW) {
                if (v1) dmma(acc[jp + 1][0], acc[jp + 1][1], a1[q4], b[q4]);
              }
            }
          }
          if (CT && coop) {
            // this warp's k-step (q4 = w) of the shared compensated tile: one 16-byte
            // fragment chunk (rows 4u'.. of the pass) and the matching right fragment
            const int line = 2 * coop_col + gh;
            const double2 x = lds128(cb + (uint32_t)(line * 128) +
                                     (uint32_t)(((rcu + (w >> 1)) ^ (line & 7)) << 4));
            const double av = (w & 1) ? x.y : x.x;
            const double bv = w == 0 ? b[0] : w == 1 ? b[1] : w == 2 ? b[2] : b[3];
            double c0 = 0.0, c1 = 0.0, sm, err;
            dmma(c0, c1, av, bv);
            two_sum(coop_hi[u][0], c0, sm, err);
            coop_hi[u][0] = sm;
            coop_lo[u][0] += err;
            two_sum(coop_hi[u][1], c1, sm, err);
            coop_hi[u][1] = sm;
            coop_lo[u][1] += err;
          }
        }
      }
      fence_proxy_async();  // generic writes of A / B before TMA refills the slot
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if ((j % kFold) == kFold - 1) fold();
      if (prof) { const unsigned long long t = clock64(); ph[4] += t - t1; if (tl && j < kTl) tl[j * 6 + 5] = t; }
    }
    fold();
    if (prof) {
      ph[5] = clock64() - t_begin;
      unsigned long long* dst = p.phase + (size_t)blockIdx.x * 16 + 8 * g;
      for (int i = 0; i < 6; ++i) atomicAdd(&dst[i], ph[i]);
      atomicAdd(&dst[6], (unsigned long long)((nst - g + 1) / 2));
    }
    // ---- combine the two groups' double-doubles in a fixed order, one slot per cluster ----
    // Both groups are past their last stage after this barrier, so every TMA write has
    // landed and the stage ring (>= MTW x 4 KB: a tile needs its unit in every slot) is free.
    bar_named(3, 32 * kConsWarps);
    const uint32_t park = sbase;
    if (g == 1) {
#pragma unroll
      for (int jj = 0; jj < MTW; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          sts128(park + (uint32_t)((((w * MTW + jj) * 2 + e) * 32 + lane) * 16), hi[jj][e], lo[jj][e]);
    }
    // the shared compensated tile: every warp's partial, [group][warp][element][lane]
    const uint32_t cpark = park + (uint32_t)(kGroupWarps * MTW * 2 * 32 * 16);
    if (CT && coop) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {  // the two row passes first (u = 0, then u = 1)
        double sm, err;
        two_sum(coop_hi[0][e], coop_hi[1][e], sm, err);
        sts128(cpark + (uint32_t)((((g * kGroupWarps + w) * 2 + e) * 32 + lane) * 16), sm,
               err + (coop_lo[0][e] + coop_lo[1][e]));
      }
    }
    bar_named(3, 32 * kConsWarps);
    if (CT && coop && g == 0 && w == 0) {
      double2* part = reinterpret_cast<double2*>(p.partial) + (size_t)cl * p.mt_out * 64;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double h = 0.0, l = 0.0;
        for (int i = 0; i < kGroups * kGroupWarps; ++i) {  // fixed order: group 0 warps 0..3, group 1 ...
          const double2 o = lds128(cpark + (uint32_t)(((i * 2 + e) * 32 + lane) * 16));
          double sm, err;
          two_sum(h, o.x, sm, err);
          h = sm;
          l += err + o.y;
        }
        part[((size_t)p.comp_t0 * 8 + ii) * 8 + 2 * kk + e] = make_double2(h, l);
      }
    }
    if (g == 0) {
      double2* part = reinterpret_cast<double2*>(p.partial) + (size_t)cl * p.mt_out * 64;
#pragma unroll
      for (int jj = 0; jj < MTW; ++jj) {
        const int t = w + kGroupWarps * jj;
        const int tg = t < own_n ? own_u0 + t : p.U0 + (t - own_n);
        if (t < mt_loc && !(CT && coop && tg == p.comp_t0)) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double2 o = lds128(park + (uint32_t)((((w * MTW + jj) * 2 + e) * 32 + lane) * 16));
            double sm, err;
            two_sum(hi[jj][e], o.x, sm, err);
            BGS_DCHECK(tg < p.mt_out, "k12: partial tile outside the slot");
            part[((size_t)tg * 8 + ii) * 8 + 2 * kk + e] = make_double2(sm, err + (lo[jj][e] + o.y));
          }
        }
      }
    }
    }  // live
  }
  if (pair) cluster_sync_all();  // no CTA leaves while its peer may still address its smem
#if defined(BGS_STEP_STAMPS) && !defined(BGS_K12_NO_STAMPS)
  if (threadIdx.x == 0 && p.kp / p.s < 512) {
    const unsigned long long t_end = k12_gtime();
    atomicMin(&g_k12_log[(size_t)(p.kp / p.s) * 8 + 4], t_end);
    atomicMax(&g_k12_log[(size_t)(p.kp / p.s) * 8 + 5], t_end);
  }
#endif
}

template <int KW, int R, bool CT, int MTW = mtw_for(KW, R), bool QUAD = false>
static cudaError_t launch_k12(const SplitParams& p, int grid, cudaStream_t st) {
  auto k = k12_kernel<KW, MTW, R, CT, QUAD>;
  const size_t smem = k12_smem_bytes(p.stages, p.slot_units, R, p.cluster);
  cudaError_t e = ensure_smem(k, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (p.cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = (unsigned)p.cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (p.pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, p);
}

template <int R, bool CT>
static cudaError_t launch_r(const SplitParams& p, int grid, cudaStream_t st) {
  if (p.mtw == mtw_for(p.kw, R) - 1) {
    switch (p.kw) {
#define BGS_NKW(K) \
  case K:          \
    if constexpr (has_narrow(K, R)) return launch_k12<K, R, CT, mtw_for(K, R) - 1>(p, grid, st); \
    break;
      BGS_NKW(2) BGS_NKW(3) BGS_NKW(4) BGS_NKW(6) BGS_NKW(7) BGS_NKW(8) BGS_NKW(10)
      BGS_NKW(11) BGS_NKW(12) BGS_NKW(14) BGS_NKW(15) BGS_NKW(16)
#undef BGS_NKW
      default: break;
    }
    return cudaErrorInvalidValue;
  }
  switch (p.kw) {
#define BGS_KW(K) \
  case K: return launch_k12<K, R, CT>(p, grid, st);
    BGS_KW(1) BGS_KW(2) BGS_KW(3) BGS_KW(4) BGS_KW(5) BGS_KW(6) BGS_KW(7) BGS_KW(8)
    BGS_KW(9) BGS_KW(10) BGS_KW(11) BGS_KW(12) BGS_KW(13) BGS_KW(14) BGS_KW(15) BGS_KW(16)
#undef BGS_KW
#define BGS_KW1(K) \
  case K:          \
    if constexpr (R == 1) return launch_k12<K, R, CT>(p, grid, st); \
    break;
    BGS_KW1(17)
#undef BGS_KW1
    default: break;
  }
  return cudaErrorInvalidValue;
}

// clusters of 4: R = 1, KW 8..16 with their MTW (and the narrow variants)
template <bool CT>
static cudaError_t launch_quad(const SplitParams& p, int grid, cudaStream_t st) {
  if (p.R != 1) return cudaErrorInvalidValue;
  const bool narrow = p.mtw == mtw_for(p.kw, 1) - 1;
  switch (p.kw) {
#define BGS_KWQ(K)                                                                          \
  case K:                                                                                   \
    if constexpr (has_narrow(K, 1))                                                         \
      if (narrow) return launch_k12<K, 1, CT, mtw_for(K, 1) - 1, true>(p, grid, st);        \
    if (p.mtw == mtw_for(K, 1)) return launch_k12<K, 1, CT, mtw_for(K, 1), true>(p, grid, st); \
    break;
    BGS_KWQ(8) BGS_KWQ(9) BGS_KWQ(10) BGS_KWQ(11) BGS_KWQ(12) BGS_KWQ(13) BGS_KWQ(14) BGS_KWQ(15)
    BGS_KWQ(16)
#undef BGS_KWQ
    default: break;
  }
  return cudaErrorInvalidValue;
}

template <bool CT>
static cudaError_t launch_any(const SplitParams& p, int grid, cudaStream_t st) {
  if (p.cluster == 4) return launch_quad<CT>(p, grid, st);
  switch (p.R) {
    case 1: return launch_r<1, CT>(p, grid, st);
    case 2: return launch_r<2, CT>(p, grid, st);
    case 4: return launch_r<4, CT>(p, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace k12d
}  // namespace bgs
