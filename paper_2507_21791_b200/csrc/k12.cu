// k12.cu — K12c host side: the planner (k12_plan) and the launch dispatch, plus the plain
// kernel instances.  The kernel itself is in k12_kernel.cuh; the compensated-tile
// instances (BCGSI+1S) are compiled separately in k12_ct.cu.
#include "k12_kernel.cuh"

namespace bgs {

using namespace k12d;

size_t k12_smem_bytes(int stages, int slot_units, int R, int C) {
  return 1024 + (size_t)stages * slot_units * R * kUnitChunkBytes + kRedBytes +
         (C >= 2 ? xchg_bytes(R, C) : 0) + (size_t)(2 * stages + 4) * sizeof(uint64_t);
}

// ------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------
namespace {
struct Cand {
  int C, R;
};
}  // namespace

bool k12_plan(SplitParams& p) {
  if (p.s < 1 || p.s > 4 || p.N < 1 || p.N > 8 || p.U0 < 1 || p.U1 < 1) return false;
  for (int j = 0; j < p.N; ++j)
    if (p.rcol1[j] < 0 || p.rcol1[j] >= 8 * p.U1) return false;
  const int na = p.upd_a ? p.U0 - p.kp / 8 : 0;  // units holding the A block (span-0 tail)
  if (na < 0 || na > p.U0) return false;
  p.s1_left = (p.lcols1 + 7) / 8;
  p.mt_out = p.U0 + p.s1_left;
  // C = 1 with the tallest stage that keeps >= 3 stages in shared memory, then the pair
  // (clusters of 4: prefixes too wide for a pair, e.g. m = 800 late in the sweep)
  const Cand cands[] = {{1, 4}, {1, 2}, {1, 1}, {2, 2}, {2, 1}, {4, 1}};
  // BGS_K12C_PLAN=CR (e.g. 21): only that candidate (tests / experiments; read per call)
  const char* fe = getenv("BGS_K12C_PLAN");
  const int forced = fe ? atoi(fe) : 0;
  for (const Cand& cd : cands) {
    if (forced && forced != 10 * cd.C + cd.R) continue;
    SplitParams q = p;
    q.cluster = cd.C;
    q.R = cd.R;
    int kmax = 0, mtmax = 0;  // most k-steps / output tiles of a rank
    for (int r = 0; r < 4; ++r) q.own_u0[r] = q.own_n[r] = q.ext_u0[r] = q.ext_n[r] = 0;
    if (cd.C == 1) {
      q.own_n[0] = p.U0;
      q.slot_units = p.U0 + p.U1;
      kmax = (p.kp + 3) / 4;
      mtmax = p.U0 + q.s1_left;
    } else {
      // the prefix-only units split evenly over the ranks (the first ranks take the
      // remainder); the last rank also owns the A-block units, the others load them as
      // extra units: every rank forms B = (srcB - Qp CB - A S2) TB^-1 and needs srcA
      const int nb = p.U0 - na;
      if (cd.C == 2) {  // (the split of round 1: ceil / floor)
        q.own_n[0] = (nb + 1) / 2;
        q.own_n[1] = p.U0 - q.own_n[0];
      } else {
        for (int r = 0; r < cd.C; ++r) q.own_n[r] = nb / cd.C + (r < nb % cd.C ? 1 : 0);
        q.own_n[cd.C - 1] += na;
      }
      int u = 0, units = 0;
      for (int r = 0; r < cd.C; ++r) {
        q.own_u0[r] = u;
        u += q.own_n[r];
        if (r < cd.C - 1) {
          q.ext_u0[r] = p.U0 - na;
          q.ext_n[r] = na;
        }
        units = std::max(units, q.own_n[r] + q.ext_n[r]);
        const int c1 = std::min(8 * (q.own_u0[r] + q.own_n[r]), p.kp), c0 = std::min(8 * q.own_u0[r], p.kp);
        kmax = std::max(kmax, (c1 - c0 + 3) / 4);
        mtmax = std::max(mtmax, q.own_n[r] + (r == 0 ? q.s1_left : 0));
      }
      q.slot_units = units + p.U1;
    }
    const int KS = 4 / cd.R;
    const int kw = (kmax + KS - 1) / KS;
    const int mtw = (mtmax + kGroupWarps - 1) / kGroupWarps;
    // one CTA at R = 1 carries up to kKwMaxR1 k-steps per warp while three stages fit
    // (BGS_K12C_KWMAX=16: the CTA pair takes those steps instead)
    const char* ke = getenv("BGS_K12C_KWMAX");
    const int kw_r1 = ke ? std::max(kKwMax, std::min(kKwMaxR1, atoi(ke))) : kKwMaxR1;
    const int kw_max = (cd.C == 1 && cd.R == 1) ? kw_r1 : kKwMax;
    int kw_t = std::max(cd.C == 4 ? 8 : 1, kw);  // (cluster-of-4 instances start at KW 8)
    while (kw_t <= kw_max && mtw_for(kw_t, cd.R) < mtw) ++kw_t;
    if (kw_t > kw_max) continue;
    const char* me = getenv("BGS_K12C_MINS");  // experiments: minimum ring depth (default 3)
    const int min_s = me ? std::max(2, atoi(me)) : 3;
    // Ring depth: deeper is not better.  Measured per step at config 2 (S = 2..8,
    // profiles/r01_stage_depth.log): the CTA-pair plans and the one-CTA R = 1 plans with
    // >= 6 output tiles per warp run 2-7% faster with 3 stages than with 4+; the taller
    // early stages (R = 2, 4) want 4.  BGS_K12C_MAXS overrides (experiments).
    const int depth = (cd.C >= 2 || (cd.R == 1 && mtw_for(kw_t, cd.R) >= 6)) ? 3 : 4;
    const char* xe = getenv("BGS_K12C_MAXS");
    const int max_s = std::max(min_s, xe ? std::min(kMaxStages, atoi(xe)) : depth);
    int S = 0;
    for (int st = max_s; st >= min_s; --st)
      if (k12_smem_bytes(st, q.slot_units, cd.R, cd.C) + kStaticSmem + 256 <= (size_t)kSmemOptin) {
        S = st;
        break;
      }
    if (!S) continue;
    q.kw = kw_t;
    q.mtw = mtw_for(kw_t, cd.R);
    // narrower instances (has_narrow): mtw_for(KW) carries one output tile per warp more
    // than the split needs at 1-5 steps of these KW (CTA pairs at s = 4: kp = 292..308 need
    // MTW 5 at KW 10, kp = 356..372 MTW 6 at KW 12, -5% each; one CTA: KW 16 would fold
    // every stage and spill at MTW 9 where 8 suffice)
    if (has_narrow(kw_t, cd.R) && mtw <= mtw_for(kw_t, cd.R) - 1) q.mtw = mtw_for(kw_t, cd.R) - 1;
    q.stages = S;
    p = q;
    static const bool verbose = getenv("BGS_K12C_VERBOSE") != nullptr;
    if (verbose)
      fprintf(stderr, "[k12c plan] kp %d U0 %d: C %d R %d KW %d (need %d) MTW %d (need %d) S %d slot %d units\n",
              p.kp, p.U0, p.cluster, p.R, p.kw, kw, p.mtw, mtw, p.stages, p.slot_units);
    return true;
  }
  return false;
}

// k12_ct.cu
cudaError_t k12_launch_ct(const SplitParams& p, int grid, cudaStream_t st);

int k12_grid_cap(int C, int sms) {
  if (C <= 2) return sms / C * C;
  // clusters of 4: ask the driver how many fit at once with a full-size CTA (every K12c
  // instance is one CTA per SM); a second wave of a few clusters would double the time
  static int cached[2] = {0, 0};
  int& c = cached[C == 4 ? 0 : 1];
  if (!c) {
    auto k = k12_kernel<13, mtw_for(13, 1), 1, false, true>;
    const size_t smem = (size_t)kSmemOptin - kStaticSmem - 256;
    int n = 0;
    if (ensure_smem(k, smem) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(sms / C * C));
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) n = 0;
      (void)cudaGetLastError();
    }
    c = n > 0 ? n : sms / C * 7 / 8;
  }
  return std::min(sms / C, c) * C;
}

cudaError_t k12_launch(const SplitParams& p, int grid, cudaStream_t st, int* launches) {
  if (grid < p.cluster || grid % p.cluster) return cudaErrorInvalidValue;
  if (launches) *launches += 1;
  if (p.comp_t0 < p.mt_out) return k12_launch_ct(p, grid, st);
  return launch_any<false>(p, grid, st);
}

}  // namespace bgs
