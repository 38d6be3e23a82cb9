// k12.cu — K12c host side: the planner (k12_plan) and the launch dispatch, plus the plain
// kernel instances.  The kernel itself is in k12_kernel.cuh; the compensated-tile
// instances (BCGSI+1S) are compiled separately in k12_ct.cu.
#include "k12_kernel.cuh"

namespace bgs {

using namespace k12d;

size_t k12_smem_bytes(int stages, int slot_units, int R, int C) {
  return 1024 + (size_t)stages * slot_units * R * kUnitChunkBytes + kRedBytes +
         (C == 2 ? xchg_bytes(R) : 0) + (size_t)(2 * stages + 4) * sizeof(uint64_t);
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
  const Cand cands[] = {{1, 4}, {1, 2}, {1, 1}, {2, 2}, {2, 1}};
  // BGS_K12C_PLAN=CR (e.g. 21): only that candidate (tests / experiments; read per call)
  const char* fe = getenv("BGS_K12C_PLAN");
  const int forced = fe ? atoi(fe) : 0;
  for (const Cand& cd : cands) {
    if (forced && forced != 10 * cd.C + cd.R) continue;
    SplitParams q = p;
    q.cluster = cd.C;
    q.R = cd.R;
    int k0, k1 = 0, mt0, mt1 = 0;
    if (cd.C == 1) {
      q.own_u0[0] = 0; q.own_n[0] = p.U0; q.ext_u0[0] = 0; q.ext_n[0] = 0;
      q.own_u0[1] = q.own_n[1] = q.ext_u0[1] = q.ext_n[1] = 0;
      q.slot_units = p.U0 + p.U1;
      k0 = (p.kp + 3) / 4;
      mt0 = p.U0 + q.s1_left;
    } else {
      const int uh = (p.U0 - na + 1) / 2;
      q.own_u0[0] = 0;         q.own_n[0] = uh;
      q.ext_u0[0] = p.U0 - na; q.ext_n[0] = na;
      q.own_u0[1] = uh;        q.own_n[1] = p.U0 - uh;
      q.ext_u0[1] = 0;         q.ext_n[1] = 0;
      q.slot_units = std::max(uh + na, p.U0 - uh) + p.U1;
      const int c0 = std::min(8 * uh, p.kp), c1 = std::max(0, p.kp - 8 * uh);
      k0 = (c0 + 3) / 4;
      k1 = (c1 + 3) / 4;
      mt0 = uh + q.s1_left;
      mt1 = p.U0 - uh;
    }
    const int KS = 4 / cd.R;
    const int kw = (std::max(k0, k1) + KS - 1) / KS;
    const int mtw = (std::max(mt0, mt1) + kGroupWarps - 1) / kGroupWarps;
    // one CTA at R = 1 carries up to kKwMaxR1 k-steps per warp while three stages fit
    // (BGS_K12C_KWMAX=16: the CTA pair takes those steps instead)
    const char* ke = getenv("BGS_K12C_KWMAX");
    const int kw_r1 = ke ? std::max(kKwMax, std::min(kKwMaxR1, atoi(ke))) : kKwMaxR1;
    const int kw_max = (cd.C == 1 && cd.R == 1) ? kw_r1 : kKwMax;
    int kw_t = std::max(1, kw);
    while (kw_t <= kw_max && mtw_for(kw_t, cd.R) < mtw) ++kw_t;
    if (kw_t > kw_max) continue;
    const char* me = getenv("BGS_K12C_MINS");  // experiments: minimum ring depth (default 3)
    const int min_s = me ? std::max(2, atoi(me)) : 3;
    // Ring depth: deeper is not better.  Measured per step at config 2 (S = 2..8,
    // profiles/r01_stage_depth.log): the CTA-pair plans and the one-CTA R = 1 plans with
    // >= 6 output tiles per warp run 2-7% faster with 3 stages than with 4+; the taller
    // early stages (R = 2, 4) want 4.  BGS_K12C_MAXS overrides (experiments).
    const int depth = (cd.C == 2 || (cd.R == 1 && mtw_for(kw_t, cd.R) >= 6)) ? 3 : 4;
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

cudaError_t k12_launch(const SplitParams& p, int grid, cudaStream_t st, int* launches) {
  if (grid < p.cluster || grid % p.cluster) return cudaErrorInvalidValue;
  if (launches) *launches += 1;
  if (p.comp_t0 < p.mt_out) return k12_launch_ct(p, grid, st);
  return launch_any<false>(p, grid, st);
}

}  // namespace bgs
