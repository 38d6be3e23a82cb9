# Per-step fused-kernel time at n = 1e6 for a given m (BGS_PROF_STEP): python tools/exp_perstep_m.py 800
import os, sys
sys.path.insert(0, ".")
os.environ["BGS_PROF_STEP"] = "1"
import torch
import paper_2507_21791_b200 as bgs
n, m, s = 1_000_000, int(sys.argv[1]) if len(sys.argv) > 1 else 800, 4
ld = (n + 31) // 32 * 32
ctx = bgs.Context(0)
X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
Q = torch.empty((m, ld), dtype=torch.float64, device="cuda")
bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
v = int(bgs.parse_variant("BCGSI+P-1S"))
for rep in range(2):
    ctx.profile(True)
    bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
    prof = ctx.read_profile()
rows = sorted((int(k.split("kp")[1]), d) for k, d in prof.items() if k.startswith("fused_update_gram@"))
tot = 0.0
for kp, d in rows:
    tot += d["ms"]
    if kp % 40 == 0 or kp > m - 16:
        print(f"kp {kp:4d}  ms {d['ms']/d['launches']:.4f}  GB/s {d['alg_bytes']/d['ms']/1e6:7.1f}")
print("fused total ms", round(tot, 3), "launches", sum(d["launches"] for _, d in rows))
for k, d in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    if not k.startswith("fused_update_gram@"):
        print(f"   {k:24s} {d['ms']:8.3f} ms  {d['launches']:4d} launches")
