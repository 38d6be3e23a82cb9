# Per-block-step device time of the fused update+Gram kernel at config 2 (BGS_PROF_STEP=1):
# ms per launch and algorithmic GB/s, to see which part of the sweep is off the roofline.
import os, sys
sys.path.insert(0, ".")
os.environ["BGS_PROF_STEP"] = "1"
import torch
import paper_2507_21791_b200 as bgs
n, m, s = 1_000_000, 400, 4
ld = (n + 31) // 32 * 32
ctx = bgs.Context(0)
X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
Q = torch.empty((m, ld), dtype=torch.float64, device="cuda")
bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
v = int(bgs.parse_variant(os.environ.get("VARIANT", "BCGSI+P-1S")))
for rep in range(2):
    ctx.profile(True)
    bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
    prof = ctx.read_profile()
rows = sorted((k, d) for k, d in prof.items() if k.startswith("fused_update_gram@"))
tot = 0.0
for k, d in rows:
    tot += d["ms"]
    kp = int(k.split("kp")[1])
    if os.environ.get("ALLSTEPS") or kp % 20 == 0 or kp <= 12 or kp >= 388:
        print(f"kp {kp:4d}  ms {d['ms']/d['launches']:.4f}  GB/s {d['alg_bytes']/d['ms']/1e6:7.1f}")
print("fused total ms", round(tot, 3), "launches", sum(d["launches"] for _, d in rows))
