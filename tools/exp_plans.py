# Per-step plan sweep of the fused kernel at config 2: for every block step, the device time
# of each K12c candidate plan (BGS_K12C_PLAN=CR, BGS_K12C_MINS=ring depth), next to the
# default plan, to see where the plan heuristic leaves time on the table.
#   python tools/exp_plans.py            (one B200)
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json
sys.path.insert(0, ".")
os.environ["BGS_PROF_STEP"] = "1"
import torch
import paper_2507_21791_b200 as bgs
n, m, s = int(os.environ.get("N", 1000000)), int(os.environ.get("M", 400)), int(os.environ.get("S", 4))
ld = (n + 31) // 32 * 32
ctx = bgs.Context(0)
X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
Q = torch.empty((m, ld), dtype=torch.float64, device="cuda")
bgs.gen_gaussian_device(ctx, 12345, 0, n, m, X.data_ptr(), ld)
v = int(bgs.parse_variant(os.environ.get("VARIANT", "BCGSI+P-1S")))
best = {}
for rep in range(3):
    ctx.profile(True)
    bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
    prof = ctx.read_profile()
    for k, d in prof.items():
        if k.startswith("fused_update_gram@"):
            kp = int(k.split("kp")[1])
            t = d["ms"] / d["launches"]
            best[kp] = min(best.get(kp, 1e9), t)
print("JSON" + json.dumps(best))
'''


def run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                       timeout=600)
    for line in r.stdout.splitlines():
        if line.startswith("JSON"):
            return {int(k): v for k, v in json.loads(line[4:]).items()}
    print("FAILED", env_extra, r.stderr[-2000:], file=sys.stderr)
    return {}


def main():
    plans = [("default", {})]
    for p in ["14", "12", "11", "22", "21"]:
        plans.append((p, {"BGS_K12C_PLAN": p}))
    for p in ["12", "11", "22", "21"]:
        plans.append((p + "s2", {"BGS_K12C_PLAN": p, "BGS_K12C_MINS": "2"}))
    extra = os.environ.get("EXTRA_PLANS")  # e.g. "name:VAR=1,VAR2=3;..."
    if extra:
        for item in extra.split(";"):
            name, kv = item.split(":")
            plans.append((name, dict(x.split("=") for x in kv.split(","))))
    res = {}
    for name, env in plans:
        res[name] = run(env)
    kps = sorted(res["default"])
    names = [n for n, _ in plans]
    print("kp    " + " ".join(f"{n:>8}" for n in names) + "   best")
    tot_def = tot_best = 0.0
    for kp in kps:
        row = [res[n].get(kp) for n in names]
        vals = [(v, n) for v, n in zip(row, names) if v is not None]
        b, bn = min(vals)
        tot_def += res["default"][kp]
        tot_best += b
        print(f"{kp:4d}  " + " ".join(f"{v*1e3:8.1f}" if v is not None else "       -" for v in row)
              + f"   {bn}")
    print(f"total default {tot_def:.3f} ms, per-step best {tot_best:.3f} ms")
    json.dump(res, open("gpurun_out/plans.json", "w"))


if __name__ == "__main__":
    main()
