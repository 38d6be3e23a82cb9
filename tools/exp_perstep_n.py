# Per-step fused-kernel time at a given shard size under forced K12c plans (BGS_K12C_PLAN):
#   python tools/exp_perstep_n.py 125000 [plans...]   -> table kp x plan (us)
import os, subprocess, sys
n = int(sys.argv[1]) if len(sys.argv) > 1 else 125000
plans = sys.argv[2:] or ["", "14", "12", "11", "22", "21"]
code = r'''
import os,sys
sys.path.insert(0,".")
import torch, paper_2507_21791_b200 as bgs
n,m,s=int(os.environ["NN"]),400,4
ld=(n+31)//32*32
ctx=bgs.Context(0)
X=torch.empty((m,ld),dtype=torch.float64,device="cuda"); Q=torch.zeros((m,ld),dtype=torch.float64,device="cuda")
bgs.gen_gaussian_device(ctx,12345,0,n,m,X.data_ptr(),ld)
v=int(bgs.parse_variant("BCGSI+P-1S"))
for rep in range(3):
    ctx.profile(True); bgs.factor_device(ctx,v,n,m,s,0,n,X.data_ptr(),ld,Q.data_ptr(),ld); prof=ctx.read_profile()
for k,d in prof.items():
    if k.startswith("fused_update_gram@"): print("ROW", int(k.split("kp")[1]), d["ms"]*1e3)
'''
res = {}
for pl in plans:
    env = dict(os.environ, BGS_PROF_STEP="1", NN=str(n))
    if pl:
        env["BGS_K12C_PLAN"] = pl
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout
    res[pl] = {int(l.split()[1]): float(l.split()[2]) for l in out.splitlines() if l.startswith("ROW")}
kps = sorted(res[plans[0]])
print("kp " + " ".join(f"{(p or 'dflt'):>7s}" for p in plans) + "   best")
tot = {p: 0.0 for p in plans}
best_tot = 0.0
for kp in kps:
    vals = [res[p].get(kp, float("nan")) for p in plans]
    for p, v in zip(plans, vals):
        tot[p] += v
    b = min(v for v in vals if v == v)
    best_tot += b
    if kp % 8 == 4:
        print(f"{kp:3d} " + " ".join(f"{v:7.1f}" for v in vals) + f"   {plans[vals.index(b)] or 'dflt'}")
print("sum " + " ".join(f"{tot[p]:7.0f}" for p in plans) + f"   best-of {best_tot:.0f}")
