# Re-run one fuzzer case through bgs_factor_device on a one-rank NCCL context (FUZZ_NCCL's path)
# under several switches: python tools/repro_case_dev.py v n m s kappa gauss seed
import os, subprocess, sys
args = sys.argv[1:8]
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_21791_b200 as bgs
from oracle.oracle import Oracle
v, n, m, s = (int(a) for a in sys.argv[1:5]); kappa = float(sys.argv[5]); gauss = sys.argv[6] == "True"; seed = int(sys.argv[7])
o = Oracle()
x = o.gen_matrix(n, m, s, kappa, seed, gauss)
ref = o.factor(v, x, s, 1, metrics=True)
import os
ctx = bgs.Context(0, 0, 1, bgs.nccl_unique_id()) if os.environ.get("CTX", "nccl") == "nccl" else bgs.Context(0)
ld = (n + 31) // 32 * 32
for rep in range(3):
    X = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    X[:, :n] = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(x).T)).cuda()
    Q = torch.full((m, ld), float(os.environ.get("QFILL", "0")), dtype=torch.float64, device="cuda")
    try:
        r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
        q = np.asfortranarray(Q[:, :n].cpu().numpy().T)
        print("rep", rep, "ok cond %.1e loo %.2e (oracle %.2e) dR %.1e" % (np.linalg.cond(x), o.loo(q), ref.loo, np.abs(r - ref.r).max() / np.abs(ref.r).max()))
    except Exception as e:
        print("rep", rep, "EXC", str(e)[:100])
'''
for name, env in [("nccl ctx", {}), ("local ctx", {"CTX": "local"}), ("nccl BGS_K2M=0", {"BGS_K2M": "0"}), ("nccl BGS_GRAPH=0", {"BGS_GRAPH": "0"}),
                  ("nccl Q=nan", {"QFILL": "nan"}), ("nccl BGS_POISON=1", {"BGS_POISON": "1"}), ("nccl BGS_DEBUG_STATUS=1", {"BGS_DEBUG_STATUS": "1"})]:
    out = subprocess.run([sys.executable, "-c", code] + args, env=dict(os.environ, **env), capture_output=True, text=True)
    print(f"--- {name}\n" + (out.stdout.strip() or out.stderr.strip()[-400:]))
