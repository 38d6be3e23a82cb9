# Device time of a factorization on one GPU under the three step transports: local (merged
# reduce + step), a one-rank peer context with the in-kernel wait (one launch / two
# launches), and the separate-launch exchange.  The exchange is an identity at P = 1; this
# measures what the per-step launch chain costs.   python tools/exp_peer_step.py 125000 1000000
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2507_21791_b200 as bgs
m, s = 400, 4
v = int(bgs.parse_variant("BCGSI+P-1S"))
for n in [int(a) for a in sys.argv[1:]] or [125000]:
    ld = (n + 31) // 32 * 32
    X = torch.empty((m, ld), dtype=torch.float64, device="cuda")
    Q = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    loc = bgs.Context(0)
    bgs.gen_gaussian_device(loc, 12345, 0, n, m, X.data_ptr(), ld)
    pc = bgs.Context(0, 0, 1, peer=True)
    pc.peer_attach([pc.peer_handle()], 2)
    def t(ctx, env):
        for k in ("BGS_NO_PEER_FUSE", "BGS_PEER_ONE", "BGS_GRAPH"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ts = []
        for _ in range(6):
            r, st, tm = bgs.factor_device(ctx, v, n, m, s, 0, n, X.data_ptr(), ld, Q.data_ptr(), ld)
            ts.append(tm.factor_ms)
        return sorted(ts)[len(ts) // 2], tm.kernel_launches
    rows = [("local, CUDA graph", loc, {}), ("local, plain launches", loc, {"BGS_GRAPH": "0"}),
            ("peer P=1: one launch per step", pc, {}), ("peer P=1: two launches per step", pc, {"BGS_PEER_ONE": "0"}),
            ("peer P=1: separate reduce/push/sum/step", pc, {"BGS_NO_PEER_FUSE": "1"})]
    for name, ctx, env in rows:
        ms, nl = t(ctx, env)
        print(f"n={n:8d} {name:42s} {ms:8.3f} ms  {nl} launches")
