"""CPU numerics study for the BCGSI+1S LOO gap.

A numpy/loop restatement of onesync_impl in SkipNorm mode (bcgs.cpp:233-369) whose
primitives can be swapped one at a time, run over many seeds of the failing shape class
(n=49, m=12, s=4, geometric kappa ~1e3).  The geometric-mean LOO of each configuration,
against the all-reference configuration, shows which rounding choice moves LOO.
Test infrastructure only (imports oracle/).
    python tools/numerics_study.py [seeds]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle.oracle import Oracle  # noqa: E402

o = Oracle()


def chol(a):
    n = a.shape[0]
    s = 0.5 * (a + a.T)
    g = np.zeros((n, n))
    for j in range(n):
        for i in range(j + 1):
            acc = s[i, j]
            for k in range(i):
                acc -= g[k, i] * g[k, j]
            if i == j:
                if not acc > 0:
                    raise ValueError("notspd")
                g[j, j] = np.sqrt(acc)
            else:
                g[i, j] = acc / g[i, i]
    return g


def at_b(a, b):  # multiply_at_b, sequential
    out = np.zeros((a.shape[1], b.shape[1]))
    for i in range(a.shape[1]):
        for j in range(b.shape[1]):
            acc = 0.0
            for k in range(a.shape[0]):
                acc += a[k, i] * b[k, j]
            out[i, j] = acc
    return out


def tri_left_trans(g, b):
    n = g.shape[0]
    w = np.zeros_like(b)
    for i in range(n):
        for j in range(b.shape[1]):
            acc = b[i, j]
            for k in range(i):
                acc -= g[k, i] * w[k, j]
            w[i, j] = acc / g[i, i]
    return w


def solve_subst(b, g):  # tri_solve_right, back-substitution by division
    n = g.shape[0]
    w = np.zeros_like(b)
    for j in range(n):
        acc = b[:, j].copy()
        for k in range(j):
            acc = acc - w[:, k] * g[k, j]
        w[:, j] = acc / g[j, j]
    return w


def solve_recip(b, g):  # substitution, multiply by the reciprocal diagonal
    n = g.shape[0]
    w = np.zeros_like(b)
    for j in range(n):
        acc = b[:, j].copy()
        for k in range(j):
            acc = acc - w[:, k] * g[k, j]
        w[:, j] = acc * (1.0 / g[j, j])
    return w


def tri_inv(g):  # upper-triangular inverse, column by column (by division)
    n = g.shape[0]
    inv = np.zeros((n, n))
    for j in range(n):
        inv[j, j] = 1.0 / g[j, j]
        for i in range(j - 1, -1, -1):
            acc = 0.0
            for k in range(i + 1, j + 1):
                acc += g[i, k] * inv[k, j]
            inv[i, j] = -acc / g[i, i]
    return inv


def solve_inv(b, g):  # explicit inverse, row times inverse (fp64 dot)
    inv = tri_inv(g)
    n = g.shape[0]
    w = np.zeros_like(b)
    for j in range(n):
        acc = np.zeros(b.shape[0])
        for k in range(j + 1):
            acc = acc + b[:, k] * inv[k, j]
        w[:, j] = acc
    return w


def gram_exact(a, b):
    return o.gram(a, b)


def gram_seq(a, b):
    return at_b(a, b)


def gram_chunk(a, b, chunk=4, chains=4):
    """DMMA-like: 4-row FMA groups, `chains` independent accumulators, summed at the end."""
    n = a.shape[0]
    acc = [np.zeros((a.shape[1], b.shape[1])) for _ in range(chains)]
    for c, r0 in enumerate(range(0, n, chunk)):
        blk = acc[c % chains]
        for r in range(r0, min(n, r0 + chunk)):
            blk += np.outer(a[r], b[r])
    out = acc[0]
    for t in acc[1:]:
        out = out + t
    return out


def gram_dd4(a, b, chunk=4):
    """fp64 4-row chunks, each chunk folded into a double-double (exact-ish sum of chunk
    results): only the 4-term products round."""
    n = a.shape[0]
    hi = np.zeros((a.shape[1], b.shape[1])); lo = np.zeros_like(hi)
    for r0 in range(0, n, chunk):
        c = np.zeros_like(hi)
        for r in range(r0, min(n, r0 + chunk)):
            c += np.outer(a[r], b[r])
        s = hi + c; bb = s - hi; e = (hi - (s - bb)) + (c - bb)
        hi = s; lo = lo + e
    return hi + lo


def split_gram(kp_of, g_prefix, g_tail):
    """Gram with the prefix-row block (Q^T .) from g_prefix and the rest from g_tail."""
    def g(a, b):
        kp = kp_of(a, b)
        out = g_tail(a, b)
        if kp:
            out[:kp] = g_prefix(a[:, :kp], b)
        return out
    return g


def gram_tp(a, b):
    """Exact products (two-prod via Dekker split) summed in double-double."""
    import math
    hi = np.zeros((a.shape[1], b.shape[1])); lo = np.zeros_like(hi)
    for r in range(a.shape[0]):
        p = np.outer(a[r], b[r])
        # exact error of the product: use fractions-free fma emulation via splitting
        sp = 134217729.0
        def split(v):
            t = sp * v; h = t - (t - v); return h, v - h
        ah, al = split(a[r][:, None] + 0 * b[r][None, :])
        bh, bl = split(b[r][None, :] + 0 * a[r][:, None])
        e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
        for t in (p, e):
            s = hi + t; bb = s - hi; err = (hi - (s - bb)) + (t - bb)
            hi = s; lo = lo + err
    return hi + lo


TAIL = lambda a, b: a.shape[1] - b.shape[1] if a.shape[1] > b.shape[1] else 0


def axpy(q, c):  # y -= (Q c), the sum formed first (local_axpy_block)
    out = np.zeros((q.shape[0], c.shape[1]))
    for k in range(c.shape[0]):
        out += np.outer(q[:, k], c[k])
    return out


def axpy_perm(q, c):  # same sum in a different order (reverse)
    out = np.zeros((q.shape[0], c.shape[1]))
    for k in reversed(range(c.shape[0])):
        out += np.outer(q[:, k], c[k])
    return out


def ip1s(x, s, gram, solve, ax=axpy):
    n, m = x.shape
    qb = m // s
    Q = np.zeros((n, m))
    q0, r00 = o.householder(x[:, :s])
    Q[:, :s] = q0
    scol = tri_left_trans(r00, gram(x[:, :s], x[:, s:2 * s]))
    U = x[:, s:2 * s] - ax(Q[:, :s], scol)
    for k in range(1, qb):
        kp = k * s
        nxt = k + 1 < qb
        left = np.hstack([Q[:, :kp], U])
        right = np.hstack([U, x[:, kp + s:kp + 2 * s]]) if nxt else U
        G = gram(left, right)
        Y, Om = G[:kp, :s], G[kp:kp + s, :s]
        yd = chol(Om - at_b(Y, Y))
        Q[:, kp:kp + s] = solve(U - ax(Q[:, :kp], Y), yd)
        if not nxt:
            break
        Z, Pm = G[:kp, s:2 * s], G[kp:kp + s, s:2 * s]
        s2 = tri_left_trans(yd, Pm - at_b(Y, Z))
        scol = np.vstack([Z, s2])
        U = x[:, kp + s:kp + 2 * s] - ax(Q[:, :kp + s], scol)
    return Q


def ip1s_fused(x, s, gram, ax=axpy_perm):
    """The K12c path: A = za TA^-1 and B = zb - za (TA^-1 S2) through one 8x8 matrix M
    (k12.cu epilogue), za = U - Qp Y, zb = X_{k+1} - Qp Z over the prefix only."""
    n, m = x.shape
    qb = m // s
    Q = np.zeros((n, m))
    q0, r00 = o.householder(x[:, :s])
    Q[:, :s] = q0
    scol = tri_left_trans(r00, gram(x[:, :s], x[:, s:2 * s]))
    U = x[:, s:2 * s] - ax(Q[:, :s], scol)
    for k in range(1, qb):
        kp = k * s
        nxt = k + 1 < qb
        left = np.hstack([Q[:, :kp], U])
        right = np.hstack([U, x[:, kp + s:kp + 2 * s]]) if nxt else U
        G = gram(left, right)
        Y, Om = G[:kp, :s], G[kp:kp + s, :s]
        yd = chol(Om - at_b(Y, Y))
        za = U - ax(Q[:, :kp], Y)
        ti = tri_inv(yd)
        if not nxt:
            Q[:, kp:kp + s] = za @ ti
            break
        Z, Pm = G[:kp, s:2 * s], G[kp:kp + s, s:2 * s]
        s2 = tri_left_trans(yd, Pm - at_b(Y, Z))
        zb = x[:, kp + s:kp + 2 * s] - ax(Q[:, :kp], Z)
        mab = -(ti @ s2)
        Aout = np.zeros((n, s)); Bout = np.zeros((n, s))
        for j in range(s):
            acc = np.zeros(n)
            for l in range(s):
                acc = acc + za[:, l] * ti[l, j]
            Aout[:, j] = acc
            acc = np.zeros(n)
            for l in range(s):
                acc = acc + za[:, l] * mab[l, j]
            Bout[:, j] = acc + zb[:, j]
        Q[:, kp:kp + s] = Aout
        U = Bout
    return Q


CONFIGS = {
    "ref (exact gram, subst)": (gram_exact, solve_subst, axpy),
    "recip-diag subst": (gram_exact, solve_recip, axpy),
    "explicit inverse": (gram_exact, solve_inv, axpy),
    "fp64 seq gram": (gram_seq, solve_subst, axpy),
    "fp64 chunk gram": (gram_chunk, solve_subst, axpy),
    "axpy reversed": (gram_exact, solve_subst, axpy_perm),
    "chunk gram + inverse": (gram_chunk, solve_inv, axpy),
    "GPU-like: chunk Q rows, tp U rows, rev axpy, inv": (split_gram(TAIL, gram_chunk, gram_tp), solve_inv, axpy_perm),
    "GPU-like: chunk Q rows, dd4 U rows, rev axpy, inv": (split_gram(TAIL, gram_chunk, gram_dd4), solve_inv, axpy_perm),
    "K12c epilogue, exact gram": (gram_exact, "fused", None),
    "K12c epilogue, chunk gram": (gram_chunk, "fused", None),
    "K12c epilogue, chunk Q + dd4 U": (split_gram(TAIL, gram_chunk, gram_dd4), "fused", None),
    "fp64 Q rows, two-prod U rows": (split_gram(TAIL, gram_chunk, gram_tp), solve_subst, axpy),
    "fp64 Q rows, dd4 U rows": (split_gram(TAIL, gram_chunk, gram_dd4), solve_subst, axpy),
    "fp64 Q rows, dd8 U rows": (split_gram(TAIL, gram_chunk, lambda a, b: gram_dd4(a, b, 8)), solve_subst, axpy),
    "fp64 Q rows, dd16 U rows": (split_gram(TAIL, gram_chunk, lambda a, b: gram_dd4(a, b, 16)), solve_subst, axpy),
    "dd-fold every 4 rows": (gram_dd4, solve_subst, axpy),
    "exact Q^T rows, fp64 U rows": (split_gram(lambda a, b: a.shape[1] - b.shape[1] if a.shape[1] > b.shape[1] else 0, gram_exact, gram_chunk), solve_subst, axpy),
    "fp64 Q^T rows, exact U rows": (split_gram(lambda a, b: a.shape[1] - b.shape[1] if a.shape[1] > b.shape[1] else 0, gram_chunk, gram_exact), solve_subst, axpy),
}


ENVELOPE = False


def main():
    global ENVELOPE
    nseeds = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    ENVELOPE = len(sys.argv) > 2 and sys.argv[2] == "envelope"
    n, m, s, kappa = 49, 12, 4, 1280.7671752796468
    rng = np.random.default_rng(7)
    logs = {k: [] for k in CONFIGS}
    orl = []
    seeds = [343794 + i for i in range(6)] + [int(t) for t in rng.integers(1, 10 ** 6, nseeds - 6)]
    for seed in seeds:
        x = o.gen_matrix(n, m, s, kappa, seed, False)
        ref = o.factor(5, x, s, 1, metrics=True)
        if ref.rc:
            continue
        if ENVELOPE:
            ref.loo = max([ref.loo] + [o.factor(5, x, s, P, metrics=True).loo for P in (2, 3, 4)])
        orl.append(np.log10(ref.loo))
        for name, (g, sv, ax) in CONFIGS.items():
            try:
                qq = ip1s_fused(x, s, g) if sv == "fused" else ip1s(x, s, g, sv, ax)
                logs[name].append(np.log10(o.loo(qq)))
            except ValueError:
                logs[name].append(np.nan)
    orl = np.array(orl)
    for name, v in logs.items():
        print(f"{name:28s} first 6 seeds ratio: " + " ".join("%.1f" % 10 ** (a - b) for a, b in zip(v[:6], orl[:6])))
    print(f"{len(orl)} seeds, n={n} m={m} s={s} kappa={kappa:.0f}; oracle geomean LOO "
          f"{10 ** orl.mean():.2e}")
    for name, v in logs.items():
        v = np.array(v)
        d = v - orl
        print(f"{name:28s} geomean {10 ** np.nanmean(v):.2e}  ratio vs oracle: geomean "
              f"{10 ** np.nanmean(d):5.2f}  max {10 ** np.nanmax(d):6.2f}  "
              f">10x: {int(np.sum(d > 1))}")


if __name__ == "__main__":
    main()
