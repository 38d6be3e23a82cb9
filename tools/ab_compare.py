# Compare two per-step logs pairs from tools/ab_perstep.sh:  python tools/ab_compare.py a b [thr%]
import re, sys
def load(f):
    d = {}
    for l in open(f):
        m = re.match(r'kp\s+(\d+)\s+ms\s+([\d.]+)', l)
        if m: d[int(m.group(1))] = float(m.group(2))
    return d
def best(tag):
    xs = [load(f'gpurun_out/ps_{tag}_{i}.log') for i in (1, 2)]
    return {k: min(x[k] for x in xs) for k in xs[0]}
A, B = best(sys.argv[1]), best(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
for kp in sorted(A):
    d = (B[kp] - A[kp]) / A[kp] * 100
    if abs(d) >= thr: print(f"{kp:4d} {A[kp]*1e3:7.1f} {B[kp]*1e3:7.1f} {d:+5.1f}%", end=" | ")
print(f"\ntotal {sum(A.values()):.3f} -> {sum(B.values()):.3f}")
