# Mean per-phase cycles of the fused kernel's CTA 0 (BGS_TILE_PROF timeline) at chosen prefix
# widths: python tools/timeline_summary.py 20 100 244 324 [n]
import os, re, subprocess, sys
kps = [int(a) for a in sys.argv[1:] if int(a) <= 4096] or [20, 100, 244, 324]
names = ["wait", "update", "exchange", "epilogue", "gram", "tail"]
for kp in kps:
    env = dict(os.environ, BGS_TILE_PROF="1", BGS_PROF_MINKP=str(kp), BGS_PROF_MAXKP=str(kp),
               BGS_TIMELINE="1")
    extra = ["--m", os.environ["M"]] if os.environ.get("M") else []
    out = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "1", "--no-cpu",
                          "--no-e2e", "--no-verify"] + extra, env=env, capture_output=True, text=True)
    rows = {}
    for l in out.stderr.splitlines():
        m = re.match(r"\[k12c timeline\] g (\d) j +(\d+): (.*)", l)
        if m:
            rows[(int(m.group(1)), int(m.group(2)))] = [int(x) for x in m.group(3).split()]
    tot = [0.0] * 6
    cnt = 0
    for (g, j), t in rows.items():
        nxt = rows.get((g, j + 1))
        if j < 4 or nxt is None:
            continue
        d = [t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4], nxt[0] - t[5]]
        tot = [a + b for a, b in zip(tot, d)]
        cnt += 1
    ph = [l for l in out.stderr.splitlines() if "k12c phases" in l]
    if cnt:
        print(f"kp {kp}: " + " ".join(f"{n} {v / cnt:.0f}" for n, v in zip(names, tot)) +
              f" | period {sum(tot) / cnt:.0f} ({cnt} group-stages of CTA 0)")
    if ph:
        print("   ", ph[-1])
