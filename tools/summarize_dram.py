# Summarise an ncu per-launch DRAM capture of the fused kernel (tools/collect_profiles.sh)
# against the algorithmic bytes of each block step of BCGSI+P-1S at config 2.
import collections, csv, json, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/k12c_dram_all.csv"
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]
idx = {n: i for i, n in enumerate(h)}
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[int(r[idx["ID"]])][r[idx["Metric Name"]]] = (float(r[idx["Metric Value"]].replace(",", "")),
                                                     r[idx["Metric Unit"]])
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "nsecond": 1, "us": 1e3,
      "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
ids = sorted(per)
tr = [per[i]["dram__bytes_read.sum"][0] * SC[per[i]["dram__bytes_read.sum"][1]] +
      per[i]["dram__bytes_write.sum"][0] * SC[per[i]["dram__bytes_write.sum"][1]] for i in ids]
dur = [per[i]["gpu__time_duration.sum"][0] * SC[per[i]["gpu__time_duration.sum"][1]] for i in ids]
n, s = 1_000_000, 4
alg = [8 * n * 16] + [8 * n * s * (k + 5) for k in range(1, len(ids))]
out = {"kernel": "k12_kernel (fused_update_gram)", "launches": len(ids),
       "traffic_bytes_per_launch": sum(tr) / len(tr), "alg_bytes_per_launch": sum(alg) / len(alg),
       "traffic_over_alg": sum(tr) / sum(alg), "ncu_total_ms": sum(dur) / 1e6,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (one factorization, "
                 "config 2, cold cache, serialised)"}
print(json.dumps(out, indent=1))
