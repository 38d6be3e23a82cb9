# Bisect the fused K12 kernel: time one factorization with parts disabled (BGS_TILE_DBG).
for d in ${DBGS:-0 2 16 4}; do
  echo "dbg=$d $(BGS_TILE_DBG=$d python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c 'import json,sys; l=[x for x in sys.stdin if x.startswith("{")]; d=json.loads(l[-1]) if l else None; k=d["kernels"].get("fused_update_gram",{}) if d else {}; print((round(d["ms_per_step"],2), "ms; fused", round(k.get("ms_total",0)/3,2), "ms", round(k.get("gbs") or 0), "GB/s") if d else "failed")')"
done
