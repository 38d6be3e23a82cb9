# Per-phase cycle counters of the fused kernel (BGS_TILE_PROF=1) over ranges of the sweep.
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-verify"
for r in ${RANGES:-"4 56" "60 124" "128 240" "244 256" "260 288" "292 352" "356 392"}; do
  set -- $r
  echo "kp $1..$2"
  BGS_TILE_PROF=1 BGS_PROF_MINKP=$1 BGS_PROF_MAXKP=$2 $CMD 2>&1 | grep "k12c phases" | tail -1
done
