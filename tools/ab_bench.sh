# Same-box A/B of whole-factorization device time (config 2) under env settings:
#   bash tools/ab_bench.sh "ENV_A=.." "ENV_B=.."   (each arm run 3x, alternating)
C="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-verify"
for rep in 1 2 3; do
  for arm in "$@"; do
    ms=$(env $arm $C 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "[$arm] rep $rep: $ms ms"
  done
done
