mkdir -p gpurun_out
C="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-verify"
for v in 0 1 2; do echo "skip=$v"; BGS_EXP_SKIP_SMALL=$v $C 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels']['fused_update_gram']['ms_total']/5)"; done
