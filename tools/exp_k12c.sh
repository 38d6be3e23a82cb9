# K12c vs single-CTA K12 on config 2: parity on the K12c path, phase counters, bench.
set -x
BGS_K12C=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
BGS_K12C=1 BGS_TILE_PROF=1 timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-verify 2>&1 | grep phases | tail -2
BGS_K12C=1 timeout 200 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('K12c ms/step', d['ms_per_step'], {k:(v['launches'], round(v['ms_total'],2)) for k,v in d['kernels'].items()}, d['verify'])"
