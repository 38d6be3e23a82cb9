# Round-2 (same recipe as round 1) measurement set (B200_PROFILING.md recipe), all on one GPU:
#  1. plain bench line (the number), 2. per-launch device times of one factorization
#  (ncu launch list, cold-cache and serialised: compare shares), 3. per-launch DRAM bytes
#  of every fused-kernel launch of one factorization, 4. --set full captures of the fused
#  kernel late in the sweep (CTA-pair plan) and of the merged reduce + step kernel.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_final.log 2>&1
tail -1 gpurun_out/r02_bench_final.log > gpurun_out/r02_bench_final.json
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-verify"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 330 -c 320 \
    --csv --log-file gpurun_out/r02_launches_final.csv $CMD > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k12_kernel -s 99 -c 99 --csv \
    --log-file gpurun_out/r02_k12c_dram_all.csv $CMD > gpurun_out/ncu_dram.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k12_kernel \
    -s 180 -c 1 -o gpurun_out/r02_k12c_k81 $CMD > gpurun_out/ncu_full_k81.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_step4 \
    -s 180 -c 1 -o gpurun_out/r02_reduce_step_k81 $CMD > gpurun_out/ncu_full_red.log 2>&1
ls -la gpurun_out | tail -12
