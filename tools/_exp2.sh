mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-verify"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_step4 -s 190 -c 1 -o gpurun_out/red_k90 $CMD > gpurun_out/ncu_red.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:reduce_step4 -s 99 -c 99 --csv --log-file gpurun_out/red_times.csv $CMD > gpurun_out/ncu_red2.log 2>&1
tail -3 gpurun_out/ncu_red.log
