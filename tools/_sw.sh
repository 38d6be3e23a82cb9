L=paper_2507_21791_b200/_lib/libbgs_gpu.so
for S in 2 3 4 5 6 8; do
  if [ $S = 2 ]; then export BGS_K12C_MINS=2; else unset BGS_K12C_MINS; fi
  BGS_K12C_MAXS=$S ALLSTEPS=1 timeout 300 python tools/exp_perstep.py > gpurun_out/ps_S${S}.log 2>&1
  echo "S=$S $(tail -1 gpurun_out/ps_S${S}.log)"
done
