# Same-box A/B of two library builds on the per-step fused-kernel times:
#   bash tools/ab_perstep.sh path/a.so path/b.so
for rep in 1 2; do
  for L in "$@"; do
    BGS_LIB_PATH=$(realpath $L) ALLSTEPS=1 timeout 300 python tools/exp_perstep.py > gpurun_out/ps_$(basename $L .so)_$rep.log 2>&1
    echo "$L rep $rep: $(tail -1 gpurun_out/ps_$(basename $L .so)_$rep.log)"
  done
done
