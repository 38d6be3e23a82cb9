# Same-box A/B of two library builds on the per-step fused-kernel times:
#   [TAG=x] bash tools/ab_perstep.sh path/a.so path/b.so     (logs: gpurun_out/ps_<lib><TAG>_<rep>.log)
for rep in 1 2; do
  for L in "$@"; do
    o=gpurun_out/ps_$(basename $L .so)${TAG}_$rep.log
    BGS_LIB_PATH=$(realpath $L) ALLSTEPS=1 timeout 300 python tools/exp_perstep.py > $o 2>&1
    echo "$L$TAG rep $rep: $(tail -1 $o)"
  done
done
