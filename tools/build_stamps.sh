# Debug library with %globaltimer stamps of the reduce + step kernel and the fused kernel's
# start (-DBGS_STEP_STAMPS) -> paper_2507_21791_b200/_lib_exp/st.so; run tools/stamp_run.py
# with BGS_LIB_PATH pointing at it.
set -e
cd "$(dirname "$0")/../paper_2507_21791_b200"
make -s
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include -DBGS_STEP_STAMPS"
mkdir -p _lib_exp
nvcc $F -c csrc/small.cu -o _build/small_st.o &
nvcc $F -c csrc/k12.cu -o _build/k12_st.o
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _lib_exp/st.so _build/gram.o _build/gram_ct.o \
  _build/k12_st.o _build/k12_ct.o _build/update.o _build/update_tma.o _build/small_st.o _build/tsqr.o _build/misc.o _build/peer.o \
  _build/runtime.o _build/matgen_host.o -ldl
