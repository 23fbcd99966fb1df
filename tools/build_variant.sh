#!/bin/bash
# build_variant.sh NAME -DFLAG=... : libmcfunm_cuda.so with mcf_diag.cu compiled under extra flags -> scratch/libs/NAME.so
# (run a variant with MCFUNM_CUDA_LIB=scratch/libs/NAME.so)
set -e
cd "$(dirname "$0")/../paper_2308_01037_b200/csrc"
name=$1; shift
make -s -j8 >/dev/null
mkdir -p ../../scratch/libs/obj_$name
NVF="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v --expt-relaxed-constexpr"
nvcc $NVF "$@" -dc mcf_diag.cu -o ../../scratch/libs/obj_$name/mcf_diag.o 2> ../../scratch/libs/obj_$name/ptxas.log
objs=""
for f in mcf_util mcf_graph mcf_alloc mcf_walk mcf_gen mcf_capi; do objs="$objs ../lib/obj/$f.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../scratch/libs/$name.so $objs ../../scratch/libs/obj_$name/mcf_diag.o -cudart static -Xcompiler -fPIC
grep -A1 "k_diag_unitILi1024" ../../scratch/libs/obj_$name/ptxas.log | grep -o "Used [0-9]* registers.*" | head -2
grep -B2 -A3 "k_diag_unitILi1024" ../../scratch/libs/obj_$name/ptxas.log | grep -o "[0-9]* bytes spill stores" | head -1
