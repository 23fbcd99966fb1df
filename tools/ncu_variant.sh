# ncu --set full of one k_diag_unit launch under a variant library: ncu_variant.sh TAG NAME [skip]
D=gpurun_out/$1; mkdir -p $D
MCFUNM_CUDA_LIB=$PWD/scratch/libs/$2.so ncu --set full --import-source on --clock-control none -k regex:k_diag_unit --launch-skip ${3:-6} -c 1 -o $D/ncu_$2 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/ncu_$2.log 2>&1
