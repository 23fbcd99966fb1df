D=gpurun_out/${1:-ncu}; mkdir -p $D
MCF_DIAG_OVERLAP=0 ncu --set full --import-source on --clock-control none -k regex:k_diag_unit --launch-skip ${2:-2} -c 1 -o $D/ncu_unit_c3 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/ncu.log 2>&1
