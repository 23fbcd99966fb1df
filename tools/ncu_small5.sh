D=gpurun_out/${1:-ns5}; mkdir -p $D
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_diag_unit<.int.256" --launch-skip 10 -c 1 -o $D/ncu_small_c5 python bench.py --config 5 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/ncu.log 2>&1
