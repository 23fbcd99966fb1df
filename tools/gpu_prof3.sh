D=gpurun_out/${1:-p3}; mkdir -p $D
MCF_DIAG_PROF=1 timeout 600 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/prof_c3.json 2> $D/prof_c3.err
