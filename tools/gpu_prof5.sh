D=gpurun_out/${1:-p5}; mkdir -p $D
MCF_DIAG_PROF=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/prof_c5.json 2> $D/prof_c5.err
