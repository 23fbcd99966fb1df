# config-3 combine diagnostics: counters + timeline, launch list
set -x
D=gpurun_out/r02b; mkdir -p $D
MCF_DIAG_PROF=1 timeout 600 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/prof_c3.json 2> $D/prof_c3.err
timeout 900 bash tools/ncu_times.sh "." $D/launches_config3.csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/launches_config3_summary.txt 2>&1
MCF_DIAG_PROF=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/prof_c5.json 2> $D/prof_c5.err
ls -la $D
