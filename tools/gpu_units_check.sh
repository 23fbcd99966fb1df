# unit combine: parity tests + config-3 timing (prof) + A/B
set -x
D=gpurun_out/units; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "diag or replay or hub or lean" > $D/pytest_parity.log 2>&1; echo "parity exit $?" >> $D/pytest_parity.log
MCF_DIAG_PROF=1 timeout 600 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/prof_c3.json 2> $D/prof_c3.err
timeout 600 python bench.py --config 3 --steps 3 --warmup 1 --no-cpu --no-e2e > $D/bench_c3.json 2> $D/bench_c3.err
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -x -k "config3" > $D/pytest_c3.log 2>&1; echo "c3 exit $?" >> $D/pytest_c3.log
ncu --set full --import-source on --clock-control none -k regex:k_diag_unit --launch-skip 2 -c 1 -o $D/ncu_unit_c3 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/ncu.log 2>&1
