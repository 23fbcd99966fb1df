# iteration check: diag/unit parity tests, config-3 and config-5 bench lines; $1 = out dir tag
set -x
D=gpurun_out/${1:-iter}; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "diag or unit or replay or hub or multibatch or subset" > $D/pytest.log 2>&1; echo "pytest exit $?" >> $D/pytest.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 1 --no-cpu --no-e2e > $D/bench_c3.json 2> $D/bench_c3.err
timeout 900 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/bench_c5.json 2> $D/bench_c5.err
