# round evidence: full GPU tests, default bench (config 3 + CPU baseline + e2e), every config, launch list, ncu of the top kernel
set -x
D=gpurun_out/${1:-round}; mkdir -p $D
nvidia-smi > $D/nvidia-smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > $D/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench_config3.json 2> $D/bench_config3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_config3_reference.json 2> $D/bench_config3_reference.err
timeout 900 python bench.py --config 1 --no-cpu > $D/bench_config1.json 2> $D/bench_config1.err
timeout 900 python bench.py --config 2 --no-cpu > $D/bench_config2.json 2> $D/bench_config2.err
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e > $D/bench_config4.json 2> $D/bench_config4.err
timeout 1200 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/bench_config5.json 2> $D/bench_config5.err
# (ncu serialises kernels: the launch list and the kernel capture use serial batches, MCF_DIAG_OVERLAP=0)
MCF_DIAG_OVERLAP=0 timeout 900 bash tools/ncu_times.sh "." $D/launches_config3.csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/launches_config3_summary.txt 2>&1
MCF_DIAG_OVERLAP=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_diag_unit --launch-skip 6 -c 1 -o $D/ncu_unit_config3 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/ncu_unit.log 2>&1
ls -la $D
