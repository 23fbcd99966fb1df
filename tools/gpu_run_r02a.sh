set -x
mkdir -p gpurun_out/r02a
nvidia-smi > gpurun_out/r02a/nvidia-smi.txt 2>&1
lscpu > gpurun_out/r02a/lscpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=30 > gpurun_out/r02a/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02a/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02a/bench_default.json 2> gpurun_out/r02a/bench_default.err
echo "bench exit $?"
