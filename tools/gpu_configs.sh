# bench lines for every config (device arm, no CPU leg) + the default line with CPU baseline
set -x
D=gpurun_out/${1:-cfg}; mkdir -p $D
timeout 900 python bench.py --config 1 --no-cpu > $D/bench_config1.json 2> $D/bench_config1.err
timeout 900 python bench.py --config 2 --no-cpu > $D/bench_config2.json 2> $D/bench_config2.err
timeout 1200 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/bench_config5.json 2> $D/bench_config5.err
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e > $D/bench_config4.json 2> $D/bench_config4.err
ls -la $D
