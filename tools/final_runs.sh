set -x
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_config2.json 2> gpurun_out/final/bench_config2.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_config2_reference.json 2> gpurun_out/final/ref.err
python bench.py --config 1 > gpurun_out/final/bench_config1.json 2> gpurun_out/final/bench_config1.err
python bench.py --config 3 --steps 2 --warmup 3 > gpurun_out/final/bench_config3.json 2> gpurun_out/final/bench_config3.err
python bench.py --config 5 --steps 2 --warmup 3 --no-e2e > gpurun_out/final/bench_config5.json 2> gpurun_out/final/bench_config5.err
python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/final/bench_config4.json 2> gpurun_out/final/bench_config4.err
bash tools/ncu_times.sh "k_" gpurun_out/final/launches_config3.csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/final/launches_config3_summary.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_diag_q" --launch-skip 4 -c 1 -o gpurun_out/final/ncu_diag_q_config3 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/final/ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_diag_qc" --launch-skip 4 -c 1 -o gpurun_out/final/ncu_diag_qc_config3 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/final/ncu3b.log 2>&1
ls -la gpurun_out/final
