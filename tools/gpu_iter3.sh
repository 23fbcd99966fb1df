# parity tests on the default library, then config-3/5 bench lines for it and the named variants; $1 = tag, rest = variants
D=gpurun_out/$1; shift; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "diag or unit or replay or hub or multibatch or subset" > $D/pytest.log 2>&1; echo "pytest exit $?" >> $D/pytest.log
tail -3 $D/pytest.log
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_default.json 2> $D/c3_default.err
timeout 900 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_default.json 2> $D/c5_default.err
for v in "$@"; do
  MCFUNM_CUDA_LIB=$PWD/scratch/libs/$v.so timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_$v.json 2> $D/c3_$v.err
  MCFUNM_CUDA_LIB=$PWD/scratch/libs/$v.so timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_$v.json 2> $D/c5_$v.err
done
python - "$D" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/c*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['ms_per_step'],1), round(d['roofline']['kernel_ms_avg'],1))
    except Exception as e: print(f,'ERR',e)
P
