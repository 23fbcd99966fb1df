# iteration check: diag/unit parity tests, config-3/5 bench lines with chunk variants; $1 = out dir tag
D=gpurun_out/${1:-iter}; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "diag or unit or replay or hub or multibatch or subset" > $D/pytest.log 2>&1; echo "pytest exit $?" >> $D/pytest.log
tail -3 $D/pytest.log
for ch in 1024 512 2048; do
MCF_UNIT_CHUNK=$ch timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_ch$ch.json 2> $D/c3_ch$ch.err
MCF_UNIT_CHUNK=$ch timeout 900 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_ch$ch.json 2> $D/c5_ch$ch.err
done
python - "$D" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/c*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['ms_per_step'],1), round(d['roofline']['kernel_ms_avg'],1))
    except Exception as e: print(f,'ERR',e)
P
