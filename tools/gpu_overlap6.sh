D=gpurun_out/${1:-ov}; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -x -k "multibatch" > $D/pytest.log 2>&1; echo "pytest exit $?" >> $D/pytest.log
tail -3 $D/pytest.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_$tag.json 2> $D/c3_$tag.err; env "$@" timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_$tag.json 2> $D/c5_$tag.err; }
run bang MCF_OVERLAP_CTRL=0
run b13 MCF_OVERLAP_BIAS=1.3
run b16 MCF_OVERLAP_BIAS=1.6
run b20 MCF_OVERLAP_BIAS=2.0
run off MCF_DIAG_OVERLAP=0
python - "$D" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/c*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['ms_per_step'],1), round(d['roofline']['kernel_ms_avg'],1))
    except Exception as e: print(f,'ERR',e)
P
