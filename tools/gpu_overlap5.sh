D=gpurun_out/${1:-ov}; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -x -k "multibatch" > $D/pytest.log 2>&1; echo "pytest exit $?" >> $D/pytest.log
tail -3 $D/pytest.log
for r in 1 2; do
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_r$r.json 2> $D/c3_r$r.err
timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_r$r.json 2> $D/c5_r$r.err
done
MCF_DIAG_PROF=1 timeout 600 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu --no-e2e 2>&1 | grep overlap > $D/traj_c3.txt
MCF_DIAG_PROF=1 timeout 600 python bench.py --config 5 --steps 1 --warmup 0 --no-cpu --no-e2e 2>&1 | grep overlap > $D/traj_c5.txt
python - "$D" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/c*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['ms_per_step'],1), round(d['roofline']['kernel_ms_avg'],1))
    except Exception as e: print(f,'ERR',e)
P
