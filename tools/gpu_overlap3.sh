D=gpurun_out/${1:-ov}; mkdir -p $D
for ov in 20 28 36 44; do
  MCF_WALK_NW=1 MCF_DIAG_OVERLAP=$ov timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_ov$ov.json 2> $D/c3_ov$ov.err
  MCF_WALK_NW=1 MCF_DIAG_OVERLAP=$ov timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_ov$ov.json 2> $D/c5_ov$ov.err
done
python - "$D" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/c*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['ms_per_step'],1), round(d['roofline']['kernel_ms_avg'],1))
    except Exception as e: print(f,'ERR',e)
P
