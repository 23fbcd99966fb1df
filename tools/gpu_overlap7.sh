D=gpurun_out/${1:-ov}; mkdir -p $D
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_$tag.json 2> $D/c3_$tag.err; env "$@" timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_$tag.json 2> $D/c5_$tag.err; }
run b13g05 MCF_OVERLAP_BIAS=1.3 MCF_OVERLAP_GAIN=0.5
run b115g05 MCF_OVERLAP_BIAS=1.15 MCF_OVERLAP_GAIN=0.5
run b13g10 MCF_OVERLAP_BIAS=1.3 MCF_OVERLAP_GAIN=1.0
run b115g10 MCF_OVERLAP_BIAS=1.15 MCF_OVERLAP_GAIN=1.0
run b145g07 MCF_OVERLAP_BIAS=1.45 MCF_OVERLAP_GAIN=0.7
python - "$D" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/c*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['ms_per_step'],1))
    except Exception as e: print(f,'ERR',e)
P
