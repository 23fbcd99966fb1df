# bench configs 3 and 5 under values of one environment variable: gpu_env_sweep.sh TAG VAR v1 v2 ...
D=gpurun_out/$1; VAR=$2; shift; shift; mkdir -p $D
for v in "$@"; do
  env $VAR=$v timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_$v.json 2> $D/c3_$v.err
  env $VAR=$v timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_$v.json 2> $D/c5_$v.err
done
python - "$D" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/c*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d['ms_per_step'],1), round(d['roofline']['kernel_ms_avg'],1))
    except Exception as e: print(f,'ERR',e)
P
