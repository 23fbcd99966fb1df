D=gpurun_out/${1:-ov}; mkdir -p $D
for ud in "4 2" "2 1" "4 1" "8 2" "2 2"; do set -- $ud; u=$1; d=$2
  MCF_OVERLAP_UP=$u MCF_OVERLAP_DOWN=$d timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/c3_u${u}d$d.json 2> $D/c3_u${u}d$d.err
  MCF_OVERLAP_UP=$u MCF_OVERLAP_DOWN=$d timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > $D/c5_u${u}d$d.json 2> $D/c5_u${u}d$d.err
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
