# env sweep on one config: tools/gpu_sweepc.sh TAG CONFIG STEPS "VAR=a" ...
D=gpurun_out/$1; C=$2; S=$3; shift 3; mkdir -p $D
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 900 python bench.py --config $C --steps $S --warmup 1 --no-cpu --no-e2e > $D/c${C}_s$i.json 2> $D/c${C}_s$i.err
  python -c "import json,sys;d=json.load(open('$D/c${C}_s$i.json'));print('c$C', '$e', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_avg'],3))" >> $D/summary.txt 2>&1
done
cat $D/summary.txt
