# env sweep on the config-3 bench: tools/gpu_sweep.sh TAG "VAR=a VAR2=b" "VAR=c" ...
D=gpurun_out/$1; shift; mkdir -p $D
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e > $D/s$i.json 2> $D/s$i.err
  python -c "import json,sys;d=json.load(open('$D/s$i.json'));print('$e', round(d['ms_per_step'],1), round(d['roofline']['kernel_ms_avg'],1))" >> $D/summary.txt 2>&1
done
cat $D/summary.txt
