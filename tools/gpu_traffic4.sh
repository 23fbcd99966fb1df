D=gpurun_out/${1:-tr4}; mkdir -p $D
for f in 64 32; do
MCF_L2_FETCH=$f ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:k_walk_action" --csv --log-file $D/traffic_c4_f$f.csv python bench.py --config 4 --steps 1 --warmup 0 --no-cpu --no-e2e > $D/traffic_c4_f$f.log 2>&1
python tools/traffic_json.py $D/traffic_c4_f$f.csv 1 > $D/traffic_config4_f$f.json
done
cat $D/*.json; tail -2 $D/traffic_c4_f64.log
