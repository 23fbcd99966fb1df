D=gpurun_out/${1:-traffic}; C=${2:-3}; mkdir -p $D
MCF_DIAG_OVERLAP=0 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:k_diag_unit|k_walk_emit|k_walk_action|k_unit_partition|k_diag_q" --csv --log-file $D/traffic_c$C.csv python bench.py --config $C --steps 1 --warmup 0 --no-cpu --no-e2e > $D/traffic_c$C.log 2>&1
python tools/traffic_json.py $D/traffic_c$C.csv 1 > $D/traffic_config$C.json
cat $D/traffic_config$C.json
