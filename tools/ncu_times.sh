#!/bin/bash
# usage: tools/ncu_times.sh <kernel-regex> <out.csv> <command...>: per-launch device times of matching kernels
re="$1"; out="$2"; shift 2
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$re" --csv --log-file "$out" "$@" > /dev/null 2>&1
python "$(dirname "$0")/launch_summary.py" "$out"
