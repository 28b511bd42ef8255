#!/bin/bash
out=gpurun_out/r02q; mkdir -p $out
cfg=${1:-c3}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$cfg.csv \
    python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/launches_$cfg.log 2>&1
echo "ncu rc=$?" >> $out/summary.txt
