#!/bin/bash
# one `ncu --set full` launch of the wide pair-block Jacobi at c4 (a step in the middle of the second sweep)
out=gpurun_out/r02x_c4; mkdir -p $out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:jacobi_wide_step --launch-skip 40 --launch-count 1 -f \
    -o $out/c4_wide python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $out/ncu_c4_wide.log 2>&1
echo "ncu rc=$?" >> $out/summary.txt
ncu -i $out/c4_wide.ncu-rep --page raw --csv > $out/c4_wide_raw.csv
