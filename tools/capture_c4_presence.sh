#!/bin/bash
# the rank check at c4 under `ncu --set full`, plus the repair / workspace / pipeline tests and c1-c3 bench lines
out=gpurun_out/r02x_c4; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_repair.py tests/test_gpu_workspace.py tests/test_gpu_pipeline.py tests/test_gpu_scale.py tests/test_gpu_c5.py -m gpu -q -x -p no:cacheprovider > $out/pytest_presence.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
timeout 900 ncu --set full --clock-control none -k regex:presence_csc --launch-count 1 -f -o $out/c4_presence python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $out/ncu_presence.log 2>&1
ncu -i $out/c4_presence.ncu-rep --page raw --csv > $out/c4_presence_raw.csv
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_c3.jsonl 2> $out/bench_c3.err
