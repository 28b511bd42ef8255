#!/bin/bash
# presence from the CSC: repair tests, c4 capture of the rank check, e2e split at c3
out=gpurun_out/r02v; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_repair.py tests/test_gpu_workspace.py tests/test_gpu_pipeline.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:presence_csc --launch-count 1 -f \
    -o $out/c4_presence_csc python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $out/ncu_c4_presence.log 2>&1
echo "ncu rc=$?" >> $out/summary.txt
ncu -i $out/c4_presence_csc.ncu-rep --page raw --csv > $out/c4_presence_csc_raw.csv
RK_HOSTPROF=1 timeout 600 python tools/e2e_probe.py c3 > $out/e2e_probe_c3.log 2>&1
echo "e2e rc=$?" >> $out/summary.txt
