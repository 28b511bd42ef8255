#!/bin/bash
# A/B of block-stage settings on the c3 bench (device time only), then the c5 full test.
out=gpurun_out/${1:-r02i}; mkdir -p $out
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/ab_$name.log 2>&1; }
run default
run rows32 RK_WIDE_ROWS=32
run q32g8 RK_JACOBI_Q=32 RK_JACOBI_GMAX=8
run g8 RK_JACOBI_GMAX=8
run g12 RK_JACOBI_GMAX=12
python -m pytest tests/test_gpu_c5_full.py tests/test_gpu_svd.py tests/test_gpu_scale.py -q -s -p no:cacheprovider > $out/pytest_c5_svd_scale.log 2>&1
