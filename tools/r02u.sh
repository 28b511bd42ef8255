#!/bin/bash
# wide pair-block Jacobi: c5 slice (timing, block 0 vs the reference), c4 full-size test, c4 bench line
out=gpurun_out/r02u; mkdir -p $out
RK_JACOBI_DEBUG=1 timeout 900 python tools/probe_c5.py 64 > $out/c5_64.log 2>&1
echo "probe rc=$?" >> $out/summary.txt
timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_c5.py tests/test_gpu_svd.py tests/test_gpu_shard.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $out/bench_c4.jsonl 2> $out/bench_c4.err
echo "bench c4 rc=$?" >> $out/summary.txt
timeout 1500 python tools/probe_c5.py 8 check > $out/c5_8_check.log 2>&1
echo "check rc=$?" >> $out/summary.txt
