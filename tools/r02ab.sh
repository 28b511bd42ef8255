#!/bin/bash
out=gpurun_out/r02ab; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_pipeline.py tests/test_gpu_svd.py tests/test_gpu_shard.py tests/test_gpu_multi.py tests/test_gpu_c5.py tests/test_gpu_acceptance.py tests/test_gpu_records.py tests/test_gpu_c_abi.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_c3.jsonl 2> $out/bench_c3.err
