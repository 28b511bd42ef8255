#!/bin/bash
out=gpurun_out/r02t; mkdir -p $out
./tools/probe_fp64_pipes > $out/fp64_pipes.log 2>&1
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_c3.jsonl 2> $out/bench_c3.err
python -m pytest tests/test_gpu_svd.py -m gpu -q -x -p no:cacheprovider > $out/pytest.log 2>&1
