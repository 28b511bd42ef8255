#!/bin/bash
out=gpurun_out/r02s; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_c5_full.py::test_c5_full_size > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
for c in c3 c2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_${c}.jsonl 2> $out/bench_${c}.err
  echo "bench $c rc=$?" >> $out/summary.txt
done
timeout 900 python tools/probe_c5.py 64 > $out/c5_64.log 2>&1
echo "c5 probe rc=$?" >> $out/summary.txt
bash tools/r02q.sh c3
