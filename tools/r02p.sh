#!/bin/bash
# after a Jacobi change: GPU tests (c5 full size left out), c3 / c2 / c1 bench lines, the c3 launch list
out=gpurun_out/r02p; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_c5_full.py::test_c5_full_size > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
for c in c3 c2 c1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_${c}.jsonl 2> $out/bench_${c}.err
  echo "bench $c rc=$?" >> $out/summary.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c3.csv \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/launches_c3.log 2>&1
