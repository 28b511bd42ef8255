#!/bin/bash
out=gpurun_out/r02ad; mkdir -p $out
for cl in 2 4 8; do
  RK_JACOBI_SMEM_CL=$cl timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_c2_cl$cl.jsonl 2> $out/bench_c2_cl$cl.err
done
