#!/bin/bash
# c4 (M=1024, N=16.8M, 17.2M nnz, 1024 blocks, NeighborRandom): the bench line
# (device only: V is 128 GiB on the host side) and ncu captures of the rank check,
# the V SpMM and the Gram-assisted warp Jacobi, one launch each.
out=gpurun_out/r02_c4; mkdir -p $out
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e > $out/bench_c4.log 2>&1
echo "bench rc=$?" >> $out/summary.txt
for k in presence_flat spmm jacobi_warp speculate neighbor_replay; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-count 1 -f \
    -o $out/c4_$k python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
    > $out/ncu_c4_$k.log 2>&1
  echo "ncu $k rc=$?" >> $out/summary.txt
done
