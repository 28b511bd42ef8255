#!/bin/bash
# One long GPU-box job (run from the repo root via gpurun): the c4/c5 merge goldens
# (the reference's proxy_svd on the GPU's records: ~1.5 h of single-threaded CPU)
# with GPU work interleaved while the reference computes.
out=gpurun_out/long
mkdir -p $out
python tests/golden/make_merge_golden.py c4 $out > $out/golden_c4.log 2>&1 &
p4=$!
sleep 60
python tests/golden/make_merge_golden.py c5 $out > $out/golden_c5.log 2>&1 &
p5=$!
# the c5 golden's GPU phase (~7 min) first
for i in $(seq 1 90); do grep -q "GPU pipeline" $out/golden_c5.log 2>/dev/null && break; sleep 10; done
for tool in memcheck racecheck synccheck; do
  for case in c1 c2s nbr dense; do
    timeout 400 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $case \
      > $out/sanitize_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" >> $out/sanitize_summary.txt
  done
done
timeout 900 python bench.py --config c4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $out/bench_c4.log 2>&1
# ncu at c4: rank check, V SpMM, the Gram-assisted warp Jacobi (one launch each)
for k in presence_flat spmm jacobi_warp; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k --launch-count 1 -f \
    -o $out/c4_$k python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
    > $out/ncu_c4_$k.log 2>&1
done
wait $p4 $p5
echo long-job-done
