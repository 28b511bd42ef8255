#!/bin/bash
# compute-sanitizer over the small cases, one tool at a time
out=gpurun_out/r02w_sanitize; mkdir -p $out
for tool in memcheck racecheck synccheck; do
  for case in c1 c2s c3s wide nbr dense; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $case \
      > $out/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -c 'ERROR SUMMARY: 0 errors' $out/${tool}_${case}.log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' $out/${tool}_${case}.log | tail -1)" >> $out/summary.txt
  done
done
timeout 1200 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/bench_c5.jsonl 2> $out/bench_c5.err
echo "bench c5 rc=$?" >> $out/summary.txt
