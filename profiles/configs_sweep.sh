#!/bin/bash
# Device time of every BASELINE config on one B200 (bench.py lines; c2 is the
# official workload, the others are parity configs measured the same way).
# CPU reference times come from `--impl reference` where it finishes in minutes.
tag=${1:-r01}
out=gpurun_out/${tag}_configs.jsonl
: > $out
python bench.py --config c1 --steps 10 --warmup 3 >> $out 2>/dev/null
python bench.py --config c1 --impl reference --steps 3 --warmup 1 >> $out 2>/dev/null
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> $out 2>/dev/null
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $out 2>/dev/null
timeout 900 python bench.py --config c3 --impl reference --steps 1 --warmup 0 >> $out 2>/dev/null
cat $out | cut -c1-300
