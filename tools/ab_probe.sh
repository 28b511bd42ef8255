#!/bin/bash
# build a probe variant of the library into /tmp and run one c3 pipeline with it
out=gpurun_out/probe; mkdir -p $out
python bench.py --config ${1:-c3} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/probe.log 2>&1
echo rc=$? >> $out/probe.log
