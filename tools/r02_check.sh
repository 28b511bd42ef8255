#!/bin/bash
# GPU check after a batch of changes: the GPU tests, c3/c2 bench lines (device only),
# the host/device stage split at c3, and the two-rank gloo dry run of bench.py's N>1
# path (both ranks on device 0, collectives through gloo; a functional check).
tag=${1:-r02x}
out=gpurun_out/$tag
mkdir -p $out
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_c3.log 2>&1
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_c2.log 2>&1
RK_HOSTPROF=1 timeout 300 python tools/hostprof.py c3 2 > $out/hostprof_c3.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-e2e > $out/gloo2.log 2>&1
echo "gloo2 rc=$?" >> $out/summary.txt
