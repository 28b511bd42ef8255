#!/bin/bash
out=gpurun_out/r02x; mkdir -p $out
RK_BENCH_WATCHDOG=150 RK_TRACE=${RK_TRACE_SET:-0} timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29514 bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --no-e2e > $out/gloo2.log 2>&1
echo "gloo2 rc=$?" >> $out/summary.txt
RK_JACOBI_SMEM=0 RK_BENCH_WATCHDOG=150 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29515 bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --no-e2e > $out/gloo2_nosmem.log 2>&1
echo "gloo2 nosmem rc=$?" >> $out/summary.txt
