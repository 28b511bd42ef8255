#!/bin/bash
out=gpurun_out/r02y; mkdir -p $out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-e2e > $out/gloo2.log 2>&1
echo "gloo2 rc=$?" >> $out/summary.txt
python -m pytest tests/test_gpu_multi.py tests/test_gpu_shard.py -m gpu -q -x -p no:cacheprovider > $out/pytest_multi.log 2>&1
echo "pytest multi rc=$?" >> $out/summary.txt
bash profiles/capture.sh r02w c3
echo "capture rc=$?" >> $out/summary.txt
