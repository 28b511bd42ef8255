out=gpurun_out/r02k; mkdir -p $out
RK_BENCH_WATCHDOG=240 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-e2e > $out/gloo2.log 2>&1
echo "gloo2 rc=$?" >> $out/summary.txt
RK_EIG_MERGE=0 RK_BENCH_WATCHDOG=240 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-e2e > $out/gloo2_noeig.log 2>&1
echo "gloo2 noeig rc=$?" >> $out/summary.txt
timeout 900 python bench.py > $out/bench_default.log 2>&1
echo "bench rc=$?" >> $out/summary.txt
bash profiles/capture.sh r02k c3 > $out/capture.log 2>&1
echo "capture rc=$?" >> $out/summary.txt
