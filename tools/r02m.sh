out=gpurun_out/r02m; mkdir -p $out
RK_BENCH_WATCHDOG=200 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29514 bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --no-e2e > $out/gloo2.log 2>&1
echo "gloo2 rc=$?" >> $out/summary.txt
python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_c5_full.py::test_c5_full_size > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_c3.log 2>&1
RK_HOSTPROF=1 timeout 300 python tools/hostprof.py c3 2 > $out/hostprof_c3.log 2>&1
