out=gpurun_out/r02h; mkdir -p $out
python -m pytest tests/test_gpu_c5_full.py -x -q -s -p no:cacheprovider > $out/c5full.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_c5_full.py::test_c5_full_size --durations=20 > $out/pytest.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $out/launches_c3.log 2>&1
RK_HOSTPROF=1 timeout 600 python tools/e2e_probe.py c3 > $out/e2e_probe.log 2>&1
