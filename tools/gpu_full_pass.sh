#!/bin/bash
# The full GPU pass of a round (run on the box from the repo root): GPU tests (c5 full size included), the default bench line (c3, e2e + cpu_baseline),
# the reference arm, c1 / c2 / c4 lines, the two-rank gloo dry run.
out=gpurun_out/r02x; mkdir -p $out
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/summary.txt
timeout 900 python bench.py > $out/bench_c3.jsonl 2> $out/bench_c3.err
echo "bench rc=$?" >> $out/summary.txt
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $out/bench_ref.jsonl 2> $out/bench_ref.err
echo "ref rc=$?" >> $out/summary.txt
for c in c1 c2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $out/bench_$c.jsonl 2> $out/bench_$c.err
done
timeout 900 python bench.py --config c4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $out/bench_c4.jsonl 2> $out/bench_c4.err
echo "c4 rc=$?" >> $out/summary.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-e2e > $out/gloo2.log 2>&1
echo "gloo2 rc=$?" >> $out/summary.txt
bash profiles/capture.sh r02x c3
echo "capture rc=$?" >> $out/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo "smoke rc=$?" >> $out/summary.txt
