#!/bin/bash
# Profile capture recipe (run on the B200 box via gpurun from the repo root).
#   profiles/capture.sh <tag> [config]
# 1. bench line without a profiler; 2. the ncu launch list of the same command
# (cold-cache, serialised per-launch times); 3. one `--set full` capture of the
# hot-path kernels of one step. Outputs go to gpurun_out/<tag>_*.
tag=${1:-r02}
cfg=${2:-c3}
set -x
python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_launches.log 2>&1 || exit 2
ncu --set full --clock-control none --import-source on \
    -k regex:'jacobi|qr_kernel|spmm|sparse_gram|cholesky|syrk_records|neighbor|speculate|presence|random_fill|apply_q|tridiag|bisect|inverse_iter' \
    --launch-count 24 -f -o /tmp/${tag}_full \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_full.log 2>&1 || exit 3
# the report itself stays on the box (gpurun_out is capped at 64 MiB): its raw page as CSV
ncu -i /tmp/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_full_raw.csv || exit 4
