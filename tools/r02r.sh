#!/bin/bash
# c5 slice: stage timings on 64 blocks; block 0 of an 8-block slice against the reference's block_svd
out=gpurun_out/r02r; mkdir -p $out
RK_JACOBI_DEBUG=1 timeout 900 python tools/probe_c5.py 64 > $out/c5_64.log 2>&1
echo "probe rc=$?" >> $out/summary.txt
timeout 1500 python tools/probe_c5.py 8 check > $out/c5_8_check.log 2>&1
echo "check rc=$?" >> $out/summary.txt
