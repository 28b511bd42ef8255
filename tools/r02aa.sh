#!/bin/bash
out=gpurun_out/r02aa; mkdir -p $out
RK_JACOBI_DEBUG=1 timeout 900 python tools/probe_c5.py 16 > $out/c5_16.log 2>&1
echo "probe rc=$?" >> $out/summary.txt
