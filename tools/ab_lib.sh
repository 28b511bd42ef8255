#!/bin/bash
# A/B of library builds on the GPU box: tools/ab_lib.sh lib1.so lib2.so ...  (each copied over the package's .so)
for l in "$@"; do
  cp "$l" paper_2009_09767_b200/libranky_b200.so
  echo "== $l"; timeout 300 python tools/tune_jacobi.py 2>&1 | grep "block jacobi" | head -1
done
