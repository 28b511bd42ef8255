"""Writes tests/golden/record_ref.rnky with the UNMODIFIED reference
(oracle/_ref: ranky::write_block_record of ranky::run_block_task's record for a
synth_bipartite block, as proj/tests/harness_test.cpp:23-28 builds its sample).
Run from the repo root after `make -C oracle ref`."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Oracle  # noqa: E402

ref = Oracle("reference")
a = ref.synth_bipartite(6, 24, 0.4, 3)
svd = ref.block_svd(a, 6)
payload = svd.u * svd.sigma  # make_block_record: U with column j scaled by sigma_j
out = os.path.join(ROOT, "tests", "golden", "record_ref.rnky")
ref.write_block_record(2, payload, out)
print(out, os.path.getsize(out), "bytes")
