"""Generate tests/golden/*.{json,npz} from the unmodified reference library
(oracle/_ref/libranky_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run once in a container that has /root/reference:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the CPU restatement (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py) on machines where the reference is absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import Oracle  # noqa: E402

R = Oracle("reference")


def coo(m):
    return m


def repair_cases():
    """(name, matrix, D, method, seed) -- instances from proj/tests/repair_test.cpp plus sweeps."""
    cases = []
    def sm(rows, cols, entries):
        e = sorted(entries)
        return (rows, cols, np.array([x[0] for x in e], np.uint64), np.array([x[1] for x in e], np.uint64),
                np.array([x[2] for x in e], np.float64))
    # repair_test.cpp:253-262 log format instance
    cases.append(("log_format", sm(2, 4, [(0, 0, 1.0), (0, 2, 1.0), (1, 2, 1.0)]), 2, "neighbor", 5))
    # :264-273 single block isolated row
    cases.append(("fallback_single", sm(3, 6, [(0, 0, 1.0), (2, 1, 1.0)]), 1, "neighbor", 0))
    # :274-284 isolated row across two blocks
    cases.append(("fallback_two", sm(3, 6, [(0, 0, 1.0), (0, 4, 1.0), (2, 1, 1.0), (2, 5, 1.0)]), 2, "neighbor", 0))
    # :187-195 empty matrix
    cases.append(("empty", sm(3, 6, []), 2, "random", 9))
    # :90-102 neighbor follows shared columns
    cases.append(("neighbor_shared", sm(3, 6, [(0, 0, 1.0), (0, 2, 1.0), (0, 5, 1.0), (1, 5, 1.0), (2, 1, 1.0)]), 2,
                  "neighbor-random", 3))
    for seed in range(6):
        m = R.synth_bipartite(16, 128, 0.05, seed)
        for D in (1, 4, 8, 16):
            for meth in ("random", "neighbor", "neighbor-random", "none"):
                cases.append((f"synth16x128_s{seed}_D{D}_{meth}", m, D, meth, 17 + seed))
    m = R.synth_bipartite(64, 8192, 0.002, 7)
    for meth in ("random", "neighbor", "neighbor-random"):
        cases.append((f"desk64x8192_D8_{meth}", m, 8, meth, 42))
        cases.append((f"desk64x8192_D32_{meth}", m, 32, meth, 42))
    return cases


def main():
    out = {}
    # KeyedRng streams (proj/src/rng.cpp) and below() draws
    out["rng"] = [{"key": [s, b, r], "next": [str(x) for x in R.rng_stream(s, b, r, 5)]}
                  for s, b, r in [(0, 0, 0), (42, 0, 8), (7, 3, 11), (2**64 - 1, 2**63, 12345)]]
    out["rng_below"] = [{"key": [s, b, r], "bound": bd, "value": R.rng_below(s, b, r, bd)}
                        for s, b, r, bd in [(42, 0, 8, 1024), (1, 2, 3, 7), (5, 0, 0, 2**63 + 5), (9, 9, 9, 1)]]
    # reference test goldens: synth nnz, first lonely row, random column (repair_test.cpp:77-88)
    desk = R.synth_bipartite(64, 8192, 0.002, 7)
    out["synth_64_8192_0.002_7"] = {"nnz": int(len(desk[2])),
                                    "lonely_block0_D8": [int(x) for x in R.find_lonely_rows(desk, 8, 0)],
                                    "random_col_seed42_row8": R.rng_below(42, 0, 8, 1024)}
    reps = {}
    arrays = {}
    for name, m, D, meth, seed in repair_cases():
        res = R.repair(m, D, meth, seed)
        reps[name] = {"rows": int(m[0]), "cols": int(m[1]), "D": D, "method": meth, "seed": seed,
                      "edges": res.edges.tolist(), "lonely": res.lonely_counts.tolist(),
                      "fallback": res.fallback_count, "log": res.to_log(),
                      "repaired_nnz": int(len(res.matrix[2]))}
        arrays[f"in_{name}_r"], arrays[f"in_{name}_c"], arrays[f"in_{name}_v"] = m[2], m[3], m[4]
    out["repair"] = reps
    # dense SVD closed forms and random shapes (svd_test.cpp:37-110, acceptance 7)
    rng = np.random.default_rng(20260101)
    dense = {"identity2": np.eye(2), "diag32": np.diag([3.0, 2.0]), "perm": np.array([[0.0, 1.0], [1.0, 0.0]]),
             "rank1": np.array([[0, 0, 0, 0], [6.0, 0, 0, 8.0]]), "zero3x5": np.zeros((3, 5))}
    for shape in [(14, 14), (6, 40), (40, 6), (16, 256), (64, 64), (33, 7)]:
        dense[f"rand{shape[0]}x{shape[1]}"] = rng.uniform(-1, 1, shape)
    low = rng.uniform(-1, 1, (12, 4)) @ rng.uniform(-1, 1, (4, 16))
    dense["lowrank12x16"] = low
    for k, a in dense.items():
        s = R.dense_svd(a)
        arrays[f"dense_{k}_a"] = a
        arrays[f"dense_{k}_sigma"] = s.sigma
        arrays[f"dense_{k}_u"] = s.u
        arrays[f"dense_{k}_v"] = s.v
    # block_svd on sparse blocks
    for seed in range(3):
        for (m_, n_, dens) in [(16, 256, 0.2), (64, 512, 0.02), (9, 4, 1.0)]:
            b = R.synth_bipartite(m_, n_, dens, 100 + seed)
            vals = np.linspace(-1.5, 2.5, len(b[2]))
            vals[vals == 0] = 0.25
            blk = (b[0], b[1], b[2], b[3], vals)
            s = R.block_svd(blk, m_)
            key = f"block_{m_}x{n_}_s{seed}"
            arrays[key + "_r"], arrays[key + "_c"], arrays[key + "_v"] = b[2], b[3], vals
            arrays[key + "_sigma"], arrays[key + "_u"] = s.sigma, s.u
    # pipelines (sigma, U, records) on desk-scale instances
    pipes = {}
    vrng = np.random.default_rng(99)
    valued = (desk[0], desk[1], desk[2], desk[3], vrng.uniform(0.5, 1.5, len(desk[2])) * vrng.choice([-1, 1], len(desk[2])))
    for name, (m, D, meth, keep, seed) in {
        "desk_D8_neighbor": (desk, 8, "neighbor", 0, 3),
        # keep < rank needs distinct singular values at the cut (value-1.0 blocks are
        # degenerate there and the kept vectors would be an arbitrary basis choice)
        "valued_D16_random_keep3": (valued, 16, "random", 3, 5),
        "synth16x96_D6_nr": (R.synth_bipartite(16, 96, 0.05, 8), 6, "neighbor-random", 0, 3),
    }.items():
        res = R.run_pipeline(m, D, meth, keep, seed, 4)
        pipes[name] = {"D": D, "method": meth, "keep": keep, "seed": seed}
        arrays[f"pipe_{name}_r"], arrays[f"pipe_{name}_c"], arrays[f"pipe_{name}_v"] = m[2], m[3], m[4]
        arrays[f"pipe_{name}_shape"] = np.array([m[0], m[1]])
        arrays[f"pipe_{name}_sigma"], arrays[f"pipe_{name}_u"] = res.sigma, res.u
        arrays[f"pipe_{name}_edges"] = res.edges
        for d, rec in enumerate(res.records):
            arrays[f"pipe_{name}_rec{d}"] = rec
        pipes[name]["records"] = len(res.records)
        v = R.recover_right_vectors(res.matrix, res.u, res.sigma, 1e-10)
        arrays[f"pipe_{name}_V"] = v
        arrays[f"pipe_{name}_rep_r"], arrays[f"pipe_{name}_rep_c"], arrays[f"pipe_{name}_rep_v"] = res.matrix[2:]
    out["pipelines"] = pipes
    json.dump(out, open(os.path.join(HERE, "reference_golden.json"), "w"), indent=1)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **arrays)
    print("wrote", len(reps), "repair cases,", len(dense), "dense cases,", len(pipes), "pipelines")


if __name__ == "__main__":
    main()
