"""Sharding plan for the one-process-per-GPU path.

Column blocks are grouped into the leaves of the fixed merge tree
(rk_merge_tree_leaves). Rank g of G owns a contiguous, aligned range of leaves:
it factors those blocks, reduces them to its subtree's Gram partial
(rk_dev_shard_factor_gram; or its R factor, rk_dev_shard_factor /
rk_dev_shard_tsqr, when the Gram route is rejected), and owns the V rows of
those blocks' columns. The G factors are all-gathered (NCCL) and every rank
finishes the same top of the pairwise tree (rk_dev_shard_finish_gram /
rk_dev_shard_finish). With leaves/G a power of two every rank's
subtree is a node of the single-GPU tree, so the result is bitwise independent
of G.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    leaf_lo: int
    leaf_hi: int
    col_lo: int
    col_hi: int


def merge_tree_leaves(rows: int, cols: int, blocks: int, keep: int) -> int:
    from .ranky import lib
    return int(lib().rk_merge_tree_leaves(rows, cols, blocks, keep))


def leaf_blocks(rows: int, cols: int, blocks: int, keep: int) -> list[tuple[int, int]]:
    """Block range [b0, b1) of every leaf: consecutive blocks until >= rows
    record columns (mirrors merge_leaves in csrc/rk_pipeline.cu)."""
    width = cols // blocks
    kept = []
    for d in range(blocks):
        w = (cols - d * width) if d + 1 == blocks else width
        k_full = min(rows, w)
        kept.append(k_full if keep == 0 else min(keep, k_full))
    out, r0 = [], 0
    while r0 < blocks:
        r1, h = r0, 0
        while r1 < blocks and h < rows:
            h += kept[r1]
            r1 += 1
        if h > 0:
            out.append((r0, r1))
        r0 = r1
    return out


def plan(rows: int, cols: int, blocks: int, keep: int, world: int, rank: int) -> Shard:
    leaves = leaf_blocks(rows, cols, blocks, keep)
    n = len(leaves)
    if world < 1 or world > n:
        raise ValueError(f"cannot shard {n} leaves over {world} ranks")
    per = n // world
    lo = rank * per
    hi = n if rank + 1 == world else (rank + 1) * per
    width = cols // blocks
    b0, b1 = leaves[lo][0], leaves[hi - 1][1]
    col_lo = b0 * width
    col_hi = cols if b1 == blocks else b1 * width
    return Shard(rank, world, lo, hi, col_lo, col_hi)


def bitwise_invariant(n_leaves: int, world: int) -> bool:
    per = n_leaves // world
    return n_leaves % world == 0 and per > 0 and (per & (per - 1)) == 0


def pairwise_tree(nodes, combine):
    """The fixed pairwise reduction of csrc/rk_pipeline.cu forest_reduce: (0,1),
    (2,3), ...; an odd last node is carried up unchanged."""
    nodes = list(nodes)
    while len(nodes) > 1:
        nxt = [combine(nodes[i], nodes[i + 1]) for i in range(0, len(nodes) - 1, 2)]
        if len(nodes) % 2:
            nxt.append(nodes[-1])
        nodes = nxt
    return nodes[0]
