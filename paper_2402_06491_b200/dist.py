"""Multi-GPU sharding of the hot path.

Trees of a node are independent, so ranks sample disjoint tree ranges of every
node with no data-path collective; their order-binned sums (ΣC, ΣC², count per
node and order — sums over disjoint tree sets add) are merged with one
all-reduce before finalisation and Padé.  With weak scaling each rank keeps
n_trees per node and the merged estimate is over world·n_trees trees.
"""
from __future__ import annotations

from typing import Tuple


def tree_range(rank: int, world: int, n_trees_per_rank: int) -> Tuple[int, int]:
    """(tree_offset, n_trees) of a rank under weak scaling: rank r samples
    trees [r·N, (r+1)·N) of every node (tree indices are uint32)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    off = rank * n_trees_per_rank
    if off + n_trees_per_rank > 1 << 32:
        raise ValueError("tree indices exceed 2^32")
    return off, n_trees_per_rank


def merge_sums(sums, group=None):
    """In-place SUM all-reduce of per-node order-binned sums [n, K+2, 3]."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    return sums
