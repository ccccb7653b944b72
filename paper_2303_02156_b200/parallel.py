"""Multi-process plumbing: one process per GPU (torch.distributed, NCCL on the box, gloo in the
CPU tests), max-over-ranks device timing, and the element partition of the sharded assembly
design.

Sharded assembly (design; this round the bench runs replicas): block rows are split into
contiguous node-id slabs; element e belongs to the rank owning its first node; every rank
assembles its elements into its rows plus a halo of rows owned by neighbours; halo partials go
to their owners (one grouped exchange) and the energy is an all-reduce of one double. The CPU
tests check the decomposition with the C oracle: the per-rank partial assemblies sum to the
global one, every element is owned exactly once, and halo rows are exactly the rows a rank
touches but does not own.
"""
from __future__ import annotations

import dataclasses
import os
from typing import List

import numpy as np


@dataclasses.dataclass
class RankInfo:
    rank: int
    world: int
    local: int


def rank_info() -> RankInfo:
    return RankInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                    int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device times are reported as the slowest rank's)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


@dataclasses.dataclass
class Shard:
    rank: int
    node_lo: int            # owned nodes [node_lo, node_hi)
    node_hi: int
    elements: np.ndarray    # element ids owned by this rank (ascending)
    halo_nodes: np.ndarray  # nodes touched by owned elements but owned by other ranks


def slab_partition(conn: np.ndarray, n_nodes: int, world: int) -> List[Shard]:
    """Contiguous node slabs (grid node ids are i-major, so slabs are spatial slabs); element
    owner = owner of its first node."""
    conn = np.asarray(conn).reshape(conn.shape[0], -1)
    bounds = np.linspace(0, n_nodes, world + 1).round().astype(np.int64)
    owner_of_node = np.searchsorted(bounds, np.arange(n_nodes), side="right") - 1
    owner = owner_of_node[conn[:, 0]]
    shards = []
    for r in range(world):
        els = np.flatnonzero(owner == r)
        touched = np.unique(conn[els].ravel()) if els.size else np.zeros(0, np.int64)
        halo = touched[(touched < bounds[r]) | (touched >= bounds[r + 1])]
        shards.append(Shard(r, int(bounds[r]), int(bounds[r + 1]), els, halo))
    return shards
