"""Multi-process plumbing and the sharded assembly.

One process per GPU (torch.distributed: NCCL on the box, gloo in the CPU tests).

Sharded assembly, owner computes: block rows (nodes) are split into contiguous slabs; a rank
owns the elements whose first node it owns and additionally evaluates the *ghost* elements
that touch one of its nodes but belong to a neighbour. Its owned block rows (and gradient rows)
are then complete -- pattern and values -- without exchanging any matrix data: the only
collective on the data path is the all-reduce of one double (the owned energy). The cost is
the ghost layer (one hex plane of n per slab at config 2, 1 %). Every rank assembles its local
pattern, whose owned rows map to the global rows by the (monotone) local -> global node ids.

The CPU tests (tests/test_parallel.py) run this decomposition at world sizes 2 and 3 over gloo
with the C oracle as the element engine and compare the gathered owned rows with the global
assembly (pattern bit-exact, values to 1e-13).
"""
from __future__ import annotations

import dataclasses
import os
from typing import Tuple

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


def sum_over_ranks(value: float, device=None) -> float:
    """The data-path collective of the sharded assembly: sum of the owned energies."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return float(t.item())


@dataclasses.dataclass
class OwnerShard:
    """A rank's share of a global element set (local node numbering, global id order)."""
    rank: int
    world: int
    node_lo: int               # owned global nodes [node_lo, node_hi)
    node_hi: int
    own: np.ndarray            # owned global element ids (ascending)
    ghost: np.ndarray          # ghost global element ids (ascending)
    global_ids: np.ndarray     # local node -> global node id (ascending)
    conn: np.ndarray           # local connectivity: own elements first, then ghosts
    row_lo: int                # owned local block rows [row_lo, row_hi)
    row_hi: int

    @property
    def n_own(self) -> int:
        return int(self.own.size)


def node_bounds(n_nodes: int, world: int) -> np.ndarray:
    return np.linspace(0, n_nodes, world + 1).round().astype(np.int64)


def owner_shard(conn: np.ndarray, n_nodes: int, world: int, rank: int) -> OwnerShard:
    """Owner-computes shard of a global connectivity over contiguous node slabs."""
    conn = np.asarray(conn).reshape(conn.shape[0], -1)
    bounds = node_bounds(n_nodes, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    first = conn[:, 0]
    own = np.flatnonzero((first >= lo) & (first < hi))
    touches = ((conn >= lo) & (conn < hi)).any(axis=1)
    ghost = np.flatnonzero(touches & ~((first >= lo) & (first < hi)))
    compute = np.concatenate([own, ghost])
    # owned nodes are local even when no element touches them (their diagonal block exists)
    nodes = np.union1d(np.unique(conn[compute]), np.arange(lo, hi))
    g2l = np.full(n_nodes, -1, dtype=np.int64)
    g2l[nodes] = np.arange(nodes.size)
    return OwnerShard(rank, world, lo, hi, own, ghost, nodes, g2l[conn[compute]],
                      int(np.searchsorted(nodes, lo)), int(np.searchsorted(nodes, hi)))


def owned_rows(b: int, row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray, grad: np.ndarray,
               row_lo: int, row_hi: int, global_ids: np.ndarray) -> Tuple[np.ndarray, ...]:
    """The owned block rows of a local BSR (columns mapped to global node ids) and gradient rows."""
    s, e = int(row_ptr[row_lo]), int(row_ptr[row_hi])
    rp = np.asarray(row_ptr[row_lo:row_hi + 1], dtype=np.int64) - s
    ci = np.asarray(global_ids)[np.asarray(col_idx[s:e], dtype=np.int64)]
    v = np.asarray(values).reshape(-1, b * b)[s:e]
    g = np.asarray(grad)[row_lo * b:row_hi * b]
    return rp, ci, v, g


def gather_rows(parts):
    """Concatenates per-rank owned rows (rank order = global row order) into one BSR."""
    rps, cis, vs, gs = zip(*parts)
    off = 0
    rp = [np.zeros(1, dtype=np.int64)]
    for r in rps:
        rp.append(r[1:] + off)
        off += int(r[-1])
    return np.concatenate(rp), np.concatenate(cis), np.concatenate(vs), np.concatenate(gs)


class ShardedTetSystem:
    """Device side of one rank (tet4 energies): own + ghost energies on one context."""

    def __init__(self, x, X, conn, n_own: int, params, row_lo: int, row_hi: int, global_ids,
                 spd: bool = False, device: int = 0):
        from . import configs
        from .systems import DeviceSystem
        case = configs.Case("shard", "tet4", x, X, conn, params)
        self.ds = DeviceSystem(case, spd=spd, device=device, n_own=n_own)
        self.n_own = n_own
        self.row_lo, self.row_hi = row_lo, row_hi
        self.global_ids = np.asarray(global_ids)

    def assemble(self, mode: str = "deterministic") -> float:
        """Assembles the local pattern; returns this rank's owned energy (to be summed)."""
        self.ds.asm.assemble(mode)
        return float(self.ds.asm.energy_parts()[0])

    def owned(self):
        A = self.ds.asm
        H = A.hessian()
        return owned_rows(H.b, H.row_ptr, H.col_idx, H.values, A.gradient(), self.row_lo, self.row_hi,
                          self.global_ids)
