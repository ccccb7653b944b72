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


# ------------------------------------------------------------------ contact pairs (config 5)
#
# Random point-triangle pairs break the locality the ghost layer relies on: a pair touches 4
# random nodes, so ghosting would evaluate most pairs on most ranks. Pairs are instead owned by
# the rank that owns their point node p (tuple slot 0) and evaluated once; their contributions
# to block rows owned by other ranks are the one real exchange step. The tets
# stay owner-computes with ghosts and the inertia energy is evaluated for owned nodes, so those
# owned rows are complete locally. Merging is in a fixed order -- local tets + inertia, then
# the pair contributions of rank 0, 1, ... -- so the result is deterministic.

@dataclasses.dataclass
class ContactShard:
    tet: OwnerShard            # tets: owned + ghost elements, local nodes
    pairs: np.ndarray          # owned pair ids (ascending): pairs whose point node this rank owns
    pair_nodes: np.ndarray     # global ids of the nodes the owned pairs touch (ascending)
    pair_conn: np.ndarray      # owned pairs in pair_nodes numbering
    node_bounds: np.ndarray    # owner slabs of all ranks (world + 1)


def contact_shard(tet_conn: np.ndarray, pairs: np.ndarray, n_nodes: int, world: int, rank: int) -> ContactShard:
    tet = owner_shard(tet_conn, n_nodes, world, rank)
    bounds = node_bounds(n_nodes, world)
    p = np.asarray(pairs).reshape(-1, 4)
    mine = np.flatnonzero((p[:, 0] >= bounds[rank]) & (p[:, 0] < bounds[rank + 1]))
    nodes = np.unique(p[mine])
    g2l = np.full(n_nodes, -1, dtype=np.int64)
    g2l[nodes] = np.arange(nodes.size)
    return ContactShard(tet, mine, nodes, g2l[p[mine]] if mine.size else np.zeros((0, 4), np.int64), bounds)


def split_rows_by_owner(b: int, row_ptr, col_idx, values, grad, global_ids, bounds):
    """A local BSR (rows/cols in `global_ids` numbering) as per-destination-rank COO lists:
    [(rows, cols, blocks (k,b,b), grow_ids, grad_rows (m,b))] indexed by owner rank."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    gid = np.asarray(global_ids, dtype=np.int64)
    nr = row_ptr.size - 1
    rows = np.repeat(np.arange(nr), np.diff(row_ptr))
    grows, gcols = gid[rows], gid[np.asarray(col_idx, dtype=np.int64)]
    v = np.asarray(values).reshape(-1, b, b)
    g = np.asarray(grad).reshape(-1, b)
    owner_of_row = np.searchsorted(bounds, grows, side="right") - 1
    owner_of_grow = np.searchsorted(bounds, gid, side="right") - 1
    out = []
    for q in range(bounds.size - 1):
        sel = owner_of_row == q
        gs = owner_of_grow == q
        out.append((grows[sel], gcols[sel], v[sel], gid[gs], g[gs]))
    return out


def merge_owned_rows(b: int, own_rows, incoming, row_lo_global: int, row_hi_global: int):
    """Owned rows (owned_rows() output, global columns) plus incoming COO contributions, summed in
    the given order (deterministic). Returns (row_ptr, col_idx, values, grad) of the owned rows."""
    rp, ci, v, g = own_rows
    n = row_hi_global - row_lo_global
    rows = [np.repeat(np.arange(n), np.diff(rp)) + row_lo_global]
    cols, vals = [np.asarray(ci, dtype=np.int64)], [np.asarray(v).reshape(-1, b, b)]
    g = np.asarray(g, dtype=np.float64).reshape(-1, b).copy()
    for (r, c, blocks, grow, grad_rows) in incoming:
        rows.append(np.asarray(r, dtype=np.int64))
        cols.append(np.asarray(c, dtype=np.int64))
        vals.append(np.asarray(blocks).reshape(-1, b, b))
        if len(grow):
            np.add.at(g, np.asarray(grow, dtype=np.int64) - row_lo_global, np.asarray(grad_rows).reshape(-1, b))
    R, Cc, V = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    key = (R - row_lo_global) * (int(Cc.max(initial=0)) + 1) + Cc
    uk, inv = np.unique(key, return_inverse=True)
    out = np.zeros((uk.size, b, b))
    np.add.at(out, inv, V)  # sequential in concatenation order
    ncol = int(Cc.max(initial=0)) + 1
    urow, ucol = uk // ncol, uk % ncol
    row_ptr = np.concatenate([[0], np.cumsum(np.bincount(urow, minlength=n))]).astype(np.int64)
    return row_ptr, ucol.astype(np.int64), out, g.ravel()


def exchange(send_lists):
    """send_lists[q] = this rank's contributions for rank q -> [contributions from rank 0, 1, ...]
    for this rank. all_gather of Python objects (gloo and NCCL); one exchange per assemble."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [send_lists[0]]
    world, rank = dist.get_world_size(), dist.get_rank()
    allsend = [None] * world
    dist.all_gather_object(allsend, send_lists)
    return [allsend[src][rank] for src in range(world)]


class ShardedContactSystem:
    """Device side of one rank of the sharded config-5 assembly: context 1 holds the tets (own +
    ghost energies) and the inertia of the owned nodes, context 2 the owned contact pairs on
    their own node set. assemble() returns this rank's owned energy part and the pair rows to
    send to each rank; finish() merges the received rows into the owned rows."""

    def __init__(self, case, world: int, rank: int, spd: bool = False, device: int = 0):
        from .device import DeviceAssembler, ENERGY_EXACT, ENERGY_SPD
        from .systems import (contact_inputs, default_tapes, inertia_inputs, solid_tet_inputs)
        tapes = default_tapes()
        self.sh = sh = contact_shard(case.conn, case.extra["pairs"], case.n_nodes, world, rank)
        self.world, self.rank = world, rank
        p, ex, t = case.params, case.extra, sh.tet
        gid = t.global_ids
        flags = ENERGY_SPD if spd else 0
        A = self.main = DeviceAssembler(device)
        x = self.x = A.add_array("x", gid.size, 3, True)
        rest = A.add_array("rest", gid.size, 3)
        A.set_array(x, case.x[gid])
        A.set_array(rest, case.X[gid])
        g2l = np.full(case.n_nodes, -1, dtype=np.int64)
        g2l[gid] = np.arange(gid.size)
        for name, sel in (("elastic", t.own), ("elastic_ghost", t.ghost)):
            cid = A.add_connectivity(name, 4)
            A.set_elements(cid, g2l[case.conn[sel]].reshape(-1, 4))
            A.add_energy(name, cid, tapes("tet4_elastic"), solid_tet_inputs(x, rest), range(12),
                         params={24: p["mu"], 25: p["lambda"]}, flags=flags)
        xp = A.add_array("x_prev", gid.size, 3)
        v = A.add_array("v", gid.size, 3)
        m = A.add_array("mass", gid.size, 1)
        A.set_array(xp, ex["x_prev"][gid])
        A.set_array(v, ex["v"][gid])
        A.set_array(m, ex["mass"][gid])
        vc = A.add_connectivity("verts", 1)
        A.set_elements(vc, np.arange(t.row_lo, t.row_hi, dtype=np.int64))
        A.add_energy("inertia", vc, tapes("inertia"), inertia_inputs(x, xp, v, m), range(3))
        self.pairs = None
        if sh.pairs.size:
            B = self.pairs = DeviceAssembler(device)
            px = B.add_array("x", sh.pair_nodes.size, 3, True)
            B.set_array(px, case.x[sh.pair_nodes])
            po = B.add_array("pair_offset", sh.pairs.size, 12)
            B.set_array(po, ex["offsets"][sh.pairs])
            pc = B.add_connectivity("pairs", 4)
            B.set_elements(pc, sh.pair_conn)
            B.add_energy("contact", pc, tapes("contact"), contact_inputs(px, po), range(12),
                         act_tape=tapes("contact_act"), act_kind=0, guard_tape=tapes("contact_guard"),
                         params={24: p["kappa"], 25: p["dhat"]}, flags=flags | ENERGY_EXACT)

    def n_owned_elements(self) -> int:
        t = self.sh.tet
        return t.n_own + (t.row_hi - t.row_lo) + int(self.sh.pairs.size)

    def assemble(self, mode: str = "deterministic"):
        """(owned energy, owned rows of context 1, send lists of the pair rows per rank)."""
        t, A = self.sh.tet, self.main
        A.assemble(mode)
        parts = A.energy_parts()  # [own tets, ghost tets, inertia]
        e_own = float(parts[0] + parts[2])
        H = A.hessian()
        own = owned_rows(H.b, H.row_ptr, H.col_idx, H.values, A.gradient(), t.row_lo, t.row_hi, t.global_ids)
        if self.pairs is None:
            empty = (np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 3, 3)), np.zeros(0, np.int64),
                     np.zeros((0, 3)))
            return e_own, own, [empty] * self.world
        e_own += self.pairs.assemble(mode)
        P = self.pairs.hessian()
        send = split_rows_by_owner(P.b, P.row_ptr, P.col_idx, P.values, self.pairs.gradient(), self.sh.pair_nodes,
                                   self.sh.node_bounds)
        return e_own, own, send

    def finish(self, own, incoming):
        b = self.sh.node_bounds
        return merge_owned_rows(3, own, incoming, int(b[self.rank]), int(b[self.rank + 1]))
