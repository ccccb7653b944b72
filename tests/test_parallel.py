"""Sharded (owner-computes) assembly, DESIGN.md §6 / SURVEY 8(e); config 5's contact pairs
owned by their point node's rank with one exchange of the rows they touch elsewhere.

CPU, gloo, world sizes 2 and 3: every rank builds its shard (owned + ghost elements, local
nodes), assembles it with the C oracle as the element engine (own and ghost as two energies,
exactly as the device ShardedTetSystem registers them), keeps its owned block rows and
all-reduces its owned energy. The gathered rows must equal the global assembly: pattern
bit-exact, values to 1e-13 (only the summation order differs), E to 1e-12.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200 import parallel as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_shard_rows(x, X, conn, n_own, params, row_lo, row_hi, gids):
    """One rank's owned rows and owned energy with the C oracle (test-side engine)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from conftest import golden_tape
    from oracle import oracle as O
    from paper_2303_02156_b200 import systems as S
    sysm = O.System()
    xa = sysm.add_array("x", x, 3, True)
    ra = sysm.add_array("rest", X, 3)
    sysm.add_energy("elastic", conn[:n_own], 4, golden_tape("tet4_elastic"), S.solid_tet_inputs(xa, ra), range(12),
                    params={24: params["mu"], 25: params["lambda"]})
    if n_own < conn.shape[0]:
        sysm.add_energy("elastic_ghost", conn[n_own:], 4, golden_tape("tet4_elastic"), S.solid_tet_inputs(xa, ra),
                        range(12), params={24: params["mu"], 25: params["lambda"]})
    r = sysm.assemble()
    e_own = sysm.element_outputs(0, 0, n_own)[:, 0].sum() if n_own else 0.0
    return P.owned_rows(3, r["row_ptr"], r["col_idx"], r["vals"], r["grad"], row_lo, row_hi, gids), e_own


def _oracle_contact_rank(case, sh, world, rank):
    """One rank of the sharded config-5 assembly with the C oracle as element engine:
    tets own + ghost and inertia over owned nodes (owned rows complete), plus the pairs this
    rank owns (point node p), whose rows owned elsewhere are exchanged."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from conftest import golden_tape
    from oracle import oracle as O
    from paper_2303_02156_b200 import systems as S
    p, ex, t = case.params, case.extra, sh.tet
    gid = t.global_ids
    m = O.System()
    xa = m.add_array("x", case.x[gid], 3, True)
    ra = m.add_array("rest", case.X[gid], 3)
    own, ghost = case.conn[t.own], case.conn[t.ghost]
    g2l = {g: i for i, g in enumerate(gid)}
    loc = lambda c: np.vectorize(g2l.get)(c) if c.size else c.reshape(-1, 4)
    m.add_energy("elastic", loc(own), 4, golden_tape("tet4_elastic"), S.solid_tet_inputs(xa, ra), range(12),
                 params={24: p["mu"], 25: p["lambda"]})
    m.add_energy("elastic_ghost", loc(ghost), 4, golden_tape("tet4_elastic"), S.solid_tet_inputs(xa, ra), range(12),
                 params={24: p["mu"], 25: p["lambda"]})
    pa = m.add_array("x_prev", ex["x_prev"][gid], 3)
    va = m.add_array("v", ex["v"][gid], 3)
    ma = m.add_array("mass", ex["mass"][gid], 1)
    m.add_energy("inertia", np.arange(t.row_lo, t.row_hi), 1, golden_tape("inertia"), S.inertia_inputs(xa, pa, va, ma),
                 range(3))
    r = m.assemble()
    assert r["status"] == 0
    outs_own = m.element_outputs(0, 0, own.shape[0])[:, 0].sum() if own.size else 0.0
    outs_in = m.element_outputs(2, 0, t.row_hi - t.row_lo)[:, 0].sum()
    own_rows = P.owned_rows(3, r["row_ptr"], r["col_idx"], r["vals"], r["grad"], t.row_lo, t.row_hi, gid)
    # owned pairs on their own node set
    pm = O.System()
    pxa = pm.add_array("x", case.x[sh.pair_nodes], 3, True)
    poa = pm.add_array("pair_offset", ex["offsets"][sh.pairs], 12)
    pm.add_energy("contact", sh.pair_conn, 4, golden_tape("contact"), S.contact_inputs(pxa, poa), range(12),
                  params={24: p["kappa"], 25: p["dhat"]}, act_tape=golden_tape("contact_act"), act_kind=0,
                  guard_tape=golden_tape("contact_guard"))
    if sh.pairs.size:
        pr = pm.assemble()
        assert pr["status"] == 0
        send = P.split_rows_by_owner(3, pr["row_ptr"], pr["col_idx"], pr["vals"], pr["grad"], sh.pair_nodes,
                                     sh.node_bounds)
        e_pairs = pr["E"]
    else:
        send = [(np.zeros(0, np.int64),) * 2 + (np.zeros((0, 3, 3)), np.zeros(0, np.int64), np.zeros((0, 3)))] * world
        e_pairs = 0.0
    incoming = P.exchange(send)
    rows = P.merge_owned_rows(3, own_rows, incoming, int(sh.node_bounds[rank]), int(sh.node_bounds[rank + 1]))
    return rows, outs_own + outs_in + e_pairs, t.n_own + sh.pairs.size + (t.row_hi - t.row_lo)


def _worker(rank, world, port, q, mode):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = P.max_over_ranks(1.5 + rank)
        if mode == "slab":   # the bench's slab generator (x-extended Kuhn grid)
            s = C.tet4_slab_case(3, world, rank)
            rows, e_own = _oracle_shard_rows(s.case.x, s.case.X, s.case.conn, s.n_own, s.case.params,
                                             s.row_lo, s.row_hi, s.global_ids)
            n_own = s.n_own
        elif mode == "contact":  # config 5: tets + inertia owner-computes, pairs by point owner
            case = C.config5(3, 80)
            sh = P.contact_shard(case.conn, case.extra["pairs"], case.n_nodes, world, rank)
            rows, e_own, n_own = _oracle_contact_rank(case, sh, world, rank)
        else:                # generic owner_shard of a global mesh
            case = C.config2(4)
            sh = P.owner_shard(case.conn, case.n_nodes, world, rank)
            rows, e_own = _oracle_shard_rows(case.x[sh.global_ids], case.X[sh.global_ids], sh.conn, sh.n_own,
                                             case.params, sh.row_lo, sh.row_hi, sh.global_ids)
            n_own = sh.n_own
        E = P.sum_over_ranks(e_own)
        n_tot = P.sum_over_ranks(n_own)
        allrows = [None] * world
        dist.all_gather_object(allrows, rows)
        if rank == 0:
            from conftest import golden_tape
            from oracle import oracle as O
            case = (C.tet4_global_slab_case(3, world) if mode == "slab" else
                    C.config5(3, 80) if mode == "contact" else C.config2(4))
            ref = O.system_for_case(case, golden_tape).assemble()
            rp, ci, v, g = P.gather_rows(allrows)
            n_ref = case.conn.shape[0] + (case.extra["pairs"].shape[0] + case.n_nodes if mode == "contact" else 0)
            q.put(dict(t=t, n_tot=n_tot, n_ref=n_ref, E=E, Eref=ref["E"],
                       pat=bool(np.array_equal(rp, ref["row_ptr"]) and np.array_equal(ci, ref["col_idx"])),
                       dH=float(np.abs(v.ravel() - ref["vals"]).max() / max(1.0, np.abs(ref["vals"]).max())),
                       dg=float(np.abs(g - ref["grad"]).max() / max(1.0, np.abs(ref["grad"]).max()))))
        else:
            q.put(dict(rank=rank))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "slab"), (3, "slab"), (2, "generic"), (3, "generic"), (2, "contact"),
                                        (3, "contact"), (4, "contact")])
def test_gloo_owner_computes_matches_global(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    main = [r for r in res if "E" in r][0]
    assert main["t"] == 0.5 + world              # max over ranks
    assert main["n_tot"] == main["n_ref"]        # every element owned exactly once
    assert main["pat"]                           # owned rows reproduce the global pattern exactly
    assert abs(main["E"] - main["Eref"]) <= 1e-12 * max(1.0, abs(main["Eref"]))
    # (contact: pair blocks are summed after the tet + inertia part, not in energy order)
    tol = 1e-12 if mode == "contact" else 1e-13
    assert main["dH"] <= tol and main["dg"] <= tol


def test_owner_shard_cover_and_ghosts():
    case = C.config2(4)
    for world in (1, 2, 3, 4):
        owned_el, owned_nodes = [], []
        for r in range(world):
            sh = P.owner_shard(case.conn, case.n_nodes, world, r)
            owned_el.append(sh.own)
            owned_nodes.append(sh.global_ids[sh.row_lo:sh.row_hi])
            assert np.array_equal(sh.global_ids[sh.row_lo:sh.row_hi], np.arange(sh.node_lo, sh.node_hi))
            # every element touching an owned node is evaluated here (own or ghost)
            touch = np.flatnonzero(((case.conn >= sh.node_lo) & (case.conn < sh.node_hi)).any(1))
            assert np.array_equal(np.union1d(sh.own, sh.ghost), np.union1d(touch, sh.own))
            assert np.intersect1d(sh.own, sh.ghost).size == 0
        assert np.array_equal(np.sort(np.concatenate(owned_el)), np.arange(case.conn.shape[0]))
        assert np.array_equal(np.concatenate(owned_nodes), np.arange(case.n_nodes))


def test_slab_generator_is_owner_shard_of_the_global_grid():
    world, n = 3, 3
    g = C.tet4_global_slab_case(n, world)
    for r in range(world):
        s = C.tet4_slab_case(n, world, r)
        gc = s.global_ids[s.case.conn]
        per_plane = 6 * n * n
        assert np.array_equal(gc[:s.n_own], g.conn[r * n * per_plane:(r + 1) * n * per_plane])
        assert np.array_equal(g.x[s.global_ids], s.case.x)
        lo, hi = s.global_ids[s.row_lo], s.global_ids[s.row_hi - 1] + 1
        ghost_ref = np.flatnonzero(((g.conn >= lo) & (g.conn < hi)).any(1) & ((g.conn[:, 0] < lo) | (g.conn[:, 0] >= hi)))
        assert np.array_equal(np.sort(gc[s.n_own:], axis=None), np.sort(g.conn[ghost_ref], axis=None))
