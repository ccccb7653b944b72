"""Sharded (owner-computes) assembly, DESIGN.md §6 / SURVEY 8(e).

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
            case = C.tet4_global_slab_case(3, world) if mode == "slab" else C.config2(4)
            ref = O.system_for_case(case, golden_tape).assemble()
            rp, ci, v, g = P.gather_rows(allrows)
            q.put(dict(t=t, n_tot=n_tot, n_ref=case.conn.shape[0], E=E, Eref=ref["E"],
                       pat=bool(np.array_equal(rp, ref["row_ptr"]) and np.array_equal(ci, ref["col_idx"])),
                       dH=float(np.abs(v.ravel() - ref["vals"]).max() / max(1.0, np.abs(ref["vals"]).max())),
                       dg=float(np.abs(g - ref["grad"]).max() / max(1.0, np.abs(ref["grad"]).max()))))
        else:
            q.put(dict(rank=rank))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "slab"), (3, "slab"), (2, "generic"), (3, "generic")])
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
    assert main["dH"] <= 1e-13 and main["dg"] <= 1e-13


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
