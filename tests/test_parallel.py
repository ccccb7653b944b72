"""CPU, world_size 2 over gloo: the multi-process plumbing (max-over-ranks timing) and the
sharded-assembly decomposition checked against the global oracle assembly."""
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


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from conftest import golden_tape
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # max over ranks
        t = P.max_over_ranks(1.5 + rank)
        # sharded assembly: each rank assembles the elements it owns, dense, then sum
        case = C.config2(3)
        shards = P.slab_partition(case.conn, case.n_nodes, world)
        mine = shards[rank]
        sub = C.Case("shard", "tet4", case.x, case.X, case.conn[mine.elements], case.params)
        r = O.system_for_case(sub, golden_tape).assemble()
        from paper_2303_02156_b200.device import Bcrs
        D = Bcrs(3, r["row_ptr"], r["col_idx"], r["vals"]).to_dense()
        g = r["grad"].copy()
        # rows this rank writes outside its slab are exactly its halo rows
        touched_rows = np.unique(np.nonzero(D)[0] // 3)
        foreign = touched_rows[(touched_rows < mine.node_lo) | (touched_rows >= mine.node_hi)]
        halo_ok = set(foreign.tolist()) <= set(mine.halo_nodes.tolist())
        tD = torch.from_numpy(D)
        tg = torch.from_numpy(g)
        tE = torch.tensor([r["E"]], dtype=torch.float64)
        dist.all_reduce(tD)
        dist.all_reduce(tg)
        dist.all_reduce(tE)
        n_el = torch.tensor([mine.elements.size], dtype=torch.int64)
        dist.all_reduce(n_el)
        if rank == 0:
            ref = O.system_for_case(case, golden_tape).assemble()
            Dref = Bcrs(3, ref["row_ptr"], ref["col_idx"], ref["vals"]).to_dense()
            q.put(dict(t=t, E=float(tE.item()), Eref=ref["E"], dH=float(np.abs(tD.numpy() - Dref).max() / np.abs(Dref).max()),
                       dg=float(np.abs(tg.numpy() - ref["grad"]).max()), n_el=int(n_el.item()), n_total=case.conn.shape[0],
                       halo_ok=halo_ok))
        else:
            q.put(dict(halo_ok=halo_ok))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_assembly_matches_global():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    main = [r for r in res if "E" in r][0]
    assert main["t"] == 2.5                       # max over ranks
    assert main["n_el"] == main["n_total"]        # every element owned exactly once
    assert all(r["halo_ok"] for r in res)
    assert abs(main["E"] - main["Eref"]) <= 1e-12 * max(1.0, abs(main["Eref"]))
    assert main["dH"] <= 1e-13 and main["dg"] <= 1e-9


def test_slab_partition_covers_and_halos():
    case = C.config2(4)
    for world in (1, 2, 3, 4):
        sh = P.slab_partition(case.conn, case.n_nodes, world)
        all_el = np.concatenate([s.elements for s in sh])
        assert np.array_equal(np.sort(all_el), np.arange(case.conn.shape[0]))
        for s in sh:
            assert np.all((s.halo_nodes < s.node_lo) | (s.halo_nodes >= s.node_hi))
