"""Host logic of the N > 1 slab path on CPU: world_size 2 with the gloo backend.

Each rank asks the library (host-only C-ABI call, no device) for its slab of cfg 4 / cfg 5,
the ranks all-gather the partitions and check that (i) the owned rows tile the axis exactly,
(ii) every halo row a rank needs is owned by its neighbour (what the NCCL send/recv of
bsde_step moves), and (iii) the 128-byte NCCL id broadcast used by paper_1909_13560_b200.dist
round-trips through torch.distributed.
"""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1909_13560_b200 import query_partition, workloads as W
    from paper_1909_13560_b200.dist import broadcast_id
    res = {}
    for name, spec in [("cfg4", W.cfg4()), ("cfg5", W.basket_3d()), ("ex4", W.ex4_2d(3, 8, npts=257))]:
        mine = query_partition(spec, world, rank)
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        res[name] = allp
    fake = bytes((7 * i + 3) % 256 for i in range(128)) if rank == 0 else None
    got = broadcast_id(fake, rank)
    res["id_ok"] = got == bytes((7 * i + 3) % 256 for i in range(128))
    if rank == 0:
        out.put(res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_partition_and_id_broadcast_gloo(world):
    from paper_1909_13560_b200 import build as b
    b.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["id_ok"]
    from paper_1909_13560_b200 import workloads as W
    for name, spec in [("cfg4", W.cfg4()), ("cfg5", W.basket_3d()), ("ex4", W.ex4_2d(3, 8, npts=257))]:
        parts = res[name]
        P0 = int(spec["npts"][0])
        assert parts[0]["own_lo"] == 0 and parts[-1]["own_hi"] == P0
        for a, b2 in zip(parts, parts[1:]):
            assert a["own_hi"] == b2["own_lo"]                      # exact tiling
            # rank r+1's lower halo rows [slab_lo, own_lo) are owned by rank r, and vice versa
            assert a["own_lo"] <= b2["slab_lo"] < b2["own_lo"]
            assert a["own_hi"] < a["slab_hi"] <= b2["own_hi"]
            assert b2["own_lo"] - b2["slab_lo"] == min(b2["own_lo"], b2["halo"])
            assert a["slab_hi"] - a["own_hi"] == min(P0 - a["own_hi"], a["halo"])
        for p in parts:
            assert p["halo"] >= 4                                   # cubic support (SPIKE: coefficient halo)


def test_spike_halo_is_reach_plus_stencil():
    """SPIKE (default) exchanges reach + 3 rows of final coefficients; the redundant-halo
    ablation adds the PCR decay rows (31) and the not-a-knot / ghost rows (6) of values."""
    from paper_1909_13560_b200 import query_partition, workloads as W
    for spec, Rs in ((W.cfg4(), (2, 4, 8)), (W.basket_3d(), (2, 4, 8)), (W.ex4_2d(3, 8, npts=257), (2,))):
        for R in Rs:
            a = query_partition(spec, R, 1)
            b = query_partition(dict(spec, slab_spline=1), R, 1)
            assert b["halo"] - a["halo"] == 37
            assert a["own_lo"] == b["own_lo"] and a["own_hi"] == b["own_hi"]


def test_partition_rejects_thin_slabs():
    from paper_1909_13560_b200 import query_partition, BsdeError, workloads as W
    with pytest.raises(BsdeError) as ei:
        query_partition(dict(W.basket_3d(P=128), slab_spline=1), 8, 0)   # 16 planes < values halo
    assert ei.value.code == 1
    with pytest.raises(BsdeError) as ei:
        query_partition(W.basket_3d(P=32), 8, 0)                   # 4 planes < coefficient halo
    assert ei.value.code == 1
    with pytest.raises(BsdeError):
        query_partition(W.cfg2(6), 2, 0)                           # 1-D runs as replicas
