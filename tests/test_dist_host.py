"""Host logic of the slab decomposition on CPU: the partition exported by
the C ABI, the per-rank slicing of the global inputs, and the world_size-2 bootstrap over
torch.distributed (gloo): NCCL id broadcast, partition agreement, max-over-ranks timing."""

import os
import socket

import numpy as np
import pytest

import paper_1909_13585_b200 as mg
from paper_1909_13585_b200 import MgError
from paper_1909_13585_b200.dist import local_inputs, rank_part
from workloads import generate, get_config


@pytest.mark.parametrize("nel,levels", [((1920, 960), 7), ((480, 240), 5), ((96, 48, 48), 4), ((256, 128, 128), 5),
                                        ((64, 32), 3)])
@pytest.mark.parametrize("S", [1, 2, 3, 4, 8])
def test_partition_tiles_axis0_at_coarsest_boundaries(nel, levels, S):
    f = 2 ** (levels - 1)
    if nel[0] // f < S:
        with pytest.raises(MgError):
            mg.mg_partition(nel, levels, S, 0)
        return
    parts = [mg.mg_partition(nel, levels, S, k) for k in range(S)]
    assert parts[0][0] == 0 and parts[-1][1] == nel[0]
    for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
        assert a1 == b0
    sizes = [b - a for a, b in parts]
    assert all(s > 0 and s % f == 0 for s in sizes)
    assert max(sizes) - min(sizes) <= f
    for a, b in parts:
        assert a % f == 0 and b % f == 0


def test_partition_rejects_bad_arguments():
    with pytest.raises(MgError):
        mg.mg_partition((30, 16), 3, 2, 0)          # 30 not divisible by 4
    with pytest.raises(MgError):
        mg.mg_partition((64, 32), 3, 4, 4)          # part out of range


@pytest.mark.parametrize("name,nranks,nslab", [("T2b", 2, 1), ("T2c", 3, 2), ("T3b", 3, 1), ("T3c", 2, 2)])
def test_rank_parts_reassemble_the_global_inputs(name, nranks, nslab):
    cfg = get_config(name)
    inp = generate(cfg)
    parts = [rank_part(cfg.nel, cfg.levels, nranks, r, nslab) for r in range(nranks)]
    loc = [local_inputs(inp, p) for p in parts]
    for key in ("E", "Es"):
        assert np.array_equal(np.concatenate([l[key] for l in loc]), inp[key])
    assert np.array_equal(np.concatenate([l["fixed"] for l in loc]), inp["fixed"])
    assert np.array_equal(np.concatenate([l["rhs"] for l in loc], axis=1), inp["rhs"])
    assert parts[0].e_begin == 0 and parts[-1].e_end == cfg.nel[0]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_1909_13585_b200.dist import bootstrap_nccl_id
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = get_config("C3")
    p = rank_part(cfg.nel, cfg.levels, world, rank)
    nid = bootstrap_nccl_id(rank, world)
    ids = [None] * world
    dist.all_gather_object(ids, nid)
    parts = [None] * world
    dist.all_gather_object(parts, (p.e_begin, p.e_end, p.dof0, p.dof1))
    # bench.py's timing reduction: max over ranks of the per-rank device time
    t = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    units = torch.tensor([float(p.dof1 - p.dof0)], dtype=torch.float64)
    dist.all_reduce(units, op=dist.ReduceOp.SUM)
    # bench.py's N > 1 self-check gathers every rank's owned slice of x into the global vector
    from paper_1909_13585_b200.dist import gather_owned
    n = 2 * (cfg.nel[0] + 1) * (cfg.nel[1] + 1)
    glob = torch.arange(3 * n, dtype=torch.float64).reshape(3, n)
    full = gather_owned(glob[:, p.dof0:p.dof1].clone(), p, n)
    gathered_ok = bool(torch.equal(full, glob))
    out.put((rank, ids, parts, float(t.item()), float(units.item()), gathered_ok))
    dist.destroy_process_group()


def test_two_rank_gloo_bootstrap():
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, ids0, parts0, t0, u0, g0), (_, ids1, parts1, t1, u1, g1) = res
    assert g0 and g1
    assert ids0 == ids1 and ids0[0] == ids0[1] and len(ids0[0]) == 128
    assert parts0 == parts1
    (a0, a1, d0, d1), (b0, b1, e0, e1) = parts0
    cfg = get_config("C3")
    n = 2 * (cfg.nel[0] + 1) * (cfg.nel[1] + 1)
    assert a0 == 0 and a1 == b0 and b1 == cfg.nel[0] and d1 == e0 and e1 == n and d0 == 0
    assert t0 == t1 == 11.0 and u0 == u1 == n
