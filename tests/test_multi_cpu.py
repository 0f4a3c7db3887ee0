"""Host logic of the multi-GPU slab decomposition on CPU: the partition (C-ABI host helper),
the B1 plane binning used to cut slabs, and a world-size-2 gloo run of the bootstrap and of the
partition agreement between ranks."""
import os
import socket

import numpy as np
import pytest

import workloads


@pytest.fixture(scope="module")
def crm():
    from paper_2507_05643_b200 import build
    build.build_library()
    from paper_2507_05643_b200 import crm as m
    m.load_library()
    return m


def test_partition_balances_and_aligns(crm):
    rng = np.random.default_rng(0)
    for world in (2, 3, 4, 8):
        counts = rng.integers(0, 1000, 97)
        b = crm.slab_partition(counts, world, 2)
        assert b[0] == 0 and b[-1] == 97 and np.all(np.diff(b) >= 2)
        assert np.all(b[1:-1] % 2 == 0)
        per = np.add.reduceat(counts, b[:-1])
        # each slab within two planes' worth of the ideal share
        assert np.all(np.abs(per - counts.sum() / world) <= 2 * counts.max() + 1)


def test_partition_uniform_bed_is_even(crm):
    counts = np.full(400, 1000)
    b = crm.slab_partition(counts, 8, 2)
    assert list(np.diff(b)) == [50] * 8


def test_partition_too_narrow(crm):
    with pytest.raises(crm.CrmError):
        crm.slab_partition(np.ones(7, np.int64), 4, 2)


def test_plane_binning_matches_b1():
    from paper_2507_05643_b200 import dist
    sc = workloads.bed(n=(64, 16, 8))
    lo, cell, n = dist.grid_planes(sc.params)
    allp = np.concatenate([sc.fluid_pos, sc.wall_pos])
    c = dist.plane_counts(allp, lo, cell, n)
    assert c.sum() == len(allp)
    # B1 on fp32: floor(fdiv(fsub(x, lo), s)) — a particle exactly on a face goes to the higher plane
    x = np.array([[lo + 3 * cell, 0, 0]])
    p = dist.plane_counts(x, lo, cell, n)
    assert np.nonzero(p)[0][0] in (2, 3)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_05643_b200 import crm as m
        from paper_2507_05643_b200 import dist as cd
        import torch
        # every rank sees the same global input and must cut the same slabs
        sc = workloads.bed(n=(96, 16, 8))
        lo, cell, n = cd.grid_planes(sc.params)
        counts = cd.plane_counts(np.concatenate([sc.fluid_pos, sc.wall_pos]), lo, cell, n)
        b = m.slab_partition(counts, world, 2)
        allb = [None] * world
        dist.all_gather_object(allb, b.tolist())
        own = torch.tensor([int(counts[b[rank]:b[rank + 1]].sum())])
        dist.all_reduce(own)
        # the NCCL id bootstrap (rank 0 creates, the group broadcasts)
        try:
            nid = cd.bootstrap_nccl_id(rank)
        except m.CrmError:
            nid = b"unavailable"
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        q.put((rank, allb, int(own.item()), int(counts.sum()), len(set(ids)), len(nid)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition_agreement_and_bootstrap():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, allb, own, total, n_ids, id_len in res:
        assert allb[0] == allb[1]                 # identical slabs on every rank
        assert own == total                       # the slabs cover every particle exactly once
        assert n_ids == 1                         # every rank holds the same NCCL id
        assert id_len in (128, len(b"unavailable"))
