"""Multi-rank host logic on CPU (gloo, world_size 2).

The GPU path shards frames into row slabs with r-row halos taken from the
host copy (filter_image(devices=[...]), bench.py under torchrun) and
batches into runs of images (filter_images, config 5), and never exchanges
data between ranks.  These tests run the PRODUCT's planners
(paper_1105_3829_b200.plan_slabs / plan_images -- the ones filter_image,
filter_images and bench.py use) with two gloo ranks on the CPU: each rank
computes its share with the CPU oracle (standing in for one device -- the
kernels themselves are covered by the -m gpu suite) and the gathered frame
must equal the single-rank result (reference band identity,
engine.py:243-262).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import workloads


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, px, radius, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1105_3829_b200 import plan_slabs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H = px.shape[0]
    sl = plan_slabs(H, world, radius)[rank]
    a, b, top, bot = sl
    # halo rows straight from the host copy, clamped at the global edges
    assert (top, bot) == (max(0, a - radius), min(H, b + radius))
    local = O.iot_filter(px[top:bot], 2 * radius + 1)[a - top:b - top]
    # timing-style reduction used by bench.py: max over ranks
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, (a, b, local))
    if rank == 0:
        q.put((float(t.item()), gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("radius", [2, 7])
def test_two_rank_slabs_reassemble_frame(radius):
    px = workloads.cfg2_blur_sp_u8(61, 47)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, px, radius, q)) for r in range(world)]
    for p in procs:
        p.start()
    tmax, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == float(world)
    out = np.empty_like(px)
    for a, b, local in gathered:
        out[a:b] = local
    from oracle import oracle as O

    assert np.array_equal(out, O.iot_filter(px, 2 * radius + 1))


def test_weak_scaling_slab_geometry():
    """bench.py's weak-scaling layout: rank k owns rows [kH,(k+1)H) of N stacked
    copies; its source slab is those rows plus r halo rows (clamped)."""
    H = 16
    base = np.arange(H * 3, dtype=np.uint8).reshape(H, 3)
    for world in (1, 2, 4, 8):
        Hg = H * world
        for rank in range(world):
            a, b = rank * H, (rank + 1) * H
            r = 5
            top, bot = max(0, a - r), min(Hg, b + r)
            slab = base[np.arange(top, bot) % H]
            assert slab.shape[0] == bot - top
            assert np.array_equal(slab[a - top:b - top], base)


def _batch_worker(rank, world, port, batch, radius, q):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1105_3829_b200 import plan_images

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    i0, i1 = plan_images(batch.shape[0], world)[rank]
    local = [(i, O.iot_filter(batch[i], 2 * radius + 1)) for i in range(i0, i1)]
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_batch_split_covers_every_image():
    """Config 5's split: plan_images gives each rank a contiguous run of
    images; the union over ranks is every image exactly once and the
    gathered outputs equal the single-rank results."""
    batch = workloads.cfg5_batch_u8(5, 40, 36)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, batch, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle as O

    got = {i: o for part in gathered for i, o in part}
    assert sorted(got) == list(range(5))
    for i in range(5):
        assert np.array_equal(got[i], O.iot_filter(batch[i], 7))


def test_planners():
    from paper_1105_3829_b200 import plan_images, plan_slabs

    for H in (1, 7, 100, 8192):
        for parts in (1, 2, 3, 8):
            for r in (0, 3, 63):
                sl = plan_slabs(H, parts, r)
                assert sl[0].a == 0 and sl[-1].b == H
                assert all(x.b == y.a for x, y in zip(sl, sl[1:]))
                assert all(s.top == max(0, s.a - r) and s.bot == min(H, s.b + r) for s in sl)
                assert len(sl) == min(parts, H)
    for count in (0, 1, 5, 64):
        for parts in (1, 2, 3, 8):
            runs = plan_images(count, parts)
            assert len(runs) == parts
            assert [i for a, b in runs for i in range(a, b)] == list(range(count))
            sizes = [b - a for a, b in runs]
            assert max(sizes) - min(sizes) <= 1
