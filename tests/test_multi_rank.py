"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic:
image sharding and the timing/result reductions the bench uses, plus the row-strip / halo
geometry for the tiled large-image mode."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_21984_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_21984_b200 as sad
    from oracle.bindings import c_backend
    from tests.fixtures import synth_target
    B = c_backend()
    seeds = shard.image_seeds(2, world, rank)
    psnrs = []
    for sd in seeds:  # each rank fits its own images: no data-path collective
        r = B.fit(synth_target(24, 16, sd), sad.TrainConfig(iters=8, n_sites=24, fp64=False, seed=sd))
        psnrs.append(r.history[-1].psnr)
    slow = shard.max_over_ranks(1.0 + rank)
    total = shard.sum_over_ranks(len(seeds))
    counts = shard.gather_counts([len(seeds) if r == rank else 0 for r in range(world)])
    out.put((rank, seeds, psnrs, slow, total, counts))
    dist.barrier()
    dist.destroy_process_group()


def test_image_sharding_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    seeds = [s for r in res for s in r[1]]
    assert sorted(seeds) == list(range(1, 1 + 2 * world))  # every image exactly once
    for r in res:
        assert r[3] == float(world)  # max over ranks
        assert r[4] == 2.0 * world
        assert r[5] == [2] * world
        assert all(np.isfinite(r[2]))
    # determinism: the same image fitted by rank 0 alone gives the same PSNR
    import paper_2604_21984_b200 as sad
    from oracle.bindings import c_backend
    from tests.fixtures import synth_target
    alone = c_backend().fit(synth_target(24, 16, 1), sad.TrainConfig(iters=8, n_sites=24, fp64=False, seed=1))
    assert alone.history[-1].psnr == res[0][2][0]


def test_assign_images_covers_batch():
    for n in (1, 3, 24, 25):
        for world in (1, 2, 4, 8):
            got = sorted(i for r in range(world) for i in shard.assign_images(n, world, r))
            assert got == list(range(n))


@pytest.mark.parametrize("height,world", [(512, 2), (512, 8), (8192, 8), (37, 4)])
def test_strips_and_halos(height, world):
    bounds = [shard.strip_bounds(height, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == height
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
    assert all(b[0] % 8 == 0 for b in bounds)  # tile-aligned (8-row backward / stats tiles)
    for step in (1, 2, 16, 1024):
        for r in range(world):
            y0, y1 = bounds[r]
            # every row a pass at `step` reads outside the strip is fetched (the fetched bands cover it)
            need = {ny for y in range(y0, y1) for ny in (y - step, y + step)
                    if 0 <= ny < height and not (y0 <= ny < y1)}
            want = {ny for ny in list(range(max(0, y0 - step), y0)) + list(range(y1, min(height, y1 + step)))}
            assert need <= want
            got = set()
            for owner, a, b in shard.halo_rows(height, world, r, step):
                o0, o1 = bounds[owner]
                assert o0 <= a < b <= o1 and owner != r
                got |= set(range(a, b))
            assert got == want
