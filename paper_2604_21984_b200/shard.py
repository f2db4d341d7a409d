"""Multi-GPU partitioning of the fitting workload, host-side logic.

* Config 4 — a batch of independent images: images are dealt to ranks; every rank fits its own
  images with no data-path collective (weak scaling), and the only communication is the timing /
  result reduction (`max_over_ranks`, `sum_over_ranks`) through torch.distributed (NCCL on B200s,
  gloo in the CPU tests).
* Config 5 — one large image in row strips (sad_fit_run_strips): `strip_bounds` / `halo_rows` give
  each rank's strip and the rows it fetches before a propagation pass at jump `step`.  The strip map
  is partition-invariant (the injection stream is keyed by the global (pass_index, cell)) and the
  gradient / stats partials are merged exactly, so every rank reproduces the single-GPU fit.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def assign_images(n_images: int, world: int, rank: int) -> List[int]:
    """Indices of the images rank `rank` fits: contiguous blocks of ceil(n/world) (block-cyclic for
    n < world, where the trailing ranks get nothing)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = (n_images + world - 1) // world
    return list(range(rank * per, min(n_images, (rank + 1) * per)))


def image_seeds(n_images_per_rank: int, world: int, rank: int, base_seed: int = 1) -> List[int]:
    """Weak scaling: every rank fits `n_images_per_rank` images with globally distinct seeds."""
    return [base_seed + rank * n_images_per_rank + i for i in range(n_images_per_rank)]


def strip_bounds(height: int, world: int, rank: int) -> Tuple[int, int]:
    """Row strip [y0, y1) of `rank` (the partition of sad_fit_run_strips, sad_runtime.cu strip_bounds):
    balanced, contiguous, every boundary a multiple of the 8-row backward / stats tiles."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    tiles = (height + 7) // 8

    def b(q):
        return min(height, 8 * (tiles * q // world))
    return b(rank), b(rank + 1)


def halo_rows(height: int, world: int, rank: int, step: int) -> List[Tuple[int, int, int]]:
    """Rows outside this rank's strip that a pass at jump `step` reads (Axial and Box3 read rows y - step
    and y + step): the bands [y0 - step, y0) and [y1, y1 + step), grouped by owner rank as
    [(owner_rank, row0, row1), ...] -- what sad_fit_run_strips fetches before the pass."""
    y0, y1 = strip_bounds(height, world, rank)
    out = []
    for owner in range(world):
        if owner == rank:
            continue
        o0, o1 = strip_bounds(height, world, owner)
        for lo, hi in ((max(0, y0 - step), y0), (y1, min(height, y1 + step))):
            a, b = max(lo, o0), min(hi, o1)
            if b > a:
                out.append((owner, a, b))
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (timing: the slowest rank defines the job time)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_counts(counts: Sequence[int], device=None) -> List[int]:
    """Element-wise sum of per-rank integer vectors (e.g. images fitted per rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(counts), dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) for x in t.tolist()]
