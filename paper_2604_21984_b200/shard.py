"""Multi-GPU partitioning of the fitting workload, host-side logic.

* Config 4 — a batch of independent images: images are dealt to ranks; every rank fits its own
  images with no data-path collective (weak scaling), and the only communication is the timing /
  result reduction (`max_over_ranks`, `sum_over_ranks`) through torch.distributed (NCCL on B200s,
  gloo in the CPU tests).
* Config 5 — one large image in row strips: `strip_bounds` / `halo_rows` give each rank's strip and
  the neighbour rows a propagation pass at jump step `step` reads (Axial: rows y +- step; Box3: the
  same rows, three columns).  The strip map is deterministic and partition-invariant: the injection
  stream is keyed by the global (pass_index, cell), so a strip rank reproduces exactly the rows a
  single-GPU pass would produce.
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
    """Row strip [y0, y1) of `rank` for a `height`-row grid (balanced, contiguous)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    y0 = height * rank // world
    y1 = height * (rank + 1) // world
    return y0, y1


def halo_rows(height: int, world: int, rank: int, step: int) -> List[Tuple[int, int, int]]:
    """Rows outside this rank's strip that a pass at jump `step` reads, grouped by owner rank:
    [(owner_rank, row0, row1), ...] with [row0, row1) inside the owner's strip.  Axial and Box3
    stencils read the same rows (y - step, y + step) for y in the strip."""
    y0, y1 = strip_bounds(height, world, rank)
    need = set()
    for y in range(y0, y1):
        for ny in (y - step, y + step):
            if 0 <= ny < height and not (y0 <= ny < y1):
                need.add(ny)
    out = []
    for owner in range(world):
        o0, o1 = strip_bounds(height, world, owner)
        rows = sorted(r for r in need if o0 <= r < o1)
        if not rows:
            continue
        # contiguous runs
        start = prev = rows[0]
        for r in rows[1:]:
            if r != prev + 1:
                out.append((owner, start, prev + 1))
                start = r
            prev = r
        out.append((owner, start, prev + 1))
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
