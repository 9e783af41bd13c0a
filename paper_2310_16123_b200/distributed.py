"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) process groups.

The pair set (Def. 1) is embarrassingly parallel: rank r owns a contiguous range of
the upper-triangular pair tiles (step a4; every tile costs the same 2L+1 dense MMA phases, so
equal tile counts are equal work).  There are exactly two exchanges:
  1. mapping is partitioned by distribution ranges balanced by point count, then the N x K
     mapped-marginal matrix H is all-gathered (all_gather_into_tensor, NVLink);
  2. each rank's slot-ordered tile results are gathered to rank 0, which scatters them into the
     N x N matrix (KN6 unpack) and zeroes the diagonal.
Every pair's arithmetic is independent of the partition, so D is bitwise identical for any
world size.

The orchestration takes its compute steps as callables so the exact same partition / gather /
assembly logic runs (a) on GPUs with the libasot kernels and (b) under gloo on CPU in the tests.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


def partition_even(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [begin, end) ranges of n units over `world` ranks, sizes differing by <= 1."""
    base, extra = divmod(n, world)
    out, a = [], 0
    for r in range(world):
        b = a + base + (1 if r < extra else 0)
        out.append((a, b))
        a = b
    return out


def partition_by_points(offsets: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous distribution ranges balanced by point count (prefix sums of offsets)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    N = offsets.shape[0] - 1
    T = int(offsets[-1])
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(offsets, T * r / world, side="left"))
        cuts.append(min(max(c, cuts[-1]), N))
    cuts.append(N)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


@dataclass
class DistSteps:
    """Compute steps used by distance_matrix_distributed (device or test stand-ins)."""
    map_range: Callable[[int, int], torch.Tensor]            # (lo, hi) -> H rows [hi-lo, K]
    tiles: Callable[[torch.Tensor, int, int], torch.Tensor]  # (H, t0, t1) -> packed [(t1-t0)*128]
    unpack: Callable[[torch.Tensor, int, int, torch.Tensor], None]  # (packed, t0, t1, D) in place
    zero_diag: Callable[[torch.Tensor], None]


def distance_matrix_distributed(n_dist: int, n_anchors: int, offsets_host: np.ndarray,
                                n_tiles: int, steps: DistSteps, group=None,
                                device: Optional[torch.device] = None,
                                hist: Optional[torch.Tensor] = None):
    """All ranks call this; rank 0 returns the N x N matrix, other ranks return None."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cpu")

    # exchange 1: partitioned mapping + all-gather of H (rows padded to equal counts)
    if hist is None:
        ranges = partition_by_points(offsets_host, world)
        rows = max(b - a for a, b in ranges)
        lo, hi = ranges[rank]
        H_local = torch.zeros((rows, n_anchors), dtype=torch.float32, device=dev)
        if hi > lo:
            H_local[: hi - lo] = steps.map_range(lo, hi)
        H_all = torch.empty((world * rows, n_anchors), dtype=torch.float32, device=dev)
        dist.all_gather_into_tensor(H_all, H_local, group=group)
        H = torch.cat([H_all[r * rows: r * rows + (b - a)] for r, (a, b) in enumerate(ranges)])
    else:
        H = hist

    # the rank's contiguous share of the upper-triangular tiles
    tranges = partition_even(n_tiles, world)
    t0, t1 = tranges[rank]
    tmax = max(b - a for a, b in tranges)
    packed = torch.zeros(tmax * 128, dtype=torch.float32, device=dev)
    if t1 > t0:
        packed[: (t1 - t0) * 128] = steps.tiles(H, t0, t1)

    # exchange 2: gather slot-ordered results to rank 0 (padded all-gather; NCCL has no
    # variable-size gather) and scatter them into the matrix there
    gathered = torch.empty(world * tmax * 128, dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(gathered, packed, group=group)
    if rank != 0:
        return None
    D = torch.zeros((n_dist, n_dist), dtype=torch.float32, device=dev)
    for r, (a, b) in enumerate(tranges):
        if b > a:
            steps.unpack(gathered[r * tmax * 128: r * tmax * 128 + (b - a) * 128], a, b, D)
    steps.zero_diag(D)
    return D


def cuda_steps(points: torch.Tensor, offsets: torch.Tensor, offsets_host: np.ndarray,
               weights: torch.Tensor, anchors: torch.Tensor, cost: torch.Tensor, eps: float,
               iters: int, precision: int, cost_max: float, status: torch.Tensor,
               workspace=None) -> DistSteps:
    """DistSteps backed by the libasot kernels (all compute on this rank's GPU)."""
    from . import asot as A

    offs_h = np.asarray(offsets_host, dtype=np.int64)

    def map_range(lo: int, hi: int) -> torch.Tensor:
        s, e = int(offs_h[lo]), int(offs_h[hi])
        sub_off_h = offs_h[lo: hi + 1] - s
        sub_off = torch.from_numpy(sub_off_h).to(points.device, non_blocking=True)
        _, H, _ = A.map_to_anchors(points[s:e].contiguous(), sub_off, weights[s:e].contiguous(),
                                   anchors, offsets_host=sub_off_h, status=status)
        return H

    def tiles(H: torch.Tensor, t0: int, t1: int) -> torch.Tensor:
        packed = torch.empty((t1 - t0) * 128, dtype=torch.float32, device=H.device)
        A.distance_matrix(None, None, None, None, cost, eps, iters, precision=precision, hist=H,
                          tile_range=(t0, t1), packed=packed, want_matrix=False, cost_max=cost_max,
                          status=status, workspace=workspace)
        return packed

    def unpack(packed: torch.Tensor, t0: int, t1: int, D: torch.Tensor) -> None:
        A.unpack_tiles(packed, D.shape[0], t0, t1, D, zero_diag=False)

    def zero_diag(D: torch.Tensor) -> None:  # KN6 with an empty tile range: diagonal only
        A.unpack_tiles(D, D.shape[0], 0, 0, D, zero_diag=True)

    return DistSteps(map_range, tiles, unpack, zero_diag)
