"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) process groups.

Exchanges, two forms:
  * "p2p" (default on GPUs): H and rank 0's N x N matrix are torch symmetric-memory buffers.  Each
    rank's histogram kernel stores its rows into every rank's H (the all-gather fused into the
    kernel that produces the rows), and every rank passes rank 0's matrix address as the Sinkhorn
    kernel's output, so each pair's distance leaves the epilogue as an NVLink store into rank 0's
    matrix -- no packed buffers, no collective on the data path, no unpack; stream syncs and
    barriers publish H and the matrix.
  * "nccl": packed slot-ordered tiles, NCCL all-gather, KN6 unpack on rank 0 (also the CPU/gloo
    test form, and the fallback when symmetric memory is unavailable).

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


class P2PResult:
    """Symmetric-memory buffers mapped into every rank: rank 0's N x N result matrix (written by
    every rank's Sinkhorn epilogue) and, when n_anchors is given, each rank's full N x K H
    (written by every rank's histogram kernel: the all-gather of H fused into the mapping)."""

    def __init__(self, n_dist: int, device: torch.device, group=None, n_anchors: Optional[int] = None):
        import torch.distributed._symmetric_memory as symm_mem

        grp = group if group is not None else dist.group.WORLD
        self.D = symm_mem.empty(n_dist, n_dist, dtype=torch.float32, device=device)
        self.handle = symm_mem.rendezvous(self.D, grp)
        self.root_ptr = int(self.handle.buffer_ptrs[0])
        self.H = None
        self.h_peers = None
        if n_anchors is not None:
            self.H = symm_mem.empty(n_dist, n_anchors, dtype=torch.float32, device=device)
            self.h_handle = symm_mem.rendezvous(self.H, grp)
            self.h_peers = torch.tensor([int(x) for x in self.h_handle.buffer_ptrs], dtype=torch.int64,
                                        device=device)


def distance_matrix_distributed_p2p(n_dist: int, n_anchors: int, offsets_host: np.ndarray,
                                    n_tiles: int, steps: "DistSteps", result: P2PResult, group=None,
                                    device: Optional[torch.device] = None,
                                    hist: Optional[torch.Tensor] = None):
    """As distance_matrix_distributed, but every rank's Sinkhorn epilogue stores its pairs straight
    into rank 0's symmetric-memory matrix (NVLink stores); returns that matrix on rank 0."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    if hist is not None:
        H = hist
    elif result.h_peers is not None and steps.map_range_bcast is not None:
        # exchange 1 fused: this rank's histogram rows are stored into every rank's H directly
        lo, hi = partition_by_points(offsets_host, world)[rank]
        if hi > lo:
            steps.map_range_bcast(lo, hi, result.h_peers)
        _sync(dev)
        dist.barrier(group=group)
        H = result.H
    else:
        H = _gather_hist(n_anchors, offsets_host, steps, world, rank, dev, group)
    t0, t1 = partition_even(n_tiles, world)[rank]
    if t1 > t0:
        steps.tiles_into(H, t0, t1, result.root_ptr)
    _sync(dev)                                   # this rank's stores have landed
    dist.barrier(group=group)                    # ... and every other rank's
    if rank != 0:
        return None
    steps.zero_diag(result.D)
    return result.D


def _sync(dev):
    """Wait for this rank's device work (its peer stores) before a barrier; no-op off-GPU (the
    gloo tests' stand-in steps are synchronous)."""
    if dev.type == "cuda":
        torch.cuda.current_stream(dev).synchronize()


def _gather_hist(n_anchors, offsets_host, steps, world, rank, dev, group):
    """Exchange 1: partitioned mapping + NCCL all-gather of H (rows padded to equal counts)."""
    ranges = partition_by_points(offsets_host, world)
    rows = max(b - a for a, b in ranges)
    lo, hi = ranges[rank]
    H_local = torch.zeros((rows, n_anchors), dtype=torch.float32, device=dev)
    if hi > lo:
        H_local[: hi - lo] = steps.map_range(lo, hi)
    H_all = torch.empty((world * rows, n_anchors), dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(H_all, H_local, group=group)
    return torch.cat([H_all[r * rows: r * rows + (b - a)] for r, (a, b) in enumerate(ranges)])


@dataclass
class DistSteps:
    """Compute steps used by distance_matrix_distributed (device or test stand-ins)."""
    map_range: Callable[[int, int], torch.Tensor]            # (lo, hi) -> H rows [hi-lo, K]
    tiles: Callable[[torch.Tensor, int, int], torch.Tensor]  # (H, t0, t1) -> packed [(t1-t0)*128]
    unpack: Callable[[torch.Tensor, int, int, torch.Tensor], None]  # (packed, t0, t1, D) in place
    zero_diag: Callable[[torch.Tensor], None]
    tiles_into: Optional[Callable[[torch.Tensor, int, int, int], None]] = None  # (H, t0, t1, D address)
    map_range_bcast: Optional[Callable[[int, int, torch.Tensor], None]] = None  # (lo, hi, H peer addresses)


def distance_matrix_distributed(n_dist: int, n_anchors: int, offsets_host: np.ndarray,
                                n_tiles: int, steps: DistSteps, group=None,
                                device: Optional[torch.device] = None,
                                hist: Optional[torch.Tensor] = None):
    """All ranks call this; rank 0 returns the N x N matrix, other ranks return None."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cpu")

    # exchange 1: partitioned mapping + all-gather of H (rows padded to equal counts)
    H = _gather_hist(n_anchors, offsets_host, steps, world, rank, dev, group) if hist is None else hist

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
    # the mapping's own scratch (tensor-core score pass): the Sinkhorn workspace stays untouched
    map_ws = A.Workspace(points.device)

    def map_range(lo: int, hi: int) -> torch.Tensor:
        s, e = int(offs_h[lo]), int(offs_h[hi])
        sub_off_h = offs_h[lo: hi + 1] - s
        sub_off = torch.from_numpy(sub_off_h).to(points.device, non_blocking=True)
        _, H, _ = A.map_to_anchors(points[s:e].contiguous(), sub_off, weights[s:e].contiguous(),
                                   anchors, offsets_host=sub_off_h, status=status, tensor_core=True,
                                   workspace=map_ws)
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

    def map_range_bcast(lo: int, hi: int, peers: torch.Tensor) -> None:
        s, e = int(offs_h[lo]), int(offs_h[hi])
        sub_off_h = offs_h[lo: hi + 1] - s
        sub_off = torch.from_numpy(sub_off_h).to(points.device, non_blocking=True)
        A.map_to_anchors_bcast(points[s:e].contiguous(), sub_off, weights[s:e].contiguous(), anchors,
                               peers, lo, offsets_host=sub_off_h, status=status, tensor_core=True,
                               workspace=map_ws)

    def tiles_into(H: torch.Tensor, t0: int, t1: int, d_addr: int) -> None:
        # part [t0, t1) of the enumeration the library picks (support order on the small-support
        # path): the ranks' parts still cover every pair once, and each rank's warps stay as
        # homogeneous as the single-GPU whole triangle
        A.distance_matrix_partition(H, cost, eps, iters, (t0, t1), precision=precision,
                                    out_ptr=d_addr, cost_max=cost_max, status=status,
                                    workspace=workspace)

    return DistSteps(map_range, tiles, unpack, zero_diag, tiles_into, map_range_bcast)
