"""Test infrastructure: the fp64 oracle's one-hot mapping (oracle.asot_oracle.map_assign, R#8)
fanned out over the host cores, so full-size assignment parity (every c3 point, a
10% sample of c5's distributions) finishes in tens of seconds.  Pure partitioning over points:
each chunk runs the oracle function unchanged, so the result is the oracle's, bit for bit."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from oracle import asot_oracle as O


def _chunk(args):
    pts, anchors = args
    return O.map_assign(pts, anchors)


def map_assign_parallel(points: np.ndarray, anchors: np.ndarray, chunk: int = 8192,
                        workers: int | None = None) -> np.ndarray:
    T = points.shape[0]
    if T == 0:
        return np.zeros(0, np.int32)
    workers = workers or max(1, min(len(os.sched_getaffinity(0)), 32))
    parts = [(points[s:s + chunk], anchors) for s in range(0, T, chunk)]
    if workers == 1 or len(parts) == 1:
        return np.concatenate([_chunk(p) for p in parts])
    # spawn, not fork: the parent holds a CUDA context
    with mp.get_context("spawn").Pool(workers) as pool:
        return np.concatenate(pool.map(_chunk, parts))


def rows_of(offsets: np.ndarray, dists: np.ndarray) -> np.ndarray:
    """Point indices of the given distributions, in distribution order."""
    return np.concatenate([np.arange(offsets[d], offsets[d + 1]) for d in dists]).astype(np.int64)
