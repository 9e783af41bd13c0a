"""Seeded synthetic inputs for the ASOT hot path (BASELINE.json configs c1..c5).

This module is the ONE piece shared by the fp64 oracle (``oracle/``) and the
CUDA path (``paper_2310_16123_b200``).  It holds none of the method's
arithmetic: it only draws points, weights and anchors, and builds the anchor
cost C_s that the C-ABI takes as an input ("C_s(i,j) := d_AS(w_i,
w_j)"; the configs fix d_AS = squared Euclidean normalised by its max,
SURVEY §8(c) reading #7).  Mapping, histograms, the Gibbs kernel, Sinkhorn and
the cost reduction live on each side separately.

Recipes (draw order means -> anchors -> sizes -> per
distribution (components, coordinates, weights)), numpy PCG64 seeded with the
config number unless overridden.  The paper measures on TUDataset graphs and
MNIST; those datasets are not available here and these synthetic
configs stand in for them.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass
class AsotInputs:
    """One workload: CSR point sets + anchors + anchor cost + solver settings."""

    name: str
    points: np.ndarray    # [T, d] float32, row-major
    offsets: np.ndarray   # [N+1] int64, offsets[0] = 0, offsets[N] = T
    weights: np.ndarray   # [T] float32, per-distribution simplex (fp32, not renormalised)
    anchors: np.ndarray   # [K, d] float32
    cost: np.ndarray      # [K, K] float32 C_s, symmetric, zero diagonal, max entry 1
    eps: np.float32       # entropic regulariser epsilon (the fp32 value as passed)
    iters: int            # Sinkhorn iterations L (one iteration = u-update then v-update)

    @property
    def n_dist(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def dim(self) -> int:
        return int(self.points.shape[1])

    @property
    def n_anchors(self) -> int:
        return int(self.anchors.shape[0])

    @property
    def n_points(self) -> int:
        return int(self.points.shape[0])

    @property
    def n_pairs(self) -> int:
        n = self.n_dist
        return n * (n - 1) // 2


# name: (N, (n_lo, n_hi), d, n_components, component_std, K, anchors_per_mean,
#        anchor_noise_std, means_std, weights, L, point_model)
CONFIGS = {
    "c1": dict(N=64, n_lo=5, n_hi=20, d=8, comps=4, comp_std=0.3, K=16, per_mean=4,
               anchor_std=0.5, means_std=2.0, weights="uniform", L=100, model="mixture"),
    "c2": dict(N=1000, n_lo=10, n_hi=60, d=32, comps=16, comp_std=0.2, K=128, per_mean=8,
               anchor_std=0.2, means_std=1.0, weights="uniform", L=200, model="mixture"),
    "c3": dict(N=2000, n_lo=50, n_hi=300, d=64, comps=32, comp_std=0.1, K=256, per_mean=8,
               anchor_std=0.2, means_std=1.0, weights="uniform", L=100, model="walk"),
    "c4": dict(N=8000, n_lo=20, n_hi=100, d=64, comps=64, comp_std=0.2, K=256, per_mean=4,
               anchor_std=0.2, means_std=1.0, weights="dirichlet", L=100, model="mixture"),
    "c5": dict(N=4000, n_lo=200, n_hi=1000, d=128, comps=128, comp_std=0.2, K=1024, per_mean=8,
               anchor_std=0.2, means_std=1.0, weights="uniform", L=50, model="mixture"),
}
CONFIG_SEEDS = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}
EPS = np.float32(0.05)


def normalized_sqeuclid_cost(anchors: np.ndarray) -> np.ndarray:
    """Input recipe for C_s: ||w_u - w_v||^2 / max, fp64 from the f32 anchors, stored f32.

    The max entry is exactly 1.0 after the division; the diagonal is exactly 0.
    """
    w = anchors.astype(np.float64)
    diff = w[:, None, :] - w[None, :, :]
    c = np.einsum("uvk,uvk->uv", diff, diff)
    m = c.max()
    if m > 0:
        c = c / m
    c = 0.5 * (c + c.T)
    np.fill_diagonal(c, 0.0)
    return c.astype(np.float32)


def anchor_sqdist_scale(anchors: np.ndarray) -> np.float32:
    """1 / max_{u,v} ||w_u - w_v||^2 as f32: the normalisation of normalized_sqeuclid_cost, for
    ground costs on the original points that must be on the anchors' scale (NEXT-4, R#32)."""
    w = anchors.astype(np.float64)
    diff = w[:, None, :] - w[None, :, :]
    m = np.einsum("uvk,uvk->uv", diff, diff).max()
    return np.float32(1.0 / m if m > 0 else 1.0)


def make_inputs(cfg: str, seed: Optional[int] = None, n_dist: Optional[int] = None,
                iters: Optional[int] = None) -> AsotInputs:
    """Build config ``cfg`` (c1..c5). ``n_dist`` shrinks N for oracle-sized parity runs
    (same recipe, first draws identical up to the size draw)."""
    p = CONFIGS[cfg]
    rng = np.random.default_rng(CONFIG_SEEDS[cfg] if seed is None else seed)
    N = p["N"] if n_dist is None else int(n_dist)
    d, C, K = p["d"], p["comps"], p["K"]

    means = rng.normal(0.0, p["means_std"], size=(C, d))
    per = K // C
    anchors = np.repeat(means, per, axis=0) + rng.normal(0.0, p["anchor_std"], size=(K, d))
    sizes = rng.integers(p["n_lo"], p["n_hi"] + 1, size=N)

    pts, wts = [], []
    for i in range(N):
        n = int(sizes[i])
        if p["model"] == "mixture":
            comp = rng.integers(0, C, size=n)
            x = means[comp] + rng.normal(0.0, p["comp_std"], size=(n, d))
        else:  # random walk around a shared centre (c3 "sequence-like")
            c = means[rng.integers(0, C)]
            steps = rng.normal(0.0, p["comp_std"], size=(n, d))
            steps[0] = 0.0
            x = c[None, :] + np.cumsum(steps, axis=0)
        if p["weights"] == "uniform":
            w = np.full(n, np.float32(1.0 / n), dtype=np.float32)
        else:
            w = rng.dirichlet(np.ones(n)).astype(np.float32)
        pts.append(x.astype(np.float32))
        wts.append(w)

    offsets = np.zeros(N + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(sizes)
    anchors32 = anchors.astype(np.float32)
    return AsotInputs(
        name=cfg,
        points=np.ascontiguousarray(np.concatenate(pts, axis=0)),
        offsets=offsets,
        weights=np.ascontiguousarray(np.concatenate(wts, axis=0)),
        anchors=np.ascontiguousarray(anchors32),
        cost=normalized_sqeuclid_cost(anchors32),
        eps=EPS,
        iters=int(p["L"] if iters is None else iters),
    )


def random_pairs(n_dist: int, n_pairs: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Seeded sample of unordered pairs i<j (for parity subsets at large N)."""
    rng = np.random.default_rng(seed)
    i = rng.integers(0, n_dist, size=4 * n_pairs + 16)
    j = rng.integers(0, n_dist, size=4 * n_pairs + 16)
    keep = i != j
    i, j = i[keep], j[keep]
    lo, hi = np.minimum(i, j), np.maximum(i, j)
    key = np.unique(lo.astype(np.int64) * n_dist + hi)
    rng.shuffle(key)
    key = key[:n_pairs]
    return (key // n_dist).astype(np.int32), (key % n_dist).astype(np.int32)
