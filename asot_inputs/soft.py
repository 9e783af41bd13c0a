"""Seeded parameters for the soft mappings (ASOT-ML / ASOT-DL inference).

Shared by the oracle and the CUDA path like ``synth``: it only DRAWS parameters (no mapping,
no histogram, no Sinkhorn arithmetic).  Trained weights do not exist here (the paper trains on
TUDataset / MNIST, which are absent), so the parameters are seeded random draws with the
paper's shapes (Table 4; widths scaled from the 5d GIN features to raw d-dim points,
DESIGN.md R#24):

  ML: mapper MLP d -> 2d -> K (He-normal weights), Mahalanobis M in R^{d x d} (h = d).
  DL: dictionary = the config's anchors scaled by 1/||A||_2 together with the points (the
      appendix's step size 1, needs ||W||_2 <= 1; R#28), lambda-MLP d -> d/2 -> 1 whose
      output bias sets a typical lambda of ``lam0`` (a recipe constant, not fitted to data).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from .synth import AsotInputs, make_inputs, normalized_sqeuclid_cost

DL_LAYERS = 20          # Table 4 P:570 "Num. of near-one-hot layers 20"


@dataclasses.dataclass
class MlModel:
    W1: np.ndarray   # [d, 2d] f32
    b1: np.ndarray   # [2d]
    W2: np.ndarray   # [2d, K]
    b2: np.ndarray   # [K]
    M: np.ndarray    # [h = d, d] Mahalanobis transform

    @property
    def layers(self):
        return [(self.W1, self.b1), (self.W2, self.b2)]


@dataclasses.dataclass
class DlModel:
    dictionary: np.ndarray  # [K, d] f32, row u = anchor w_u (the paper's W = dictionary^T)
    V1: np.ndarray          # [d, h] f32, h = max(1, d // 2)
    c1: np.ndarray          # [h]
    v2: np.ndarray          # [h, 1]
    c2: np.ndarray          # [1]
    n_layers: int = DL_LAYERS

    @property
    def lam_layers(self):
        return [(self.V1, self.c1), (self.v2, self.c2)]


def make_ml_model(d: int, K: int, seed: int = 101) -> MlModel:
    rng = np.random.default_rng(seed)
    h = 2 * d
    f = lambda a: np.ascontiguousarray(a.astype(np.float32))
    return MlModel(
        W1=f(rng.normal(0.0, np.sqrt(2.0 / d), size=(d, h))),
        b1=f(rng.normal(0.0, 0.1, size=h)),
        W2=f(rng.normal(0.0, np.sqrt(1.0 / h), size=(h, K))),
        b2=f(rng.normal(0.0, 0.1, size=K)),
        M=f(rng.normal(0.0, np.sqrt(1.0 / d), size=(d, d))),
    )


def make_dl_inputs(cfg: str = "c2", n_dist: Optional[int] = None, iters: Optional[int] = None,
                   seed: int = 202, lam0: float = 0.01) -> tuple[AsotInputs, DlModel]:
    """The config's points and anchors scaled by 1 / ||anchors||_2 (R#28) + a seeded DL model."""
    base = make_inputs(cfg, n_dist=n_dist, iters=iters)
    s = float(np.linalg.norm(base.anchors.astype(np.float64), 2))
    dictionary = np.ascontiguousarray((base.anchors.astype(np.float64) / s).astype(np.float32))
    points = np.ascontiguousarray((base.points.astype(np.float64) / s).astype(np.float32))
    d = base.dim
    h = max(1, d // 2)
    rng = np.random.default_rng(seed)
    f = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))
    model = DlModel(
        dictionary=dictionary,
        V1=f(rng.normal(0.0, np.sqrt(2.0 / d), size=(d, h))),
        c1=f(rng.normal(0.0, 0.1, size=h)),
        v2=f(rng.normal(0.0, 0.1 * np.sqrt(1.0 / h), size=(h, 1))),
        c2=f([np.log(np.expm1(lam0))]),   # softplus^-1(lam0): the typical lambda
    )
    inp = AsotInputs(base.name + "-dl", points, base.offsets, base.weights, dictionary,
                     normalized_sqeuclid_cost(dictionary), base.eps, base.iters)
    return inp, model


def make_kmeans_draws(points: np.ndarray, K: int, iters: int, batch: int,
                      seed: int = 303) -> tuple[np.ndarray, np.ndarray]:
    """NEXT-2 random draws of mini-batch k-means (passed to both sides, R#30): Forgy
    initialisation (K distinct point indices -> their coordinates) and iters x batch point
    indices drawn with replacement."""
    rng = np.random.default_rng(seed)
    T = points.shape[0]
    init_idx = rng.choice(T, size=K, replace=False)
    batch_idx = rng.integers(0, T, size=(iters, batch), dtype=np.int64)
    return np.ascontiguousarray(points[init_idx]), np.ascontiguousarray(batch_idx)
