"""BASELINE.json workloads as seeded synthetic models and inputs.

SURVEY §8(d): no dataset is used by the reference; seeded numpy PCG64 draws
stand in for MNIST/CIFAR-shaped inputs. Seed 0 draws the weights (per layer:
W_b then S, knots deterministic), seed 1 draws the inputs. Each layer's SiLU
polynomial is fitted on that layer's calibration inputs (the exact plaintext
forward of the previous layers) with the reference's recipe:
estimate_range(x, x_min=min, x_max=max, factor=5) -> WeightScheme.from_moments
-> fit_weighted_ls (approx.py:129-179, PAPER §4.1).

configs:
  c1  [2,5,1]        G=5 k=3 [-1,1]  W~N(0,0.1)   128 x U[-1,1]^2        SiLU deg 10
  c3  [4,8,4,1]      G=10 k=3 [-2,2] W~N(0,0.1)   4096 x clip(N(0,1),+-2) SiLU deg 63
  c4  [784,64,10]    G=5 k=3 [-1,1]  W~N(0,0.05)  64 x U[0,1]^784         SiLU deg 10
  c5  [3072,128,10]  G=5 k=3 [-1,1]  W~N(0,0.02)  32 x std(U[0,1]^3072)   SiLU deg 10
c4/c5 use an explicit per-layer R = 1.2 max(max|calibration input|, max|knot|)
(the default R lets layer-2 comparator inputs leave [-1, 1]).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .approx import WeightScheme, estimate_range, fit_weighted_ls
from .bspline import GridMatrix
from .model import KanLayer, KanModel, layer_forward_plain, silu


@dataclass(frozen=True)
class KanConfig:
    name: str
    dims: tuple
    g: int
    k: int
    lo: float
    hi: float
    w_std: float
    batch: int
    silu_degree: int
    input_shape: tuple
    explicit_R: bool = False


CONFIGS = {
    "c1": KanConfig("c1", (2, 5, 1), 5, 3, -1.0, 1.0, 0.1, 128, 10, (1, 1, 2)),
    "c3": KanConfig("c3", (4, 8, 4, 1), 10, 3, -2.0, 2.0, 0.1, 4096, 63, (1, 1, 4)),
    "c4": KanConfig("c4", (784, 64, 10), 5, 3, -1.0, 1.0, 0.05, 64, 10, (28, 28, 1), explicit_R=True),
    "c5": KanConfig("c5", (3072, 128, 10), 5, 3, -1.0, 1.0, 0.02, 32, 10, (32, 32, 3), explicit_R=True),
}


def make_inputs(cfg: KanConfig, seed: int = 1, rows: int | None = None) -> np.ndarray:
    """(rows, n_in) synthetic inputs with the config's distribution (default
    rows = the config's batch). Draws are sequential, so the first cfg.batch
    rows are the same for any rows >= cfg.batch (a multi-GPU global batch
    extends the single-GPU one); c5 standardises with the first cfg.batch
    rows' per-channel statistics."""
    rng = np.random.default_rng(seed)
    n = cfg.dims[0]
    rows = cfg.batch if rows is None else max(int(rows), 1)
    draw = max(rows, cfg.batch)
    if cfg.name == "c1":
        x = rng.uniform(-1.0, 1.0, (draw, n))
    elif cfg.name == "c3":
        x = np.clip(rng.normal(0.0, 1.0, (draw, n)), -2.0, 2.0)
    elif cfg.name == "c4":
        x = rng.uniform(0.0, 1.0, (draw, n))
    elif cfg.name == "c5":
        img = rng.uniform(0.0, 1.0, (draw, 32, 32, 3))
        mu = img[:cfg.batch].mean(axis=(0, 1, 2), keepdims=True)
        sd = img[:cfg.batch].std(axis=(0, 1, 2), keepdims=True)
        x = ((img - mu) / sd).reshape(draw, n)  # HWC raster (inference.py:110-112)
    else:
        raise KeyError(cfg.name)
    return x[:rows]


def build_model(cfg: KanConfig, calib: np.ndarray, seed: int = 0) -> KanModel:
    rng = np.random.default_rng(seed)
    layers = []
    x = np.asarray(calib, dtype=float)
    for n_i, n_o in zip(cfg.dims, cfg.dims[1:]):
        grid = GridMatrix.uniform(n_i, cfg.g, cfg.k, cfg.lo, cfg.hi)
        if cfg.explicit_R:
            R = 1.2 * max(float(np.max(np.abs(x))), float(np.max(np.abs(grid.entries))))
            grid = GridMatrix.uniform(n_i, cfg.g, cfg.k, cfg.lo, cfg.hi, R=R)
        W_b = rng.normal(0.0, cfg.w_std, (n_o, n_i))
        S = rng.normal(0.0, cfg.w_std, (n_o, n_i, grid.n_basis))
        act = estimate_range(x, x_min=float(np.min(x)), x_max=float(np.max(x)), factor=5.0)
        poly = fit_weighted_ls(silu, act, cfg.silu_degree, w=WeightScheme.from_moments(act.mu, act.sigma))
        layer = KanLayer(W_b=W_b, S=S, grid=grid, silu_poly=poly, act_stats=(act.mu, act.sigma),
                         fit_range=(act.lo, act.hi))
        layers.append(layer)
        x = np.stack([layer_forward_plain(layer, row, mode="exact") for row in x])
    return KanModel(layers=layers, input_shape=cfg.input_shape)


def workload(name: str, batch: int | None = None):
    """(KanConfig, model, inputs[batch, n_in]) for a named config."""
    cfg = CONFIGS[name]
    model = build_model(cfg, make_inputs(cfg))
    return cfg, model, make_inputs(cfg, rows=batch)
