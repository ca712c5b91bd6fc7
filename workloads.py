"""The five BASELINE.json workloads as seeded synthetic inputs.

Bench / test infrastructure, independent of the product package: every array is
generated from the reference's xorshift64* Rng stream (util.hpp:83-98). The
stream is injected (`rng(seed, n) -> float64[n]`): the product arm passes the
library's own pwb_rng_uniform (paper_2111_01083_b200.configs), the reference arm
of bench.py the reference's own periwave::Rng compiled into oracle/_ref
(oracle.pyoracle.rng_uniform), so the reference arm never loads the product
library. Both streams are the same bytes (tests/test_abi.py, tests/test_configs.py).
No public dataset is involved.

Conventions (fixed; documented in DESIGN.md):
  * positions: x1, x2 ~ U[-1/2, 1/2) from stream `seed` (interleaved), p = x1 e1 + x2 e2
    (as periwave_cli.cpp:108-132);
  * normals N(0,1): Box-Muller z = sqrt(-2 ln(1-u1)) cos(2 pi u2) on stream seed + 7919;
  * neutral strengths: mean subtracted per component, then |sum| <= 1e-12 sum|.| checked;
  * c4 clusters: 16 centres uniform in the cell (stream seed + 104729), centre index
    floor(16 u), offset 0.02 (n1, n2); x wrapped into [-1/2, 1/2) (periodic direction),
    y rejection-resampled until |y| <= 1/2 (SURVEY.md §8(d) recommendation);
  * separate targets (c2): stream seed + 1299709;
  * oracle target subsample: the first S indices of a stable argsort of the
    uniforms on stream seed + 15485863.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

# ordinals of periwave::Pde / Periodicity (proj/include/periwave/cell.hpp); the product's
# IntEnums compare and hash equal to these ints
POISSON, MODHELMHOLTZ, STOKES = 0, 1, 2
SINGLY, DOUBLY = 1, 2


@dataclass(frozen=True)
class Config:
    name: str
    pde: int
    beta: float
    cell: tuple  # (d, xi, eta, periodicity)
    n_src: int
    separate_targets: bool
    strength: str  # "charge" | "force"
    neutral: bool
    eps: float
    outputs: tuple
    oracle_sample: int
    seed: int
    clustered: bool = False
    gradient: bool = False


CONFIGS = {
    "c1": Config("c1", POISSON, 0.0, (1.0, 0.0, 1.0, DOUBLY), 1000, False, "charge", True, 1e-10,
                 ("u",), 1000, 1001),
    "c2": Config("c2", MODHELMHOLTZ, 10.0, (1.0, 0.3, 0.8, DOUBLY), 100000, True, "charge", False,
                 1e-10, ("u", "dudx", "dudy"), 4096, 1002, gradient=True),
    "c3": Config("c3", STOKES, 0.0, (1.0, 0.0, 1.0, DOUBLY), 1000000, False, "force", True, 1e-8,
                 ("u1", "u2"), 2048, 1003),
    "c4": Config("c4", POISSON, 0.0, (1.0, 0.0, 1.0, SINGLY), 1000000, False, "charge", True, 1e-10,
                 ("u",), 2048, 1004, clustered=True),
    "c5": Config("c5", MODHELMHOLTZ, 1.0, (100.0, 0.0, 1.0, DOUBLY), 10000000, False, "charge", False,
                 1e-8, ("u",), 256, 1005),
}


def normals(rng, seed: int, n: int) -> np.ndarray:
    u = rng(seed, 2 * n)
    u1 = 1.0 - u[0::2]  # (0, 1]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u[1::2])


def uniform_points(rng, seed: int, n: int, d: float, xi: float, eta: float) -> np.ndarray:
    u = rng(seed, 2 * n)
    x1 = u[0::2] - 0.5
    x2 = u[1::2] - 0.5
    return np.ascontiguousarray(np.stack([x1 * d + x2 * xi, x2 * eta], axis=1))


def clustered_points(rng, seed: int, n: int, k: int = 16, sigma: float = 0.02) -> np.ndarray:
    centres = uniform_points(rng, seed + 104729, k, 1.0, 0.0, 1.0)
    which = np.minimum((rng(seed, n) * k).astype(np.int64), k - 1)
    gx = normals(rng, seed + 7, n)
    pool = normals(rng, seed + 11, 2 * n + 4096)
    x = centres[which, 0] + sigma * gx
    x = x - np.floor(x + 0.5)  # wrap into [-1/2, 1/2)
    y = centres[which, 1] + sigma * pool[:n]
    nxt = n
    bad = np.nonzero(np.abs(y) > 0.5)[0]
    while bad.size:
        if nxt + bad.size > pool.size:
            pool = np.concatenate([pool, normals(rng, seed + 13 + nxt, 2 * bad.size + 4096)])
        y[bad] = centres[which[bad], 1] + sigma * pool[nxt:nxt + bad.size]
        nxt += bad.size
        bad = bad[np.abs(y[bad]) > 0.5]
    return np.ascontiguousarray(np.stack([x, y], axis=1))


def neutralize(a: np.ndarray) -> np.ndarray:
    a = a - a.mean(axis=0)
    s = np.abs(a.sum(axis=0))
    tot = np.abs(a).sum(axis=0) if a.ndim == 1 else np.hypot(a[:, 0], a[:, 1]).sum()
    assert np.all(s <= 1e-12 * tot), "neutrality check failed"
    return np.ascontiguousarray(a)


@dataclass
class Inputs:
    config: Config
    sources: np.ndarray
    charges: Optional[np.ndarray]
    forces: Optional[np.ndarray]
    targets: np.ndarray  # full target set (== sources when not separate)
    sample: np.ndarray   # oracle subsample: indices into targets


def generate(name: str, n_src: Optional[int] = None, rng=None) -> Inputs:
    """Inputs for config `name` from the uniform stream `rng(seed, n)`; n_src overrides the
    size (tests use small N)."""
    if rng is None:
        raise TypeError("workloads.generate needs the uniform stream rng(seed, n)")
    c = CONFIGS[name]
    n = c.n_src if n_src is None else n_src
    d, xi, eta, per = c.cell
    src = clustered_points(rng, c.seed, n) if c.clustered else uniform_points(rng, c.seed, n, d, xi, eta)
    charges = forces = None
    if c.strength == "charge":
        q = normals(rng, c.seed + 7919, n)
        charges = neutralize(q) if c.neutral else np.ascontiguousarray(q)
    else:
        g = normals(rng, c.seed + 7919, 2 * n).reshape(n, 2)
        forces = neutralize(g) if c.neutral else np.ascontiguousarray(g)
    tgt = uniform_points(rng, c.seed + 1299709, n, d, xi, eta) if c.separate_targets else src
    m = min(c.oracle_sample, n)
    order = np.argsort(rng(c.seed + 15485863, n), kind="stable")
    sample = np.sort(order[:m])
    return Inputs(c, src, charges, forces, tgt, sample)
