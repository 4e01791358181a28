"""BASELINE.json configs C1..C5 as seeded synthetic workloads.

Seeds: graph seed 1; opinion column j uses seed 2 + j (SURVEY §8(d) "Stand-in statement").
Each config returns the RAW edge list (self-loops / duplicates kept; the CSR build
of row a1 removes them) plus the opinion matrix S [n][k] in row-major order.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    desc: str
    n: int
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray | None          # None = unit weights; else uint8 weights
    S: np.ndarray                 # [n][k] float64, row-major
    kinds: list = field(default_factory=list)  # opinion distribution per column

    @property
    def k(self) -> int:
        return self.S.shape[1]


CONFIGS = {
    "c1": "BA n=2000 m=3 unit, s~U[0,1], k=1 (BASELINE configs[0])",
    "c2": "ER n=1e6 p=10/(n-1) unit, s~U[0,1], k=1 (BASELINE configs[1])",
    "c3": "BA n=4e6 m=8 unit, s in {uniform, exponential, powerlaw} (BASELINE configs[2])",
    "c4": "R-MAT scale 22 ef 16 (.57,.19,.19,.05), w in 1..5 (u8), k=64 U[0,1] (BASELINE configs[3])",
    "c5": "R-MAT scale 26 ef 16 (.57,.19,.19,.05) unit, s~U[0,1] (BASELINE configs[4])",
}


def _S(n: int, kinds: list[str]) -> np.ndarray:
    from . import opinions
    S = np.empty((n, len(kinds)), dtype=np.float64)
    for j, kind in enumerate(kinds):
        S[:, j] = opinions(kind, n, 2 + j)
    return S


def make_config(name: str, *, k: int | None = None, kinds: list[str] | None = None,
                scale: int | None = None, n: int | None = None) -> Workload:
    """Build a config's raw inputs.  Optional overrides shrink a config for tests
    (same recipe, smaller size): `n` for BA/ER, `scale` for R-MAT, `k`/`kinds` for opinions."""
    from . import barabasi_albert, erdos_renyi, rmat, weights_u8
    name = name.lower()
    if name == "c1":
        nn = n or 2000
        u, v = barabasi_albert(nn, 3, 1)
        kinds = kinds or ["uniform"] * (k or 1)
        return Workload(name, CONFIGS[name], nn, u, v, None, _S(nn, kinds), kinds)
    if name == "c2":
        nn = n or 1_000_000
        u, v = erdos_renyi(nn, 10.0 / (nn - 1), 1)
        kinds = kinds or ["uniform"] * (k or 1)
        return Workload(name, CONFIGS[name], nn, u, v, None, _S(nn, kinds), kinds)
    if name == "c3":
        nn = n or 4_000_000
        u, v = barabasi_albert(nn, 8, 1)
        kinds = kinds or ["uniform", "exponential", "powerlaw"]
        return Workload(name, CONFIGS[name], nn, u, v, None, _S(nn, kinds), kinds)
    if name == "c4":
        sc = scale or 22
        u, v = rmat(sc, 16, 0.57, 0.19, 0.19, 1)
        w = weights_u8(u, v, 1)
        kinds = kinds or ["uniform"] * (k or 64)
        nn = 1 << sc
        return Workload(name, CONFIGS[name], nn, u, v, w, _S(nn, kinds), kinds)
    if name == "c5":
        sc = scale or 26
        u, v = rmat(sc, 16, 0.57, 0.19, 0.19, 1)
        kinds = kinds or ["uniform"] * (k or 1)
        nn = 1 << sc
        return Workload(name, CONFIGS[name], nn, u, v, None, _S(nn, kinds), kinds)
    raise KeyError(name)
