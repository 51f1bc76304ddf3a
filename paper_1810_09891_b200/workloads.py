"""Seeded synthetic workloads for the five BASELINE.json configurations.

No public dataset is involved: the reference paper's inputs are synthetic
 and the generators below follow the reference CLI
(``cli.gen_nodes``, /root/reference/pkg/src/nfftk/cli.py:46-51) and
SURVEY.md section 8(d):

* uniform nodes   ``default_rng(seed).random((M, d)) - 0.5``
* clustered nodes (C4) 16 isotropic Gaussians, sigma = 0.02, centres uniform,
  wrapped onto the torus with ``mod(x + 1/2, 1) - 1/2`` and clamped below 1/2
  (``np.mod(-1e-18, 1.0) - 0.5 == 0.5`` would be rejected by the range check)
* coefficients / samples iid complex standard normal.
"""

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    N: tuple
    n: tuple
    M: int
    m: int
    dist: str = "uniform"

    @property
    def d(self):
        return len(self.N)

    @property
    def num_freqs(self):
        return int(np.prod(self.N))

    @property
    def grid_size(self):
        return int(np.prod(self.n))


CONFIGS = {
    "C1": Workload("C1", (1024,), (2048,), 4096, 8),
    "C2": Workload("C2", (256, 256), (512, 512), 65536, 8),
    "C3": Workload("C3", (64, 64, 64), (128, 128, 128), 262144, 6),
    "C4": Workload("C4", (2048, 2048), (4096, 4096), 1 << 24, 6, "clustered"),
    "C5": Workload("C5", (256, 256, 256), (512, 512, 512), 1 << 26, 4),
}

# Development sizes (tools/ only): C5's density and cutoff on a grid 8x smaller,
# for quick kernel A/B runs and ncu captures.
DEV_CONFIGS = {
    "C5q": Workload("C5q", (128, 128, 128), (256, 256, 256), 1 << 23, 4),
}


def lookup(name):
    return CONFIGS.get(name) or DEV_CONFIGS[name]


NODE_SEED = 0
FHAT_SEED = 1
F_SEED = 2


def uniform_nodes(M, d, seed=NODE_SEED):
    return np.random.default_rng(seed).random((int(M), int(d))) - 0.5


def clustered_nodes(M, d=2, seed=NODE_SEED, clusters=16, sigma=0.02):
    rng = np.random.default_rng(seed)
    centres = rng.random((clusters, d)) - 0.5
    labels = rng.integers(0, clusters, int(M))
    x = centres[labels] + sigma * rng.standard_normal((int(M), d))
    x = np.mod(x + 0.5, 1.0) - 0.5
    x[x >= 0.5] = -0.5
    return x


def nodes(w, seed=NODE_SEED):
    if w.dist == "clustered":
        return clustered_nodes(w.M, w.d, seed)
    return uniform_nodes(w.M, w.d, seed)


def complex_normal(K, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(int(K)) + 1j * rng.standard_normal(int(K))


def fhat(w, seed=FHAT_SEED):
    return complex_normal(w.num_freqs, seed)


def samples(w, seed=F_SEED):
    return complex_normal(w.M, seed)


def scaled(w, M):
    """Same grid/cutoff with a different node count (bounded CPU samples)."""
    return Workload(w.name, w.N, w.n, int(M), w.m, w.dist)
