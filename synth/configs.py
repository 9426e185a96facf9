"""The five BASELINE.json configs (verbatim) and small analogues.

A ConfigSpec only names sizes, seeds and solver parameters; ``build_config``
returns the CSR matrix from ``generators``.  The starting block is
``generators.gaussian_block(n, w, seed)`` (or row slices of it).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import generators as g


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    kind: str            # lap1d | lap2d | lap3dV | zipf | st27
    size: int            # n (1-D, zipf) or grid edge N
    k: int
    d: int
    p: int
    seed: int
    tol: float = 1e-10
    maxit: int = 300
    s_max: int = 5
    gpus: str = "1"
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        if self.kind in ("lap1d", "zipf"):
            return self.size
        if self.kind == "lap2d":
            return self.size ** 2
        return self.size ** 3

    @property
    def q(self) -> int:
        """Guard vectors: the paper's default q = round(0.1 k)."""
        return int(round(0.1 * self.k))

    @property
    def w(self) -> int:
        """Block width w = k + q (reading R4)."""
        return self.k + self.q


CONFIGS = {
    1: ConfigSpec("cfg1_lap1d_n2000", "lap1d", 2000, k=20, d=10, p=1, seed=0),
    2: ConfigSpec("cfg2_lap2d_300x300", "lap2d", 300, k=200, d=20, p=1, seed=1),
    3: ConfigSpec("cfg3_lap3d_100^3_plusV", "lap3dV", 100, k=500, d=20, p=2, seed=2, gpus="1/2/4/8"),
    4: ConfigSpec("cfg4_zipf_n4e6", "zipf", 4_000_000, k=1000, d=15, p=1, seed=3, gpus="1/2/4/8"),
    # cfg5: the sweeps cap s_max = 10 (R6): |T_30| amplifies the top Ritz direction only
    # ~2.4x per sweep, so the dynamic-range rule would allow ~30 sweeps and the cap binds; measured
    # on B200 (profiles/r02/cfg5_smax.log): s_max 5 -> 14 outer / 97.5 s, 10 -> 7 outer / 68.9 s
    5: ConfigSpec("cfg5_st27_256^3", "st27", 256, k=256, d=30, p=2, seed=4, gpus="1/2/4/8", s_max=10),
}

# Small analogues of every config generator (oracle-solvable in seconds).
SMALL_ANALOGS = {
    "lap1d": ConfigSpec("small_lap1d_n300", "lap1d", 300, k=8, d=10, p=1, seed=0),
    "lap2d": ConfigSpec("small_lap2d_24x24", "lap2d", 24, k=16, d=12, p=1, seed=1),
    "lap3dV": ConfigSpec("small_lap3dV_9^3", "lap3dV", 9, k=12, d=10, p=2, seed=2),
    "zipf": ConfigSpec("small_zipf_n1500", "zipf", 1500, k=16, d=15, p=1, seed=3),
    "st27": ConfigSpec("small_st27_8^3", "st27", 8, k=12, d=12, p=2, seed=4),
}


def build_matrix(kind: str, size: int, seed: int) -> g.CSR:
    if kind == "lap1d":
        return g.laplacian_1d(size)
    if kind == "lap2d":
        return g.laplacian_2d(size)
    if kind == "lap3dV":
        return g.laplacian_3d_potential(size, seed)
    if kind == "zipf":
        return g.zipf_random(size, seed)
    if kind == "st27":
        return g.stencil27_3d(size)
    raise ValueError(kind)


def starting_block(spec: ConfigSpec, n: int | None = None):
    """X0 (n x w): the config's seeded n x k Gaussian block (stream 0) followed by
    q guard columns from stream 2 (R4, R11)."""
    import numpy as np
    n = spec.n if n is None else n
    X0 = g.gaussian_block(n, spec.k, spec.seed)
    if spec.q == 0:
        return X0
    G = g.gaussian_block(n, spec.q, spec.seed, stream=2)
    return np.ascontiguousarray(np.hstack([X0, G]))


_CACHE: dict = {}


def build_config(spec_or_id) -> tuple[g.CSR, ConfigSpec]:
    """(CSR, spec).  The most recently built full-size matrix (n >= 1e6) is kept, so a
    process that needs it twice (the GPU test suite) generates it once; treat it as
    read-only."""
    spec = CONFIGS[spec_or_id] if isinstance(spec_or_id, int) else spec_or_id
    key = (spec.kind, spec.size, spec.seed)
    if key in _CACHE:
        return _CACHE[key], spec
    A = build_matrix(spec.kind, spec.size, spec.seed)
    if spec.n >= 1_000_000:
        _CACHE.clear()
        _CACHE[key] = A
    return A, spec
