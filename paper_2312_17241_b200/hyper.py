"""Shape knobs and grid geometry, mirroring the reference's public types.

``HyperParams`` has the reference's fields, defaults and validation
(model.py:35-87); the level ladder follows indexing.py:66-101 exactly so the
same dense/hashed split and resolutions come out.  ``grid_struct`` packs it
into the C ABI's ``pg_grid``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from enum import Enum

import numpy as np

from . import _lib
from .errors import InvalidHyperparameter

PRIMARY_PRIMES = (1, 2654435761, 805459861)   # indexing.py:22
AUX_PRIMES = (1, 3674653429, 2097192037)      # indexing.py:23

# seed-stream domains (model.py:21-24)
SEED_FEATURES, SEED_CONFIDENCE, SEED_MLP, SEED_BATCH = 0, 1, 2, 3


class LevelMode(Enum):
    DENSE = "dense"
    HASHED = "hashed"


@dataclass(frozen=True)
class LevelSpec:
    level: int
    resolution: int
    mode: LevelMode

    @property
    def vertex_count_1d(self) -> int:
        return self.resolution + 1


def level_resolution(level: int, n_min: int, n_max: int, n_levels: int) -> int:
    """floor(n_min * b^level) on the geometric ladder, endpoints exact and a
    1e-9 guard against exp() landing just under an integer (indexing.py:66-90)."""
    if n_min < 1 or n_max < n_min:
        raise InvalidHyperparameter(f"need n_max >= n_min >= 1, got {n_min}, {n_max}")
    if n_levels < 1 or not 0 <= level < n_levels:
        raise InvalidHyperparameter(f"level {level} outside [0, {n_levels})")
    if level == 0 or n_levels == 1:
        return n_min
    if level == n_levels - 1:
        return n_max
    growth = (math.log(n_max) - math.log(n_min)) / (n_levels - 1)
    scaled = n_min * math.exp(level * growth)
    r = math.floor(scaled)
    return r + 1 if scaled - r > 1.0 - 1e-9 else r


def build_level_specs(n_min, n_max, n_levels, n_f, d) -> list[LevelSpec]:
    """Dense whenever the full (res+1)^d vertex grid fits the table (indexing.py:93-101)."""
    out = []
    for lv in range(n_levels):
        res = level_resolution(lv, n_min, n_max, n_levels)
        out.append(LevelSpec(lv, res, LevelMode.DENSE if (res + 1) ** d <= n_f else LevelMode.HASHED))
    return out


def _pow2(name, v):
    if v < 1 or v & (v - 1):
        raise InvalidHyperparameter(f"{name}={v} must be a power of two")


@dataclass(frozen=True)
class HyperParams:
    """Model shape; defaults are the reference's recommended image settings."""

    n_f: int = 2**6
    n_c: int = 2**14
    n_p: int = 2**4
    n_levels: int = 16
    feature_dim: int = 2
    n_min: int = 16
    n_max: int = 512
    n_neurons: int = 64
    n_hidden_layers: int = 2
    d: int = 2
    out_dim: int = 3
    out_sigmoid: bool = False

    def validate(self) -> "HyperParams":
        _pow2("n_f", self.n_f)
        _pow2("n_c", self.n_c)
        _pow2("n_p", self.n_p)
        if self.n_f % self.n_p:
            raise InvalidHyperparameter(f"n_p={self.n_p} does not divide n_f={self.n_f}")
        if self.n_p > 256:
            raise InvalidHyperparameter("n_p beyond 8-bit baked storage")
        if self.n_levels < 1:
            raise InvalidHyperparameter("need at least one level")
        if not 1 <= self.n_min <= self.n_max:
            raise InvalidHyperparameter(f"need 1 <= n_min <= n_max, got {self.n_min}, {self.n_max}")
        if self.d not in (2, 3):
            raise InvalidHyperparameter(f"d={self.d} unsupported (need 2 or 3)")
        if self.feature_dim < 1 or self.n_neurons < 1 or self.n_hidden_layers < 1:
            raise InvalidHyperparameter("degenerate decoder shape")
        if self.out_dim < 1:
            raise InvalidHyperparameter("output dimension must be positive")
        # limits of the compiled kernels (cython_backend.py:9-21, model_io.py:207-214)
        if self.feature_dim > _lib.PG_MAX_FEATURE or self.n_levels > _lib.PG_MAX_LEVELS:
            raise InvalidHyperparameter("feature dim / level count beyond compiled limit")
        if self.n_hidden_layers + 1 > _lib.PG_MAX_LAYERS:
            raise InvalidHyperparameter("too many hidden layers for the compiled MLP")
        return self

    @property
    def encoded_width(self) -> int:
        return self.n_levels * self.feature_dim

    def mlp_widths(self) -> list[int]:
        return [self.encoded_width] + [self.n_neurons] * self.n_hidden_layers + [self.out_dim]

    def with_updates(self, **kw) -> "HyperParams":
        return replace(self, **kw)


def seeded_rng(seed: int, domain: int, index: int = 0) -> np.random.Generator:
    """Independent numpy stream per (domain, index) (model.py:24-32) — the
    device model is initialised from these on the host so it starts from the
    reference's exact values."""
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(domain, index)))


def log2_int(n: int) -> int:
    return int(n).bit_length() - 1


def grid_struct(hyper: HyperParams, specs, probed_levels) -> _lib.PgGrid:
    """Pack geometry into pg_grid; ``probed_levels`` lists the probed levels in
    slot order (slot i owns conf[i] / baked[i])."""
    g = _lib.PgGrid()
    g.d, g.n_levels, g.feature_dim = hyper.d, hyper.n_levels, hyper.feature_dim
    g.n_f, g.n_c, g.log2_np = hyper.n_f, hyper.n_c, log2_int(hyper.n_p)
    slot_of = {lv: i for i, lv in enumerate(probed_levels)}
    for s in specs:
        g.res[s.level] = s.resolution
        if s.mode is LevelMode.DENSE:
            g.kind[s.level] = _lib.PG_LEVEL_DENSE
        elif s.level in slot_of:
            g.kind[s.level] = _lib.PG_LEVEL_PROBED
        else:
            g.kind[s.level] = _lib.PG_LEVEL_HASHED
        g.slot[s.level] = slot_of.get(s.level, -1)
    for i in range(3):
        g.primary[i] = PRIMARY_PRIMES[i]
        g.aux[i] = AUX_PRIMES[i]
    return g


def mlp_struct(widths) -> _lib.PgMlp:
    m = _lib.PgMlp()
    m.n_layers = len(widths) - 1
    for i, w in enumerate(widths):
        m.widths[i] = w
    return m
