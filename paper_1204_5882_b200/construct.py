"""construct -- the reference's code construction with density evolution on the GPU.

SURVEY.md 8(f) f2.  The reference builds frozen sets with a discretised
density evolution (DE) that is single-threaded and takes hours at n = 20..24
(construction.py:313-391; `_f_scatter` is ~90 % of it).  Here the grid
tables, base densities and the frozen-set rules stay on the host, restated
from the reference with its own numpy formulas (so the tables are identical
bit for bit), and the tree walk with its f/g transforms runs on the GPU
(`csrc/de.cu`, C ABI `pq_de_*`).

Same names and argument meaning as the reference:
  DeGrid(bins=2048, max_llr=30.0)                         construction.py:70-82
  density_evolution(ch, n, quant, prune_z_eps, prune_i_eps, mass_floor)
                                                          construction.py:313-391
  select_frozen(res, target_fer) -> PolarCode             construction.py:397-418
  select_rate(res, rate) -> PolarCode  (rate-K rule of the BASELINE configs,
                                        over the same lexsort((arange, pe)) order)
with the reference's ValueErrors for invalid arguments.  pe agrees with the
reference to floating-point summation order (tests pin it against fixtures
the reference generated; frozen sets are identical).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .channel import BiAwgn, Bsc
from .codes import PolarCode


@dataclass(frozen=True)
class DeGrid:
    """Density-evolution grid: bin count and LLR half-range (construction.py:70-82)."""

    bins: int = 2048
    max_llr: float = 30.0

    def __post_init__(self):
        if self.bins < 256:
            raise ValueError(f"DE grid needs at least 256 bins, got {self.bins}")
        if self.bins % 2 != 0:
            raise ValueError(f"DE grid bin count must be even, got {self.bins}")
        if not self.max_llr > 0:
            raise ValueError(f"DE grid max_llr must be positive, got {self.max_llr}")


@dataclass(frozen=True)
class ConstructionResult:
    n: int
    channel: object
    pe: np.ndarray
    quantization: DeGrid


def _boxplus_magnitude(a, b):
    # exact |f| for positive magnitudes (construction.py:132-135)
    m = np.minimum(a, b)
    return m + np.log1p(np.exp(-(a + b))) - np.log1p(np.exp(-np.abs(a - b)))


class GridTables:
    """The reference's _GridOps tables (construction.py:164-190), same formulas."""

    def __init__(self, grid: DeGrid):
        self.grid = grid
        self.step = 2.0 * grid.max_llr / grid.bins
        self.center = grid.bins // 2
        self.size = grid.bins + 1
        self.ni = grid.bins - 1
        self.values = (np.arange(1, grid.bins) - self.center) * self.step
        vmin = self.values[0]
        a = self.values[:, None]
        b = self.values[None, :]
        fval = np.sign(a) * np.sign(b) * _boxplus_magnitude(np.abs(a), np.abs(b))
        pos = (fval - vmin) / self.step
        idx = np.floor(pos).astype(np.int32)
        np.clip(idx, 0, self.ni - 2, out=idx)
        self.f_idx = np.ascontiguousarray(idx)
        self.f_whi = np.ascontiguousarray(np.clip(pos - idx, 0.0, 1.0))
        self.z_weights = np.ascontiguousarray(np.exp(-0.5 * self.values))
        self.i_loss = np.ascontiguousarray(np.logaddexp(0.0, -self.values) / np.log(2.0))
        self.z_lo_bound = float(np.exp(grid.max_llr))


_TABLES: dict = {}


def grid_tables(grid: DeGrid) -> GridTables:
    key = (grid.bins, grid.max_llr)
    if key not in _TABLES:
        _TABLES[key] = GridTables(grid)
    return _TABLES[key]


def base_density(ch, t: GridTables) -> np.ndarray:
    """Channel LLR density on the lattice (construction.py:264-296)."""
    grid = t.grid
    m = np.zeros(t.size)
    if isinstance(ch, Bsc):
        if ch.p == 0.0:
            m[-1] = 1.0
            return m
        c = np.log((1.0 - ch.p) / ch.p) if ch.p < 0.5 else 0.0
        for mag, mass in ((c, 1.0 - ch.p), (-c, ch.p)):
            if mag >= grid.max_llr:
                m[-1] += mass
            elif mag <= -grid.max_llr:
                m[0] += mass
            else:
                pos = (mag - t.values[0]) / t.step
                k = int(np.floor(pos))
                frac = pos - k
                m[1 + k] += mass * (1.0 - frac)
                m[1 + k + 1] += mass * frac
        return m
    if isinstance(ch, BiAwgn):
        from scipy.stats import norm

        mu, sd = 2.0 * ch.snr, 2.0 * np.sqrt(ch.snr)
        lo_edge = t.values[0] - 0.5 * t.step
        cdf = norm.cdf(np.concatenate(([lo_edge], t.values + 0.5 * t.step)), mu, sd)
        m[0] = cdf[0]
        m[1:-1] = np.diff(cdf)
        m[-1] = 1.0 - cdf[-1]
        return m
    raise TypeError(f"unsupported channel model: {ch!r}")


class DeEngine:
    """GPU DE for one grid: the tables are uploaded once (pq_de_create)."""

    def __init__(self, grid: DeGrid = DeGrid(), device: int = 0):
        t = grid_tables(grid)
        self.t = t
        self._keep = (t.f_idx, t.f_whi, t.z_weights, t.i_loss)
        self._h = ctypes.c_void_p()
        L = _lib.load()
        _lib.check(L.pq_de_create(ctypes.byref(self._h), grid.bins, t.z_lo_bound, t.f_idx.ctypes.data,
                                  t.f_whi.ctypes.data, t.z_weights.ctypes.data, t.i_loss.ctypes.data,
                                  int(device)), "pq_de_create")

    def run(self, base: np.ndarray, n: int, prune_z_eps: float, prune_i_eps: float, mass_floor: float):
        base = np.ascontiguousarray(base, dtype=np.float64)
        pe = np.empty(1 << n)
        _lib.check(_lib.load().pq_de_run(self._h, base.ctypes.data, n, prune_z_eps, prune_i_eps, mass_floor,
                                         pe.ctypes.data), "pq_de_run")
        return pe

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().pq_de_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ENGINES: dict = {}


def density_evolution(ch, n: int, quant: DeGrid = DeGrid(), prune_z_eps: float = 1e-9,
                      prune_i_eps: float = 1e-3, mass_floor: float = 1e-30) -> ConstructionResult:
    """Per-bit error probabilities of all 2^n synthetic channels, in decoding
    order (construction.py:313-391), computed on the GPU."""
    if not 1 <= n <= 27:
        raise ValueError(f"n must be in [1, 27], got {n}")
    key = (quant.bins, quant.max_llr)
    if key not in _ENGINES:
        _ENGINES[key] = DeEngine(quant)
    eng = _ENGINES[key]
    base = base_density(ch, eng.t)
    if np.count_nonzero(base[1:-1]) == 1 and base[0] == 0.0 and base[-1] == 0.0:
        raise ValueError("DE grid too coarse: the base channel density collapses into a single bin")
    pe = eng.run(base, n, prune_z_eps, prune_i_eps, mass_floor)
    return ConstructionResult(n=n, channel=ch, pe=pe, quantization=quant)


def select_frozen(res: ConstructionResult, target_fer: float) -> PolarCode:
    """Greedy maximum-rate frozen set under the FER union bound
    (construction.py:397-418): information bits in ascending pe (ties by index)
    while the running sum stays within target_fer."""
    if not 0.0 < target_fer < 1.0:
        raise ValueError(f"target FER must be in (0, 1), got {target_fer}")
    order = np.lexsort((np.arange(res.pe.size), res.pe))
    budget = np.cumsum(res.pe[order])
    k = int(np.searchsorted(budget, target_fer, side="right"))
    mask = np.ones(res.pe.size, dtype=np.uint8)
    mask[order[:k]] = 0
    return PolarCode(n=res.n, frozen_mask=mask, channel=res.channel, target_fer=target_fer)


def select_rate(res: ConstructionResult, rate: float) -> PolarCode:
    """Rate-K frozen set: the K = round(rate N) best
    positions of the reference's lexsort((arange, pe)) order are information."""
    if not 0.0 <= rate <= 1.0:
        raise ValueError(f"rate must be in [0, 1], got {rate}")
    N = res.pe.size
    order = np.lexsort((np.arange(N), res.pe))
    mask = np.ones(N, dtype=np.uint8)
    mask[order[: int(round(rate * N))]] = 0
    return PolarCode(n=res.n, frozen_mask=mask, channel=res.channel, target_fer=float("nan"))


__all__ = ["DeGrid", "ConstructionResult", "GridTables", "grid_tables", "base_density", "DeEngine",
           "density_evolution", "select_frozen", "select_rate"]
