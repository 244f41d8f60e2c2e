"""The BASELINE.json workloads as RunConfigs (SURVEY.md §8d fixes the draw rules
and seeds; configs 2-5 use the kog2 generator extension KOG_REGIME_RANGED).

  cfg1: 2^20 general f64, uniform (-1,1)          -> Shape::gen, Regime::circ, seed 0xC0FFEE
  cfg2: 2^26 upper-triangular f64, e in [-1000,1000]                       seed 0x05B1
  cfg3: 2^28 general f64, e in [-500,500], 1/8 zero patterns               seed 0x0F1E2D3C
  cfg4: 2^28 general f32, e in [-60,60] + 1% tail e in [-126,-100]         seed 0xF32
  cfg5: 2^31 general f64, the cfg3 rule and seed, sharded by index range
"""
from __future__ import annotations

from . import capi
from .kogsvd2 import RunConfig


def cfg(k: int, count: int | None = None) -> RunConfig:
    if k == 1:
        return RunConfig(single_precision=False, shape=capi.SHAPE_GEN, regime=capi.REGIME_CIRC,
                         count=count if count is not None else 1 << 20, seed=0xC0FFEE)
    if k == 2:
        return RunConfig(single_precision=False, shape=capi.SHAPE_TRI, regime=capi.REGIME_RANGED,
                         count=count if count is not None else 1 << 26, seed=0x05B1, elo=-1000, ehi=1000)
    if k in (3, 5):
        return RunConfig(single_precision=False, shape=capi.SHAPE_GEN, regime=capi.REGIME_RANGED,
                         count=count if count is not None else (1 << 28 if k == 3 else 1 << 31),
                         seed=0x0F1E2D3C, elo=-500, ehi=500, zero_mask_rule=1)
    if k == 4:
        return RunConfig(single_precision=True, shape=capi.SHAPE_GEN, regime=capi.REGIME_RANGED,
                         count=count if count is not None else 1 << 28, seed=0xF32, elo=-60, ehi=60,
                         tail_lo=-126, tail_hi=-100, tail_mod=100)
    raise ValueError(f"unknown config {k}")


FULL_SIZE = {1: 1 << 20, 2: 1 << 26, 3: 1 << 28, 4: 1 << 28, 5: 1 << 31}

# bytes per matrix of the decomposition (SoA in + compact out)
BYTES_PER_MATRIX = {"f64": 32 + 64, "f32": 16 + 40}
