"""Stress parity of the specialised svd2 path (kog2_fast.cuh) against the
reference svd2 (svd2.hpp:603-687) on adversarial distributions, 2^21 matrices
each, binary64 and binary32, default Options (the path kog_svd2_batch_f64 specialises): wide and
narrow exponent spreads, every zero pattern, mono/simple patterns with
extreme ratios, near-ties that reach the diag_equal / offdiag_equal / small
ratio / overflow / degenerate branches, rank-one and orthogonal columns.
Every output field bit-exact (tests/test_gpu_parity.py:compare_svd)."""
from __future__ import annotations

import zlib

import numpy as np
import pytest
import torch

from oracle import refbind
from paper_2407_13116_b200 import kogsvd2 as K
from tests import _gen
from tests.test_gpu_parity import compare_svd

pytestmark = pytest.mark.gpu

N = 1 << 21


def _pattern(g: np.ndarray, seed: int) -> np.ndarray:
    """zero a random subset of entries in 1/4 of the matrices (all 16 patterns)"""
    z = _gen.draws(seed, g.shape[1], 7)
    sel = (z & np.uint64(3)) == 0
    m = (z >> np.uint64(2)) & np.uint64(15)
    for row, bit in ((0, 1), (2, 2), (1, 4), (3, 8)):  # g11, g21, g12, g22 in classify's bit order
        g[row] = np.where(sel & ((m & np.uint64(bit)) != 0), 0.0, g[row])
    return g


# exponent ranges per precision: (wide lo, wide hi, huge-condition shift, rank spread)
_RANGES = {np.float64: (-1022, 1023, -1000 + 80, 300), np.float32: (-126, 127, -100, 40)}


def _dist(name: str, seed: int, dt=np.float64) -> np.ndarray:
    elo, ehi, huge, spread = _RANGES[dt]
    rng = np.random.default_rng(seed)
    if name == "wide":  # every normal exponent, zero patterns
        g = np.stack([_gen.stratified(dt, seed, N, elo, ehi, k) for k in range(4)])
        return _pattern(g, seed)
    if name == "narrow":  # one binade: cancellation, near-equal entries
        g = np.stack([_gen.stratified(dt, seed, N, 0, 1, k) for k in range(4)])
        return _pattern(g, seed)
    if name == "near_ties":  # r11 ~ r22, r12 ~ r22, h ~ r22, tan2phi overflow, t13 small ratios
        a = _gen.stratified(dt, seed, N, -40, 40, 0)
        eps = np.ldexp(rng.integers(-4, 5, N).astype(dt), -(np.finfo(dt).nmant))  # a few ulps
        kind = rng.integers(0, 6, N)
        g11, g12, g21, g22 = a.copy(), a * (1 + eps), np.zeros(N), a * (1 - eps)
        g12 = np.where(kind == 1, np.ldexp(a, -60), g12)          # tiny off-diagonal
        g22 = np.where(kind == 2, a, g22)                          # exactly equal diagonal
        g12 = np.where(kind == 3, g22, g12)                        # offdiag == diag
        g21 = np.where(kind == 4, np.ldexp(a, -30), g21)           # full, nearly triangular
        g22 = np.where(kind == 5, np.ldexp(a, huge), g22)          # huge condition number
        g = np.stack([g11, g12, g21, g22]).astype(dt)
        sg = rng.integers(0, 2, (4, N)) * 2 - 1
        return (g * sg).astype(dt)
    if name == "rank":  # rank one / orthogonal columns / permuted diagonal
        x = _gen.stratified(dt, seed, N, -spread, spread, 0)
        y = _gen.stratified(dt, seed, N, -spread, spread, 1)
        k = _gen.stratified(dt, seed, N, -20, 20, 2)
        kind = rng.integers(0, 3, N)
        g11, g21 = x, y
        g12 = np.where(kind == 0, x * np.ldexp(1.0, 3), np.where(kind == 1, -y, y))  # exact multiples / orthogonal
        g22 = np.where(kind == 0, y * np.ldexp(1.0, 3), np.where(kind == 1, x, -x))
        g12 = np.where(kind == 2, x * k, g12)
        g22 = np.where(kind == 2, y * k, g22)
        return np.stack([g11, g12, g21, g22]).astype(dt)
    if name == "mono_simple":  # one nonzero row/column or a permuted diagonal, extreme ratios
        v = np.stack([_gen.stratified(dt, seed, N, elo, ehi, k) for k in range(4)])
        pats = np.array([3, 12, 5, 10, 1, 2, 4, 8, 6, 9, 0])
        t = pats[rng.integers(0, pats.size, N)]
        for row, bit in ((0, 1), (2, 2), (1, 4), (3, 8)):
            v[row] = np.where((t & bit) != 0, v[row], 0.0)
        return v
    if name == "moderate":  # entry ratios within 2^+-90: tan(2phi) and tan(psi) sweep the closed-form
        # thresholds of the fast path (2^-27 and 2^54) continuously
        g = np.stack([_gen.stratified(dt, seed, N, -45, 45, k) for k in range(4)])
        g[2] = np.where(rng.integers(0, 2, N) == 0, 0.0, g[2])  # half upper-triangular (t ~ 13)
        return g
    if name == "subnormal_mix":  # subnormal entries next to normal ones (deferred lanes)
        g = np.stack([_gen.any_finite(dt, seed, N, k) for k in range(4)])
        return g
    raise ValueError(name)


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("name", ["wide", "narrow", "near_ties", "rank", "mono_simple", "moderate", "subnormal_mix"])
def test_fast_path_stress(cuda, ref, name, dt):
    g = np.ascontiguousarray(_dist(name, 0x5EED0000 + zlib.crc32(name.encode()) % 1000, dt))
    assert np.isfinite(g).all()
    got = K.svd2(torch.from_numpy(g).cuda())
    want = refbind.svd2(ref, g)
    compare_svd(got, want, f"stress {name}")
