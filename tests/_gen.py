"""Seeded numpy input generators and exact references for the tests.

The distributions follow the reference's test RNG (proj/tests/test_rng.hpp:
any_finite 45-60, stratified 36-42, positive 63-66) but are drawn with a
counter-based splitmix64 so they vectorise: every element owns its draws
mix64(seed + gamma * (4*i + k + 1)), k = 0..3.  hypot_exact follows the
integer-arithmetic reference of proj/tests/exact_ref.hpp:66-99 with Python
big integers in place of Boost cpp_int.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

FMT = {np.float64: (53, 1023, -1022), np.float32: (24, 127, -126)}


def mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def draws(seed: int, n: int, k: int, salt: int = 0) -> np.ndarray:
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        c = np.uint64(seed) + GAMMA * (np.uint64(8) * i + np.uint64(k + 1 + 4 * salt))
    return mix64(c)


def unit(u: np.ndarray) -> np.ndarray:
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def stratified(dt, seed: int, n: int, elo: int, ehi: int, salt: int = 0) -> np.ndarray:
    """sign * mantissa in [1,2) * 2^e, e uniform in [elo, ehi] (test_rng.hpp:36-42)."""
    ue, uf, us = draws(seed, n, 0, salt), draws(seed, n, 1, salt), draws(seed, n, 2, salt)
    e = elo + (ue % np.uint64(ehi - elo + 1)).astype(np.int64)
    f = np.minimum(dt(1) + unit(uf).astype(dt), np.nextafter(dt(2), dt(0)))  # never round up to 2
    v = np.ldexp(f, e.astype(np.int32)).astype(dt)
    return np.where((us & np.uint64(1)) != 0, -v, v).astype(dt)


def any_finite(dt, seed: int, n: int, salt: int = 0) -> np.ndarray:
    """any finite value incl. subnormals and the extremes (test_rng.hpp:45-60)."""
    p, emax, emin = FMT[dt]
    fi = np.finfo(dt)
    sub_min = dt(fi.smallest_subnormal)
    case = draws(seed, n, 3, salt) % np.uint64(16)
    sgn = (draws(seed, n, 2, salt) & np.uint64(1)) != 0
    out = stratified(dt, seed, n, emin, emax, salt)
    sub = stratified(dt, seed + 1, n, emin - p + 1, emin - 1, salt)
    out = np.where(case == 4, sub, out)
    out = np.where(case == 0, dt(0), out)
    out = np.where(case == 1, np.where(sgn, -sub_min, sub_min), out)
    out = np.where(case == 2, np.where(sgn, -fi.max, fi.max), out)
    out = np.where(case == 3, np.where(sgn, -fi.tiny, fi.tiny), out)
    return out.astype(dt)


def positive(dt, seed: int, n: int, elo: int, ehi: int, salt: int = 0) -> np.ndarray:
    return np.abs(stratified(dt, seed, n, elo, ehi, salt))


def matrices(dt, seed: int, n: int, kind: str = "any_finite") -> np.ndarray:
    """(4, n) batch g11, g12, g21, g22."""
    if kind == "any_finite":
        rows = [any_finite(dt, seed, n, salt=k) for k in range(4)]
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(np.stack(rows))


def bits(a: np.ndarray) -> np.ndarray:
    """Bit patterns for exact comparison (distinguishes -0.0 and NaN payloads)."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        return a.view(np.uint64)
    if a.dtype == np.float32:
        return a.view(np.uint32)
    return a


def assert_bits_equal(got: np.ndarray, want: np.ndarray, what: str = "") -> None:
    g, w = bits(got), bits(want)
    bad = np.nonzero(g != w)[0]
    if bad.size:
        i = bad[0]
        raise AssertionError(f"{what}: {bad.size} mismatches; first at {i}: got {got[i]!r} want {want[i]!r}")


# ------------------------------------------------------ exact references
def _dyadic(x: float, p: int) -> tuple[int, int]:
    """x = m * 2^t exactly, |m| < 2^p (exact_ref.hpp:27-35)."""
    fr, be = math.frexp(float(x))
    m = int(math.ldexp(fr, p))
    return m, be - p


def hypot_exact(a: float, b: float, dt) -> float:
    """Correctly rounded sqrt(a^2+b^2) in format dt by integer arithmetic
    (exact_ref.hpp:66-99)."""
    p, emax, emin = FMT[dt]
    if math.isinf(a) or math.isinf(b):
        return math.inf
    if math.isnan(a) or math.isnan(b):
        return math.nan
    big, small = abs(float(a)), abs(float(b))
    if big < small:
        big, small = small, big
    if small == 0:
        return big
    ma, ta = _dyadic(big, p)
    mb, tb = _dyadic(small, p)
    tmin = min(2 * ta, 2 * tb)
    s = (ma * ma << (2 * ta - tmin)) + (mb * mb << (2 * tb - tmin))
    lbits = s.bit_length() - 1
    k = max(0, p + 3 - lbits // 2)
    n = s << (2 * k)
    isq = math.isqrt(n)
    exact = isq * isq == n
    t = tmin // 2 - k
    er = (isq.bit_length() - 1) + t
    tg = max(er - (p - 1), emin - (p - 1))
    sh = tg - t
    n0 = isq >> sh
    guard = (isq >> (sh - 1)) & 1
    sticky = (isq & ((1 << (sh - 1)) - 1)) != 0 or not exact
    if guard and (sticky or (n0 & 1)):
        n0 += 1
    try:
        v = math.ldexp(float(n0), tg)
    except OverflowError:
        v = math.inf
    if dt == np.float32:
        return float(np.float32(v)) if v <= float(np.finfo(np.float32).max) else math.inf
    return v


def exact_fraction(x: float) -> Fraction:
    return Fraction(x)


import contextlib


@contextlib.contextmanager
def study_chunk(log2: int):
    """The phased study's chunk at 2^log2 matrices for the enclosed calls (kog_study_set_chunk_log2): the
    multi-chunk pipeline is exercised at counts the CPU reference finishes in seconds."""
    from paper_2407_13116_b200 import capi
    lib = capi.load()
    before = lib.kog_study_set_chunk_log2(log2)
    try:
        yield
    finally:
        lib.kog_study_set_chunk_log2(before)
