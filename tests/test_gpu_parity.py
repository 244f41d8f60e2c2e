"""CUDA path vs the oracle: bit-exact parity through the C-ABI (libkog2.so).

The oracle here is the reference itself (oracle/_ref/libkogref.so, compiled
from the unmodified headers) and, where the two are interchangeable, the
plain-C restatement.  Every comparison is on bit patterns (signed zeros
included).  Mirrors the reference's suites: fpcore_test.cpp (hypot vs exact,
ties, edges), svd2_test.cpp (phases, options), oracle_test.cpp, harness_test.cpp.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import refbind
from paper_2407_13116_b200 import capi, configs
from paper_2407_13116_b200 import kogsvd2 as K
from tests import _gen

pytestmark = pytest.mark.gpu

DTS = [np.float64, np.float32]
TDT = {np.float64: torch.float64, np.float32: torch.float32}


def dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def compare_svd(got: dict, want: dict, what: str) -> None:
    """Bit-exact on every field; where the reference threw (non-finite input,
    KOG_F_DOMAIN_ERROR) only the error bit itself is compared."""
    gf = (host(got["flags"]) if isinstance(got["flags"], torch.Tensor) else got["flags"]).view(np.uint32)
    err = (want["flags"] & np.uint32(capi.F_DOMAIN_ERROR)) != 0
    assert ((gf & np.uint32(capi.F_DOMAIN_ERROR)) != 0).tolist() == err.tolist(), f"{what}: domain-error bits"
    ok = ~err
    for k in refbind.OUT_DTYPES:
        g = host(got[k]) if isinstance(got[k], torch.Tensor) else got[k]
        if k == "flags":
            g = g.view(np.uint32)
        _gen.assert_bits_equal(g[ok], want[k][ok], f"{what}.{k}")


def records_equal(got, want, what: str) -> None:
    """Field-by-field byte equality of two ctypes record arrays (padding ignored)."""
    rt = type(got[0])
    for name, ft in rt._fields_:
        off, size = getattr(rt, name).offset, C.sizeof(ft)
        gb = np.frombuffer(bytes(got), np.uint8).reshape(len(got), -1)[:, off:off + size]
        wb = np.frombuffer(bytes(want), np.uint8).reshape(len(want), -1)[:, off:off + size]
        bad = np.nonzero((gb != wb).any(axis=1))[0]
        assert bad.size == 0, f"{what}.{name}: {bad.size} records differ, first {bad[0]}"


ALL_OPTIONS = [capi.kog_options(h, o, w, 0) for h in (1, 0) for o in (0, 1) for w in (0, 1)]


def K_opt(o: capi.kog_options) -> K.Options:
    return K.Options(bool(o.hypot_is_cr), bool(o.ominus_for_d), int(o.wide_channel))


# ------------------------------------------------------------ fpcore
@pytest.mark.parametrize("dt", DTS)
def test_hypot_matches_reference_and_exact(cuda, ref, dt):
    """fpcore_test.cpp:40-50 (10^6 any_finite pairs vs the exact reference)."""
    n = 1_000_000
    a = _gen.any_finite(dt, 0x68790001, n, 0)
    b = _gen.any_finite(dt, 0x68790001, n, 1)
    got = host(K.hypot_cr(dev(a), dev(b)))
    want = np.empty_like(a)
    (ref.hypot_f64 if dt == np.float64 else ref.hypot_f32)(a.ctypes.data, b.ctypes.data, want.ctypes.data, n)
    _gen.assert_bits_equal(got, want, "hypot vs reference")
    ex = np.array([_gen.hypot_exact(x, y, dt) for x, y in zip(a[:20000], b[:20000])], dtype=dt)
    _gen.assert_bits_equal(got[:20000], ex, "hypot vs exact integer reference")


@pytest.mark.parametrize("dt", DTS)
def test_hypot_exact_ties(cuda, dt):
    """fpcore_test.cpp:53-73: scaled 3-4-5 triples whose hypotenuse is a midpoint."""
    p = 53 if dt == np.float64 else 24
    lo, hi = (1 << p) // 5 + 1, ((1 << (p + 1)) - 1) // 5
    rng = np.random.default_rng(0x68790002)
    q = rng.integers(lo, hi + 1, size=20000, dtype=np.int64) | 1
    q = q[(5 * q >= (1 << p)) & (5 * q < (1 << (p + 1)))]
    x = rng.integers(-40, 41, size=q.size)
    a = np.ldexp((3 * q).astype(np.float64), x).astype(dt)
    b = np.ldexp((4 * q).astype(np.float64), x).astype(dt)
    got = host(K.hypot_cr(dev(a), dev(b)))
    ex = np.array([_gen.hypot_exact(u, v, dt) for u, v in zip(a, b)], dtype=dt)
    assert q.size > 1000
    _gen.assert_bits_equal(got, ex, "hypot ties")


def test_divf_near_midpoints(cuda):
    """binary32 quotients as close to a rounding midpoint as 24-bit operands
    allow: for an odd 25-bit M, Y = c M^-1 mod 2^25 (24 bits) makes
    M Y = X 2^25 + c with |c| <= 8, so X 2^25 / Y lies c/(M Y) ~ 2^-49 .. 2^-45
    (relative) from the midpoint M; a quotient approximation off by 2^-46
    misrounds ~28% of them.  The unit kernel's div_rn<float>, which shares
    div_mant_f (kog2_fp.cuh) with svd2's fast path, equals IEEE x / y."""
    rng = np.random.default_rng(0xD21)
    n = 4_000_000
    mod = np.int64(1) << 25
    M = rng.integers(1 << 24, 1 << 25, size=n, dtype=np.int64) | 1
    inv = M.copy()
    for _ in range(5):  # Newton's iteration for M^-1 mod 2^25
        inv = (inv * ((2 - M * inv) % mod)) % mod
    c = rng.integers(1, 9, size=n) * np.where(rng.random(n) < 0.5, 1, -1)
    Y = (inv * (c % mod)) % mod
    P = M * Y
    ok = (Y >= 1 << 23) & (Y < 1 << 24) & (P - c >= np.int64(1) << 48)
    Y, P, c = Y[ok], P[ok], c[ok]
    X = (P - c) >> 25
    assert ((X << 25) + c == P).all() and (X >= 1 << 23).all() and (X < 1 << 24).all() and X.size > 500_000
    m = X.size
    e = rng.integers(-60, 61, size=m)
    x = np.ldexp(X.astype(np.float64), e + 2).astype(np.float32)
    y = np.ldexp(Y.astype(np.float64), e - 23 - rng.integers(0, 8, size=m)).astype(np.float32)
    x = np.where(rng.random(m) < 0.5, x, -x).astype(np.float32)
    got = torch.empty(m, dtype=torch.float32, device="cuda")
    dx, dy = dev(x), dev(y)
    capi.check(capi.load().kog_div_batch_f32(dx.data_ptr(), dy.data_ptr(), got.data_ptr(), m,
                                             torch.cuda.current_stream().cuda_stream))
    _gen.assert_bits_equal(host(got), x / y, "binary32 division near midpoints")


def test_divf_every_divisor_significand(cuda):
    """Every binary32 divisor significand Y (2^23 of them) against a dividend
    whose quotient lies next to a midpoint: with Y = 2^j Yo (Yo odd),
    M = c' Yo^-1 mod 2^(25-j) lifted into [2^24, 2^25) makes M Y = X 2^25 + c,
    c = c' 2^j, |c'| < 130 (found for 99.6% of the significands; the rest are
    dropped).  This pins rcp_mant_f's single Newton step for every seed the
    reciprocal instruction can see (kog2_fp.cuh)."""
    rng = np.random.default_rng(0xD22)
    Y = np.arange(1 << 23, 1 << 24, dtype=np.int64)
    j = np.zeros_like(Y)
    Yo = Y.copy()
    for _ in range(23):
        ev = (Yo & 1) == 0
        Yo[ev] >>= 1
        j[ev] += 1
    mod = np.int64(1) << 25
    inv = Yo.copy()
    for _ in range(5):  # Newton's iteration for Yo^-1 mod 2^25
        inv = (inv * ((2 - Yo * inv) % mod)) % mod
    modj = np.int64(1) << (25 - j)
    M = np.zeros_like(Y)
    c = np.zeros_like(Y)
    sgn = np.where(rng.random(Y.size) < 0.5, 1, -1)
    todo = np.arange(Y.size)
    for cp in range(1, 130, 2):
        mj = modj[todo]
        cs = cp * sgn[todo]
        M0 = ((cs % mj) * inv[todo]) % mj
        lo = ((np.int64(1) << 24) - M0 + mj - 1) // mj
        hi = ((np.int64(1) << 25) - 1 - M0) // mj
        t = np.minimum(lo + (rng.random(todo.size) * (hi - lo + 1)).astype(np.int64), hi)
        ok = lo <= hi
        M[todo[ok]] = (M0 + t * mj)[ok]
        c[todo[ok]] = (cs << j[todo])[ok]
        todo = todo[~ok]
        if todo.size == 0:
            break
    keep = M != 0
    assert keep.mean() > 0.99
    M, c, Y = M[keep], c[keep], Y[keep]
    P = M * Y
    assert ((P - c) % mod == 0).all() and (M >= 1 << 24).all() and (M < 1 << 25).all() and (M & 1).all()
    X = (P - c) >> 25
    assert (X > 0).all() and (X < 1 << 24).all()
    e = rng.integers(-60, 61, size=Y.size)
    x = np.ldexp(X.astype(np.float64), e + 2).astype(np.float32)
    y = np.ldexp(Y.astype(np.float64), e - 23).astype(np.float32)
    x = np.where(rng.random(Y.size) < 0.5, x, -x).astype(np.float32)
    got = torch.empty(Y.size, dtype=torch.float32, device="cuda")
    dx, dy = dev(x), dev(y)
    capi.check(capi.load().kog_div_batch_f32(dx.data_ptr(), dy.data_ptr(), got.data_ptr(), Y.size,
                                             torch.cuda.current_stream().cuda_stream))
    _gen.assert_bits_equal(host(got), x / y, "binary32 division, every divisor significand")


def _subnormal_tie_quotients(rng, n: int):
    """binary32 pairs whose exact quotient is a subnormal midpoint k 2^-150
    (k odd, up to 2^23 + ...), e.g. 0x1.74d94ap-101 / 0x1.f121b8p+47 = 3 2^-150:
    y = Y 2^ey, x = k Y 2^(ey-150) with k Y < 2^24.  Half of them are nudged to
    the neighbouring dividend (x +- 1 ulp), which lies just off the tie."""
    kbits = rng.integers(1, 24, size=n)
    k = (rng.integers(0, 1 << 62, size=n) >> (62 - kbits)) | 1
    ybits = 24 - np.ceil(np.log2(k + 1)).astype(np.int64)
    Y = np.maximum(rng.integers(0, 1 << 62, size=n) >> (62 - np.maximum(ybits, 1)), 1)
    Y = np.where(k * Y < (1 << 24), Y, 1)
    ey = rng.integers(1, 128 - 24, size=n)  # x on the binary32 grid: ey - 150 >= -149
    y = np.ldexp(Y.astype(np.float64), ey).astype(np.float32)
    x = np.ldexp((k * Y).astype(np.float64), ey - 150).astype(np.float32)
    assert (np.ldexp((k * Y).astype(np.float64), ey - 150) == x.astype(np.float64)).all()
    nudge = rng.random(n) < 0.5
    x = np.where(nudge, np.nextafter(x, np.where(rng.random(n) < 0.5, np.float32(0), np.float32(1))), x)
    sgn = np.where(rng.random(n) < 0.5, np.float32(1), np.float32(-1))
    return (x * sgn).astype(np.float32), np.where(rng.random(n) < 0.5, y, -y).astype(np.float32)


def test_divf_subnormal_ties(cuda):
    """binary32 quotients that are exact subnormal midpoints (round half to
    even on the 2^-149 grid) and their neighbours: div_rn<float> (quot_f's
    residual step, kog2_fp.cuh) equals IEEE x / y."""
    rng = np.random.default_rng(0xD23)
    x, y = _subnormal_tie_quotients(rng, 1 << 20)
    ties = (np.abs(x.astype(np.float64) / y.astype(np.float64)) < 2.0 ** -126)
    assert ties.mean() > 0.9
    got = torch.empty(x.size, dtype=torch.float32, device="cuda")
    dx, dy = dev(x), dev(y)
    capi.check(capi.load().kog_div_batch_f32(dx.data_ptr(), dy.data_ptr(), got.data_ptr(), x.size,
                                             torch.cuda.current_stream().cuda_stream))
    _gen.assert_bits_equal(host(got), x / y, "binary32 subnormal tie quotients")


def test_svd2_f32_subnormal_tan_theta(cuda, ref):
    """binary32 svd2 whose tan(theta) = |g21| / |g11| is an exact subnormal
    midpoint (or next to one): the fast path's div_n<float> and the general
    kernel's div_rn<float> (every Options combination) equal the reference."""
    rng = np.random.default_rng(0x5B7)
    n = 1 << 18
    x, y = _subnormal_tie_quotients(rng, n)
    y = np.where(np.abs(y) < 2.0 ** -100, np.float32(1.5), y).astype(np.float32)
    small = lambda: (np.where(rng.random(n) < 0.5, -1.0, 1.0) * (1 + rng.random(n))
                     * np.exp2(rng.integers(-40, -20, n)) * np.abs(y.astype(np.float64))).astype(np.float32)
    g = np.ascontiguousarray(np.stack([y, small(), x, small()]).astype(np.float32))
    for o in ALL_OPTIONS:
        compare_svd(K.svd2(dev(g), K_opt(o)), refbind.svd2(ref, g, o), f"f32 subnormal tan(theta) {K_opt(o)}")


def test_hypotf_near_midpoints(cuda, ref):
    """binary32 hypot whose exact value lies 2^-58 .. 2^-41.6 (relative) from
    a rounding midpoint (28% below 2^-46, median 2^-44.8): either side of the
    fast path's decision tolerance (kog2_fp.cuh hypot_main<float>).
    m = M 2^-24 (M odd, 25 bits) is a midpoint, a = (M - 1 - 2t) 2^-24 a float below it, and b the float
    nearest sqrt(m^2 - a^2) moved by j ulps, so a^2 + b^2 - m^2 is about
    j 2^-24 of b^2.  Results equal the reference and the exact value."""
    rng = np.random.default_rng(0x68790005)
    n = 60_000
    M = rng.integers(1 << 24, 1 << 25, size=n, dtype=np.int64) | 1
    t = rng.integers(0, 4, size=n)
    A = M - 1 - 2 * t
    c = M * M - A * A
    b0 = np.sqrt(c.astype(np.float64)) * 2.0 ** -24
    b = b0.astype(np.float32)
    j = rng.integers(-3, 4, size=n).astype(np.int32)
    b = (b.view(np.int32) + j).view(np.float32)
    x = rng.integers(-40, 41, size=n)
    a = np.ldexp(A.astype(np.float64) * 2.0 ** -24, x).astype(np.float32)
    b = np.ldexp(b.astype(np.float64), x).astype(np.float32)
    a = np.where(rng.random(n) < 0.5, a, -a).astype(np.float32)
    sw = rng.random(n) < 0.5
    a, b = np.where(sw, b, a).astype(np.float32), np.where(sw, a, b).astype(np.float32)
    got = host(K.hypot_cr(dev(a), dev(b)))
    want = np.empty_like(a)
    ref.hypot_f32(a.ctypes.data, b.ctypes.data, want.ctypes.data, n)
    _gen.assert_bits_equal(got, want, "hypotf near midpoints vs reference")
    ex = np.array([_gen.hypot_exact(u, v, np.float32) for u, v in zip(a[:20000], b[:20000])], dtype=np.float32)
    _gen.assert_bits_equal(got[:20000], ex, "hypotf near midpoints vs exact")


@pytest.mark.parametrize("dt", DTS)
def test_hypot_near_the_early_out(cuda, ref, dt):
    """Ratios small/big around kog2's widened early-out (2^-27 in double,
    2^-12 in single): results equal the reference and the exact value, incl.
    sec = hypot(t, 1) and big mantissas near 2 (largest relative half-ulp)."""
    n = 400_000
    rng = np.random.default_rng(0x68790003)
    p = 53 if dt == np.float64 else 24
    k = -np.arange(p // 2 - 8, p // 2 + 8)[rng.integers(0, 16, n)] if dt == np.float64 else \
        -np.arange(4, 20)[rng.integers(0, 16, n)]
    mb = np.where(rng.random(n) < 0.5, 2 - rng.random(n) * 2.0 ** -20, 1 + rng.random(n))
    big = np.ldexp(mb, rng.integers(-60, 60, n))
    small = big * np.ldexp(1 + rng.random(n), k)
    a = big.astype(dt)
    b = np.where(rng.random(n) < 0.25, np.ones(n), small).astype(dt)
    a, b = np.where(rng.random(n) < 0.5, a, -a).astype(dt), b
    sw = rng.random(n) < 0.5
    a, b = np.where(sw, b, a).astype(dt), np.where(sw, a, b).astype(dt)
    got = host(K.hypot_cr(dev(a), dev(b)))
    want = np.empty_like(a)
    (ref.hypot_f64 if dt == np.float64 else ref.hypot_f32)(a.ctypes.data, b.ctypes.data, want.ctypes.data, n)
    _gen.assert_bits_equal(got, want, "hypot near the early-out")
    ex = np.array([_gen.hypot_exact(x, y, dt) for x, y in zip(a[:20000], b[:20000])], dtype=dt)
    _gen.assert_bits_equal(got[:20000], ex, "hypot near the early-out vs exact")
    t = np.ldexp(1 + rng.random(n), -np.arange(10, 40)[rng.integers(0, 30, n)]).astype(dt)
    sec = host(K.sec_from_tan(dev(t)))
    want = np.empty_like(t)
    one = np.ones_like(t)
    (ref.hypot_f64 if dt == np.float64 else ref.hypot_f32)(t.ctypes.data, one.ctypes.data, want.ctypes.data, n)
    _gen.assert_bits_equal(sec, want, "sec near the early-out")


@pytest.mark.parametrize("dt", DTS)
def test_hypot_adversarial_edges(cuda, ref, dt):
    """fpcore_test.cpp:75-89 plus inf/NaN conventions (fpcore.hpp:142-143)."""
    fi = np.finfo(dt)
    mc, mu, nu = fi.smallest_subnormal, fi.tiny, fi.max
    edge = np.array([0, mc, 2 * mc, mu, mu / 2, 1, 1 + fi.eps, nu, nu / 2, nu / 4, np.sqrt(nu), np.sqrt(mu),
                     3, 4, 0.5, 1.5], dtype=dt)
    e = np.concatenate([edge, -edge])
    a, b = np.meshgrid(e, e)
    a, b = a.ravel().astype(dt), b.ravel().astype(dt)
    got = host(K.hypot_cr(dev(a), dev(b)))
    want = np.empty_like(a)
    (ref.hypot_f64 if dt == np.float64 else ref.hypot_f32)(a.ctypes.data, b.ctypes.data, want.ctypes.data, a.size)
    _gen.assert_bits_equal(got, want, "hypot edges")
    sp = np.array([np.inf, -np.inf, np.nan, 1.0, np.nan], dtype=dt)
    sq = np.array([2.0, 1.0, 1.0, -np.inf, -np.inf], dtype=dt)
    g2 = host(K.hypot_cr(dev(sp), dev(sq)))
    assert np.isinf(g2[0]) and np.isinf(g2[1]) and np.isnan(g2[2]) and np.isinf(g2[3]) and np.isinf(g2[4])
    # a NaN in either place next to every edge value (normal, subnormal, zero): NaN (a + b)
    nan = np.full(e.size, np.nan, dtype=dt)
    assert np.isnan(host(K.hypot_cr(dev(e), dev(nan)))).all()
    assert np.isnan(host(K.hypot_cr(dev(nan), dev(e)))).all()
    assert float(host(K.hypot_cr(dev(np.array([nu], dt)), dev(np.array([1], dt))))[0]) == float(nu)


@pytest.mark.parametrize("dt", DTS)
def test_division_correctly_rounded(cuda, dt):
    """div_rn (the division every svd2 quotient uses) == IEEE x / y (numpy),
    on any-finite pairs, significand-only pairs and near-1/near-2 patterns."""
    n = 4_000_000
    x = _gen.any_finite(dt, 0xD1F, n, 0)
    y = _gen.any_finite(dt, 0xD1F, n, 1)
    p = 53 if dt == np.float64 else 24
    ut = np.uint64 if dt == np.float64 else np.uint32
    one = np.array([1.0], dtype=dt).view(ut)[0]
    m = _gen.draws(0xD20, n, 0) >> np.uint64(64 - (p - 1))
    k = _gen.draws(0xD20, n, 1) >> np.uint64(64 - (p - 1))
    xm = (one | m.astype(ut)).view(dt)
    ym = (one | k.astype(ut)).view(dt)
    lo_bits = (np.arange(n) % 64).astype(ut)
    near = (one | lo_bits).view(dt)  # 1 + j ulp
    far = (np.array([np.nextafter(dt(2), dt(0))], dt).view(ut)[0] - lo_bits).view(dt)  # 2 - j ulp
    cases = [(x, y), (xm, ym), (near, far), (far, near), (xm * dt(2.0) ** 900 if dt == np.float64 else xm * dt(2.0) ** 100, ym)]
    for a, b in cases:
        a, b = np.ascontiguousarray(a, dtype=dt), np.ascontiguousarray(b, dtype=dt)
        got = torch.empty(n, dtype=TDT[dt], device="cuda")
        da, db = dev(a), dev(b)  # keep both alive across the launch
        capi.check(getattr(capi.load(), f"kog_div_batch_{'f64' if dt == np.float64 else 'f32'}")(
            da.data_ptr(), db.data_ptr(), got.data_ptr(), n, torch.cuda.current_stream().cuda_stream))
        with np.errstate(all="ignore"):
            want = a / b
        g = host(got)
        nan = np.isnan(want)
        bad = np.nonzero(np.isnan(g) != nan)[0]
        assert bad.size == 0, f"{bad.size} NaN mismatches, first {a[bad[0]]!r} / {b[bad[0]]!r} -> {g[bad[0]]!r}"
        _gen.assert_bits_equal(g[~nan], want[~nan], "div_rn")


@pytest.mark.parametrize("dt", DTS)
def test_split_assemble_tan_sec(cuda, ref, dt):
    """fpcore_test.cpp:115-213 surfaces, bit-exact against the reference."""
    n = 300_000
    x = _gen.any_finite(dt, 0x68790005, n)
    x[:6] = np.array([0, -0.0, np.inf, -np.inf, np.nan, 1.5], dtype=dt)
    e, f = K.split(dev(x))
    we, wf = np.empty(n, np.int64), np.empty_like(x)
    (ref.split_f64 if dt == np.float64 else ref.split_f32)(x.ctypes.data, we.ctypes.data, wf.ctypes.data, n)
    assert (host(e) == we).all()
    _gen.assert_bits_equal(host(f)[6:], wf[6:], "split.f")
    ee = (np.arange(n, dtype=np.int64) % 4000) - 2000
    ee[:4] = [-200000, 200000, -1100, 1100]
    got = host(K.assemble(dev(ee), dev(wf)))
    want = np.empty_like(x)
    (ref.assemble_f64 if dt == np.float64 else ref.assemble_f32)(ee.ctypes.data, wf.ctypes.data, want.ctypes.data, n)
    _gen.assert_bits_equal(got[6:], want[6:], "assemble")
    t = _gen.any_finite(dt, 0x68790006, n)
    t[:4] = np.array([np.inf, -np.inf, 0, 4 / 3], dtype=dt)
    for name, fn, rf in (("tan2", K.tan_from_double_angle, "tan2"), ("sec", K.sec_from_tan, "sec")):
        got = host(fn(dev(t)))
        want = np.empty_like(t)
        getattr(ref, f"{rf}_{'f64' if dt == np.float64 else 'f32'}")(t.ctypes.data, want.ctypes.data, n)
        _gen.assert_bits_equal(got, want, name)


@pytest.mark.parametrize("dt", DTS)
def test_epair_ops(cuda, ref, dt):
    """epair_test.cpp: every EPair operation incl. the throwing cases."""
    p, emax, emin = _gen.FMT[dt]
    n = 200_000
    x = _gen.positive(dt, 0x45500002, n, emin - p + 1, emax, 0)
    y = _gen.positive(dt, 0x45500002, n, emin - p + 1, emax, 1)
    y[::97] = x[::97]  # x == y cases
    xs = np.where(np.arange(n) % 3 == 0, -x, x).astype(dt)
    xs[::1009] = 0
    ex = ((np.arange(n) * 7919) % 2001 - 1000).astype(np.int64)
    ey = ((np.arange(n) * 104729) % 2001 - 1000).astype(np.int64)
    suf = "f64" if dt == np.float64 else "f32"
    for op in range(7):
        xf = x if op in (capi.EPAIR_OPLUS, capi.EPAIR_OMINUS) else xs
        ge, gf, gs = K.epair_op(op, dev(xf), dev(y), dev(ex), dev(ey))
        we, wf, ws = np.empty(n, np.int64), np.empty_like(x), np.empty(n, np.uint8)
        getattr(ref, f"epair_{suf}")(op, ex.ctypes.data, xf.ctypes.data, ey.ctypes.data, y.ctypes.data,
                                     we.ctypes.data, wf.ctypes.data, ws.ctypes.data, n)
        assert (host(gs) == ws).all(), f"op {op} status"
        ok = ws == 0
        assert (host(ge)[ok] == we[ok]).all(), f"op {op} e"
        _gen.assert_bits_equal(host(gf)[ok], wf[ok], f"op {op} f")


# ------------------------------------------------------- classify / phases
def ref_classify(ref, g):
    n = g.shape[1]
    o = {"t": np.empty(n, np.uint8), "s_type": np.empty(n, np.int32), "s": np.empty(n, np.int64),
         "e_G": np.empty(n, np.int64), "inexact_underflow": np.empty(n, np.uint8), "status": np.empty(n, np.uint8)}
    gp = np.empty_like(g)
    co = capi.kog_classify_out(*[o[k].ctypes.data for k in ("t", "s_type", "s", "e_G", "inexact_underflow", "status")])
    fn = ref.classify_prescale_f64 if g.dtype == np.float64 else ref.classify_prescale_f32
    fn(C.byref(refbind.mat(g)), C.byref(co), C.byref(refbind.mat(gp)), n)
    o["gp"] = gp
    return o


@pytest.mark.parametrize("dt", DTS)
def test_classify_prescale(cuda, ref, dt):
    """classify_test.cpp: type table, e_G, s, prescale, inexact underflow."""
    n = 200_000
    g = _gen.matrices(dt, 0xC1A50002, n)
    mask = (_gen.draws(7, n, 0) % np.uint64(16)).astype(np.int64)
    for k, bit in enumerate((1, 4, 2, 8)):  # rows g11,g12,g21,g22 <- bits 0,2,1,3
        g[k][(mask & bit) == 0] = 0
    g[:, 0] = [np.finfo(dt).max, np.finfo(dt).smallest_subnormal, np.finfo(dt).smallest_subnormal,
               np.finfo(dt).smallest_subnormal]
    g[:, 1] = [np.inf, 0, 0, 1]
    got = K.classify_prescale(dev(g))
    want = ref_classify(ref, g)
    assert (host(got["status"]) == want["status"]).all()
    ok = want["status"] == 0
    for k in ("t", "s_type", "s", "e_G", "inexact_underflow"):
        assert (host(got[k])[ok] == want[k][ok]).all(), k
    _gen.assert_bits_equal(host(got["gp"])[:, ok].ravel(), want["gp"][:, ok].ravel(), "gp")


@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("wide", [0, 1])
def test_urv15(cuda, ref, dt, wide):
    """urv15 on full matrices (svd2_test.cpp:156-191, 395-428), both wide channels."""
    n = 200_000
    p, emax, emin = _gen.FMT[dt]
    g = np.ascontiguousarray(np.stack([_gen.stratified(dt, 0x57D20006, n, emin, emax - 2, k) for k in range(4)]))
    g[:, 0] = [2, 1, 1, 2]
    g[:, 1] = [1, 1, 1, -1]
    g[:, 2] = [2, 4, 1, 2]
    opt = K.Options(wide_channel=wide)
    got = K.urv15(dev(g), opt)
    rt = capi.kog_urv15_f64 if dt == np.float64 else capi.kog_urv15_f32
    want = refbind.records(rt, n)
    (ref.urv15_f64 if dt == np.float64 else ref.urv15_f32)(C.byref(refbind.mat(g)), C.addressof(want), n,
                                                           C.byref(opt.c()))
    records_equal(got, want, "urv15")


@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("opt", ALL_OPTIONS[:4], ids=lambda o: f"cr{o.hypot_is_cr}om{o.ominus_for_d}")
def test_tri_svd(cuda, ref, dt, opt):
    """tri_svd / tan2phi (svd2_test.cpp:193-285), every Alg. 1 branch."""
    n = 200_000
    p, emax, emin = _gen.FMT[dt]
    a = _gen.positive(dt, 0x57D20007, n, emin, emax - 2, 0)
    b = _gen.positive(dt, 0x57D20007, n, emin, emax - 2, 1)
    c = _gen.positive(dt, 0x57D20007, n, emin, emax - 2, 2)
    a, c = np.maximum(a, c), np.minimum(a, c)
    fi = np.finfo(dt)
    mu, nu = dt(fi.tiny), dt(fi.max)
    special = [(1, 1, 1), (2, 1, 1), (4, 3, 2), (mu, 1, mu * dt(0.5)), (2 * mu, nu / 2, mu), (2, fi.smallest_subnormal, 1)]
    for i, (x, y, z) in enumerate(special):
        a[i], b[i], c[i] = x, y, z
    a, b, c = a.astype(dt), b.astype(dt), c.astype(dt)
    t13 = (np.arange(n) % 2).astype(np.uint8)
    got = K.tri_svd(dev(a), dev(b), dev(c), dev(t13), K_opt(opt))
    rt = capi.kog_trisvd_f64 if dt == np.float64 else capi.kog_trisvd_f32
    want = refbind.records(rt, n)
    (ref.tri_svd_f64 if dt == np.float64 else ref.tri_svd_f32)(a.ctypes.data, b.ctypes.data, c.ctypes.data,
                                                               t13.ctypes.data, C.addressof(want), n, C.byref(opt))
    records_equal(got, want, "tri_svd")


@pytest.mark.parametrize("dt", DTS)
def test_compose_left_and_triangularize13(cuda, ref, dt):
    """compose_left (svd2_test.cpp:287-327) and triangularize13 (123-154)."""
    n = 200_000
    tp = (_gen.unit(_gen.draws(1, n, 0)) * 2).astype(dt)
    tt = _gen.unit(_gen.draws(1, n, 1)).astype(dt)
    tp[:4] = [np.inf, np.inf, 0, 1]
    tt[:4] = [1, 1, 0.75, 1]
    m = (np.arange(n) % 2).astype(np.uint8)
    gc, gs = K.compose_left(dev(tp), dev(tt), dev(m))
    wc, ws = np.empty_like(tp), np.empty_like(tp)
    (ref.compose_left_f64 if dt == np.float64 else ref.compose_left_f32)(tp.ctypes.data, tt.ctypes.data,
                                                                         m.ctypes.data, wc.ctypes.data,
                                                                         ws.ctypes.data, n)
    _gen.assert_bits_equal(host(gc), wc, "compose c")
    _gen.assert_bits_equal(host(gs), ws, "compose s")
    types = np.array([7, 11, 13, 14], dtype=np.uint8)[(_gen.draws(2, n, 0) % np.uint64(4)).astype(np.int64)]
    g = np.ascontiguousarray(np.stack([_gen.stratified(dt, 0x57D20002, n, -40, 40, k) for k in range(4)]))
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][(types & bit) == 0] = 0
    r, up, vp = K.triangularize13(dev(g), dev(types))
    wr = np.empty_like(g)
    wup, wvp = np.empty((n, 4), np.int8), np.empty((n, 4), np.int8)
    (ref.triangularize13_f64 if dt == np.float64 else ref.triangularize13_f32)(
        C.byref(refbind.mat(g)), types.ctypes.data, C.byref(refbind.mat(wr)), wup.ctypes.data, wvp.ctypes.data, n)
    _gen.assert_bits_equal(host(r).ravel(), wr.ravel(), "tri13 R")
    assert (host(up) == wup).all() and (host(vp) == wvp).all()


# --------------------------------------------------------------- svd2
@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("opt", ALL_OPTIONS, ids=lambda o: f"cr{o.hypot_is_cr}om{o.ominus_for_d}w{o.wide_channel}")
def test_svd2_any_finite_all_options(cuda, ref, dt, opt):
    """svd2 on any-finite matrices with every Options combination
    (svd2_test.cpp:329-359, acceptance.cpp:518-561 totality fuzz)."""
    n = 1 << 18
    g = _gen.matrices(dt, 0x57D20004, n)
    mask = (_gen.draws(11, n, 0) % np.uint64(16)).astype(np.int64)
    sel = (_gen.draws(11, n, 1) % np.uint64(4)) == 0
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][sel & ((mask & bit) == 0)] = 0
    got = K.svd2(dev(g), K_opt(opt))
    want = refbind.svd2(ref, g, opt)
    compare_svd(got, want, "svd2")


def test_svd2_f32_secant_boundary(cuda, ref):
    """binary32 svd2 whose tan(theta) = |g21| / |g11| lies in [2^-14, 2^-11]:
    the fast path's sec_le1<float> (kog2_fast.cuh) returns 1 below 2^-12
    and takes the root above; every field equals the reference's."""
    n = 1 << 18
    rng = np.random.default_rng(0x5EC1)
    sgn = lambda: np.where(rng.random(n) < 0.5, -1.0, 1.0)
    g11 = sgn() * (1 + rng.random(n)) * np.exp2(rng.integers(-4, 5, n))
    g21 = sgn() * np.abs(g11) * np.exp2(rng.uniform(-14, -11, n))
    g12 = sgn() * (1 + rng.random(n)) * np.exp2(rng.integers(-9, -4, n)) * np.abs(g11)
    g22 = sgn() * (1 + rng.random(n)) * np.exp2(rng.integers(-9, -4, n)) * np.abs(g11)
    g = np.ascontiguousarray(np.stack([g11, g12, g21, g22]).astype(np.float32))
    compare_svd(K.svd2(dev(g)), refbind.svd2(ref, g), "f32 secant boundary")


TARGETED = [  # harness_test.cpp:181-193 + svd2_test.cpp known answers
    (1, 1, 0, 1), (2, 1, 0, 1), (4, 3, 0, 2), (1, 3, 0, 4), (2, 0, 0, 1), (3, 0, 4, 0), (1, 1, 0, 0),
    (1, 1, 1, -1), (2, 4, 1, 2), (0, 3, 2, 0), (-5, 0, 0, 0), (2, 1, 1, 2), (0, 2, 0, 1), (0, 0, 0, 0),
]


@pytest.mark.parametrize("dt", DTS)
def test_svd2_targeted(cuda, ref, dt):
    fi = np.finfo(dt)
    mu, nu, mc = fi.tiny, fi.max, fi.smallest_subnormal
    rows = list(TARGETED) + [(mu, 1, 0, mu / 2), (mu, nu / 4, 0, mu), (mu, 1, 0, 1), (mc, -mc, 3 * mc, 2 * mc),
                             (nu, mc, mc, mc), (nu, 1, 1, 1)]
    g = np.ascontiguousarray(np.array(rows, dtype=dt).T)
    for o in ALL_OPTIONS:
        compare_svd(K.svd2(dev(g), K_opt(o)), refbind.svd2(ref, g, o), "targeted")
    r = K.svd2(dev(g))
    path = (host(r["flags"]).view(np.uint32) >> capi.F_PATH_SHIFT) & 7
    assert set(path.tolist()) >= {0, 1, 2, 3, 4, 5, 6}


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_svd2_baseline_configs(cuda, ref, k):
    """BASELINE configs 1-4: on-device generator == host generator and svd2
    bit-exact on 2^20 matrices of each distribution."""
    cfg = configs.cfg(k, count=1 << 20)
    g_dev = K.generate(cfg, 0, cfg.count)
    g_ref = refbind.generate(ref, cfg.c(), 0, cfg.count)
    _gen.assert_bits_equal(host(g_dev).ravel(), g_ref.ravel(), f"cfg{k} generate")
    compare_svd(K.svd2(g_dev), refbind.svd2(ref, g_ref), f"cfg{k} svd2")
    # a later index window (cfg5 sharding: index offsets must reproduce)
    off = 123_456_789
    g2 = K.generate(cfg, off, 4096)
    _gen.assert_bits_equal(host(g2).ravel(), refbind.generate(ref, cfg.c(), off, 4096).ravel(), "offset window")


@pytest.mark.parametrize("k,count", [(3, 1 << 28), (4, 1 << 28), (2, 1 << 26)])
def test_svd2_full_size_sampled(cuda, ref, k, count):
    """BASELINE configs at their full sizes (the bench workloads): one svd2 call
    over the whole on-device batch, then bit-exact parity on 64 seeded windows
    of 4096 matrices (the counter-based generator reproduces any window on the
    host), plus size-independent properties over every matrix: no domain
    errors, sigma1 >= sigma2 >= 0 as pairs, and |u11|^2 + |u12|^2 = 1 to
    working accuracy."""
    cfg = configs.cfg(k, count=count)
    g = K.generate(cfg, 0, count)
    r = K.svd2(g)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0xF0115)
    W = 4096
    offs = sorted(rng.integers(0, count - W, 64).tolist()) + [0, count - W]
    for off in offs:
        gw = refbind.generate(ref, cfg.c(), off, W)
        want = refbind.svd2(ref, gw)
        got = {key: v[off:off + W] for key, v in r.items()}
        compare_svd(got, want, f"cfg{k} window {off}")
    assert capi.F_DOMAIN_ERROR == 1 << 31
    assert int((r["flags"].view(torch.int32) < 0).sum()) == 0  # the domain-error bit is the sign bit
    e1, e2 = r["sig1_e"].long(), r["sig2_e"].long()
    f1, f2 = r["sig1_f"].double(), r["sig2_f"].double()
    assert bool((f2 >= 0).all()) and bool((f1 >= 0).all())
    z2 = f2 == 0
    assert bool((z2 | (e1 > e2) | ((e1 == e2) & (f1 >= f2))).all()), "sigma1 < sigma2"
    u11, u12 = r["u11"].double(), r["u12"].double()
    eps = 4 * float(np.finfo(np.float32 if k == 4 else np.float64).eps)
    assert float((u11 * u11 + u12 * u12 - 1).abs().max()) < eps
    del g, r
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dt", DTS)
def test_svd2_host_pipeline(cuda, ref, dt):
    """kog_svd2_host_*: host buffers through the chunked H2D/kernel/D2H pipeline."""
    n = (1 << 22) * 2 + 12345  # several chunks and a ragged tail
    g = _gen.matrices(dt, 0x51D, n)
    gt = torch.from_numpy(g).pin_memory()
    got = K.svd2_host(gt)
    want = refbind.svd2(ref, g)
    compare_svd({k: v.numpy() for k, v in got.items()}, want, "svd2_host")


def test_empty_and_null(cuda):
    g = torch.empty((4, 0), dtype=torch.float64, device="cuda")
    r = K.svd2(g)
    assert r["flags"].numel() == 0
    with pytest.raises(capi.KogError):
        capi.check(capi.load().kog_svd2_batch_f64(None, None, 1, None, None))


# ------------------------------------------------------ oracle + metrics
@pytest.mark.parametrize("dt", DTS)
def test_svd2_ext_and_metrics(cuda, ref, dt):
    """svd2_ext and the error measures, bit-exact (oracle_test.cpp surfaces)."""
    n = 1 << 16
    g = _gen.matrices(dt, 0xE1F00003, n)
    mask = (_gen.draws(5, n, 0) % np.uint64(16)).astype(np.int64)
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][(mask & bit) == 0] = 0
    got = K.svd2_ext(dev(g))
    want = refbind.records(capi.kog_extsvd, n)
    (ref.svd2_ext_f64 if dt == np.float64 else ref.svd2_ext_f32)(C.byref(refbind.mat(g)), C.addressof(want), n)
    records_equal(got, want, "svd2_ext")
    gm = K.metrics(dev(g))
    wm = refbind.records(capi.kog_metrics, n)
    (ref.metrics_f64 if dt == np.float64 else ref.metrics_f32)(C.byref(refbind.mat(g)), C.addressof(wm), n,
                                                               C.byref(capi.default_options()), 0)
    gb = np.frombuffer(bytes(gm), dtype=np.uint8).reshape(n, -1)
    wb = np.frombuffer(bytes(wm), dtype=np.uint8).reshape(n, -1)
    bad = np.nonzero((gb != wb).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} metric records differ; first {bad[0]}: {g[:, bad[0]]}"


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_metrics_records_on_configs(cuda, ref, k):
    """Per-matrix error measures (svd2 -> svd2_ext -> metrics, the inline Xf
    arithmetic on finite data) bit-exact against the reference's metrics() on
    each BASELINE config's generated matrices (the study's own inputs)."""
    n = 1 << 15
    cfg = configs.cfg(k, count=n)
    off = 0 if k < 5 else (1 << 28) + 12345  # config 5: an index window past config 3's range
    g = refbind.generate(ref, cfg.c(), off, n)
    gm = K.metrics(dev(g))
    wm = refbind.records(capi.kog_metrics, n)
    (ref.metrics_f64 if g.dtype == np.float64 else ref.metrics_f32)(C.byref(refbind.mat(g)), C.addressof(wm), n,
                                                                    C.byref(capi.default_options()), 0)
    gb = np.frombuffer(bytes(gm), dtype=np.uint8).reshape(n, -1)
    wb = np.frombuffer(bytes(wm), dtype=np.uint8).reshape(n, -1)
    bad = np.nonzero((gb != wb).any(axis=1))[0]
    assert bad.size == 0, f"config {k}: {bad.size} metric records differ; first {bad[0]}: {g[:, bad[0]]}"


# ----------------------------------------------------------- harness
APPENDIX_B = [  # reference CSV rows captured in the survey container
    "double,gen,circ,0,1048576,0000000000c0ffee,kog,5.262556799095865e-16,4.469753940626907e-16,5.475477442600766e-16,4.740088882553483e-16,4.726642799363624e-16,14512464.951216837",
    "double,tri,bullet,0,1048576,00000000000005b1,kog,3.6629159219119507e-16,3.1751026529124164e-16,3.3703653551936313e-16,4.657287832316551e-16,4.700986429951113e-16,2.9702909105091426e+1218",
    "double,gen,bullet,0,1048576,00000000feedbeef,kog,3.366846414194082e-16,3.805030544364915e-16,1,4.689522663061862e-16,4.658513990744075e-16,1.5833298576379424e+615",
    "double,gen,sigma,1024,1048576,000000000f1e2d3c,kog,3.5758175247668104e-16,3.579491957323541e-16,4.550667095394166e-16,4.646732779855881e-16,4.61552054390659e-16,3.8630772656508938e+306",
    "single,gen,circ,0,1048576,0000000000c0ffee,kog,2.8583080828580647e-07,2.3807519202657365e-07,3.222986020883533e-07,2.534061500807315e-07,2.5379602539148014e-07,12409701.427193983",
]


def _cfg_of_row(row: str) -> K.RunConfig:
    f = row.split(",")
    return K.RunConfig(single_precision=f[0] == "single", shape=capi.SHAPE_TRI if f[1] == "tri" else capi.SHAPE_GEN,
                       regime={"circ": 0, "bullet": 1, "sigma": 2}[f[2]], varsigma=int(f[3]), count=int(f[4]),
                       seed=int(f[5], 16), routine=capi.ROUTINE_KOG)


@pytest.mark.parametrize("row", APPENDIX_B, ids=lambda r: ",".join(r.split(",")[:3]))
def test_run_batch_csv_matches_reference_rows(cuda, row):
    """GPU-backed run_batch + csv_row byte-identical to the reference's rows."""
    cfg = _cfg_of_row(row)
    st = K.run_batch(cfg)
    assert K.csv_row(cfg, st) == row


def test_run_batch_vs_reference_counts(cuda, ref):
    """ErrorStats incl. all 19 BranchCounts equal the reference's run_batch
    (harness.hpp:226-271) on the branch-coverage batch of harness_test.cpp:164-217."""
    wants = {}
    for cfg in (K.RunConfig(shape=capi.SHAPE_GEN, regime=capi.REGIME_BULLET, count=1 << 18, seed=77),
                K.RunConfig(shape=capi.SHAPE_TRI, regime=capi.REGIME_CIRC, count=1 << 18, seed=78),
                K.RunConfig(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=50000, seed=0x1234ABCD,
                            routine=capi.ROUTINE_LASV2),
                configs.cfg(3, count=1 << 18), configs.cfg(4, count=1 << 18), configs.cfg(2, count=1 << 18),
                # more than one chunk of the phased study (chunks of 2^20 here)
                (configs.cfg(5, count=(1 << 20) + 4099), 20),
                # four chunks: both chunk buffers reused by the producer/consumer pipeline, a 5-matrix tail
                (configs.cfg(5, count=3 * (1 << 22) + 5), 22),
                # the same at the default chunk (one chunk: the two-speed svd2 kernel inside the study)
                (configs.cfg(5, count=3 * (1 << 22) + 5), None),
                # non-default Options: the general svd2 kernel inside the study
                K.RunConfig(shape=capi.SHAPE_GEN, regime=capi.REGIME_BULLET, count=1 << 17, seed=79,
                            options=K.Options(hypot_is_cr=False, ominus_for_d=True)),
                K.RunConfig(single_precision=True, shape=capi.SHAPE_GEN, regime=capi.REGIME_BULLET, count=1 << 17,
                            seed=80, options=K.Options(hypot_is_cr=False))):
        cfg, chunk = cfg if isinstance(cfg, tuple) else (cfg, None)
        if chunk is None:
            st = K.run_batch(cfg)
        else:
            with _gen.study_chunk(chunk):
                st = K.run_batch(cfg)
        key = bytes(cfg.c())
        if key not in wants:  # (the reference's run_batch over 12.6 million matrices once)
            rc, want, msg = refbind.run_batch(ref, cfg.c())
            assert rc == 0, msg
            wants[key] = want
        want = wants[key]
        got_row, want_row = K.csv_row(cfg, st).split(","), refbind.csv_row(ref, cfg.c(), want).split(",")
        if cfg.regime == capi.REGIME_RANGED:  # the reference's csv_row has no name for the extension
            got_row[2] = want_row[2]
        assert got_row == want_row
        for f in ("t2p", "path"):
            assert list(getattr(st, f)) == list(getattr(want, f)), f
        for f in ("tanpsi_inf", "diag_swap", "compose_minus", "sigma_swap", "prescale_inexact", "kappa_inf"):
            assert getattr(st, f) == getattr(want, f), f
        assert (st.max_kappa2.e, st.max_kappa2.hi, st.max_kappa2.lo) == \
               (want.max_kappa2.e, want.max_kappa2.hi, want.max_kappa2.lo)


def test_run_batch_validation_and_empty(cuda):
    """harness_test.cpp:63-86."""
    st = K.run_batch(K.RunConfig(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=0, seed=1))
    assert (st.reG, st.reS1, st.reS2, st.reU, st.reV) == (0, 0, 0, 0, 0) and st.max_kappa2.hi == 0
    with pytest.raises(ValueError):
        K.run_batch(K.RunConfig(shape=capi.SHAPE_GEN, routine=capi.ROUTINE_LASV2, count=10))
    with pytest.raises(ValueError):
        K.run_batch(K.RunConfig(regime=capi.REGIME_SIGMA, varsigma=0, count=10))
    with pytest.raises(ValueError):
        K.run_batch(K.RunConfig(regime=capi.REGIME_SIGMA, varsigma=5000, count=10))


def test_study_split_equals_fused(cuda):
    """The split study (seven instruction-cache-sized launches per chunk, the default) and the fused k_study
    (KOG2_STUDY_SPLIT=0, read once at load: a second interpreter) give the same bytes of ErrorStats — binary64
    and binary32, several chunks, zero patterns and non-default Options included."""
    import os
    import subprocess
    import sys
    code = (
        "import sys\n"
        "from paper_2407_13116_b200 import capi, configs\n"
        "from paper_2407_13116_b200 import kogsvd2 as K\n"
        "capi.load().kog_study_set_chunk_log2(20)\n"
        "cfgs = [configs.cfg(5, count=3 * (1 << 20) + 77), configs.cfg(4, count=(1 << 20) + 5), configs.cfg(2, count=1 << 18),\n"
        "        K.RunConfig(shape=capi.SHAPE_GEN, regime=capi.REGIME_BULLET, count=1 << 17, seed=79,\n"
        "                    options=K.Options(hypot_is_cr=False, ominus_for_d=True))]\n"
        "for c in cfgs:\n"
        "    s = K.StudyStats(); s.add(c, 0, c.count); print(bytes(s.read()).hex())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    # (and the pipeline's stream modes: everything on the caller's stream, one consumer stream, two)
    for split, streams in (("1", "1"), ("0", "1"), ("1", "0"), ("1", "2")):
        env = dict(os.environ, KOG2_STUDY_SPLIT=split, KOG2_STUDY_STREAMS=streams, PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=root, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.split())
    assert len(outs[0]) == 4 and all(o == outs[0] for o in outs[1:])


def test_study_sharding_bit_identical(cuda):
    """cfg5 sharding: any split of the index range merges to the same stats."""
    cfg = configs.cfg(5, count=3 * (1 << 16) + 77)
    whole = K.StudyStats()
    whole.add(cfg, 0, cfg.count)
    a = whole.read()
    cuts = [0, 1000, 70000, 150000, cfg.count]
    merged = K.new_stats()
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        s = K.StudyStats()
        s.add(cfg, lo, hi - lo)
        K.merge_stats(merged, s.read())
    assert bytes(merged) == bytes(a)


@pytest.mark.parametrize("dt", DTS)
def test_lasv2(cuda, ref, dt):
    """lasv2_ref on triangular triples (lasv2_test.cpp surfaces)."""
    n = 200_000
    p, emax, emin = _gen.FMT[dt]
    f = _gen.stratified(dt, 0x1A5, n, emin, emax - 2, 0)
    g = _gen.stratified(dt, 0x1A5, n, emin, emax - 2, 1)
    h = _gen.stratified(dt, 0x1A5, n, emin, emax - 2, 2)
    g[::7] = 0
    got = host(K.lasv2(dev(f), dev(g), dev(h)))
    want = np.empty((n, 6), dtype=dt)
    (ref.lasv2_f64 if dt == np.float64 else ref.lasv2_f32)(f.ctypes.data, g.ctypes.data, h.ctypes.data,
                                                           want.ctypes.data, n)
    _gen.assert_bits_equal(got.ravel(), want.ravel(), "lasv2")
