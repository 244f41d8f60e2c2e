"""CPU: the C restatement (oracle/_build/libkog_oracle.so) pinned against the
reference compiled in place (oracle/_ref/libkogref.so) and the exact integer
hypot, bit for bit.  Runs without a GPU (`-m "not gpu"`)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle import refbind
from paper_2407_13116_b200 import capi
from tests import _gen

DTS = [np.float64, np.float32]
SUF = {np.float64: "f64", np.float32: "f32"}
ALL_OPTIONS = [capi.kog_options(h, o, w, 0) for h in (1, 0) for o in (0, 1) for w in (0, 1)]


def fn(lib, name, dt):
    return getattr(lib, f"{name}_{SUF[dt]}")


def both_svd(ref, ora, g, opt=None):
    return refbind.svd2(ref, g, opt, threads=0), refbind.svd2(ora, g, opt, threads=0)


def assert_svd_equal(a, b, what):
    for k in refbind.OUT_DTYPES:
        _gen.assert_bits_equal(a[k], b[k], f"{what}.{k}")


@pytest.mark.parametrize("dt", DTS)
def test_hypot_oracle_vs_reference_vs_exact(ref, ora, dt):
    n = 200_000
    a = _gen.any_finite(dt, 0x68790001, n, 0)
    b = _gen.any_finite(dt, 0x68790001, n, 1)
    w, o = np.empty_like(a), np.empty_like(a)
    fn(ref, "hypot", dt)(a.ctypes.data, b.ctypes.data, w.ctypes.data, n)
    fn(ora, "hypot", dt)(a.ctypes.data, b.ctypes.data, o.ctypes.data, n)
    _gen.assert_bits_equal(o, w, "oracle hypot vs reference")
    ex = np.array([_gen.hypot_exact(x, y, dt) for x, y in zip(a[:5000], b[:5000])], dtype=dt)
    _gen.assert_bits_equal(w[:5000], ex, "reference hypot vs exact integer")


@pytest.mark.parametrize("dt", DTS)
def test_unit_routines_oracle_vs_reference(ref, ora, dt):
    n = 50_000
    p, emax, emin = _gen.FMT[dt]
    x = _gen.any_finite(dt, 0x68790005, n)
    for name in ("tan2", "sec"):
        w, o = np.empty_like(x), np.empty_like(x)
        fn(ref, name, dt)(x.ctypes.data, w.ctypes.data, n)
        fn(ora, name, dt)(x.ctypes.data, o.ctypes.data, n)
        _gen.assert_bits_equal(o, w, name)
    we, wf, oe, of = np.empty(n, np.int64), np.empty_like(x), np.empty(n, np.int64), np.empty_like(x)
    fn(ref, "split", dt)(x.ctypes.data, we.ctypes.data, wf.ctypes.data, n)
    fn(ora, "split", dt)(x.ctypes.data, oe.ctypes.data, of.ctypes.data, n)
    assert (we == oe).all()
    _gen.assert_bits_equal(of, wf, "split")
    ee = (np.arange(n, dtype=np.int64) % 4000) - 2000
    fn(ref, "assemble", dt)(ee.ctypes.data, wf.ctypes.data, we.ctypes.data, n)
    fn(ora, "assemble", dt)(ee.ctypes.data, wf.ctypes.data, oe.ctypes.data, n)
    _gen.assert_bits_equal(oe.view(dt)[:n] if False else oe, we, "assemble")
    # EPair ops
    xp = _gen.positive(dt, 0x45500002, n, emin - p + 1, emax, 0)
    yp = _gen.positive(dt, 0x45500002, n, emin - p + 1, emax, 1)
    yp[::97] = xp[::97]
    ex = ((np.arange(n) * 7919) % 2001 - 1000).astype(np.int64)
    ey = ((np.arange(n) * 104729) % 2001 - 1000).astype(np.int64)
    for op in range(7):
        res = []
        for lib in (ref, ora):
            oe, of, st = np.empty(n, np.int64), np.empty_like(xp), np.empty(n, np.uint8)
            fn(lib, "epair", dt)(op, ex.ctypes.data, xp.ctypes.data, ey.ctypes.data, yp.ctypes.data, oe.ctypes.data,
                                 of.ctypes.data, st.ctypes.data, n)
            res.append((oe, of, st))
        assert (res[0][2] == res[1][2]).all()
        ok = res[0][2] == 0
        assert (res[0][0][ok] == res[1][0][ok]).all()
        _gen.assert_bits_equal(res[1][1][ok], res[0][1][ok], f"epair op {op}")


@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("opt", ALL_OPTIONS, ids=lambda o: f"cr{o.hypot_is_cr}om{o.ominus_for_d}w{o.wide_channel}")
def test_svd2_oracle_vs_reference(ref, ora, dt, opt):
    n = 1 << 15
    g = _gen.matrices(dt, 0x57D20004, n)
    mask = (_gen.draws(11, n, 0) % np.uint64(16)).astype(np.int64)
    sel = (_gen.draws(11, n, 1) % np.uint64(4)) == 0
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][sel & ((mask & bit) == 0)] = 0
    w, o = both_svd(ref, ora, g, opt)
    assert_svd_equal(o, w, "svd2")


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_generator_and_svd2_configs(ref, ora, k):
    from paper_2407_13116_b200 import configs

    cfg = configs.cfg(k, count=1 << 15).c()
    gw = refbind.generate(ref, cfg, 1000, cfg.count)
    go = refbind.generate(ora, cfg, 1000, cfg.count)
    _gen.assert_bits_equal(go.ravel(), gw.ravel(), "generate")
    w, o = both_svd(ref, ora, gw)
    assert_svd_equal(o, w, f"cfg{k}")


@pytest.mark.parametrize("dt", DTS)
def test_phases_oracle_vs_reference(ref, ora, dt):
    n = 30_000
    p, emax, emin = _gen.FMT[dt]
    g = np.ascontiguousarray(np.stack([_gen.stratified(dt, 0x57D20006, n, emin, emax - 2, k) for k in range(4)]))
    for wide in (0, 1):
        opt = capi.kog_options(1, 0, wide, 0)
        rt = capi.kog_urv15_f64 if dt == np.float64 else capi.kog_urv15_f32
        a, b = refbind.records(rt, n), refbind.records(rt, n)
        fn(ref, "urv15", dt)(C.byref(refbind.mat(g)), C.addressof(a), n, C.byref(opt))
        fn(ora, "urv15", dt)(C.byref(refbind.mat(g)), C.addressof(b), n, C.byref(opt))
        assert bytes(a) == bytes(b)
    r11 = np.maximum(np.abs(g[0]), np.abs(g[3]))
    r22 = np.minimum(np.abs(g[0]), np.abs(g[3]))
    r12 = np.abs(g[1])
    t13 = (np.arange(n) % 2).astype(np.uint8)
    rt = capi.kog_trisvd_f64 if dt == np.float64 else capi.kog_trisvd_f32
    for opt in ALL_OPTIONS[:4] + ALL_OPTIONS[4:5]:
        a, b = refbind.records(rt, n), refbind.records(rt, n)
        for lib, rec in ((ref, a), (ora, b)):
            fn(lib, "tri_svd", dt)(r11.ctypes.data, r12.ctypes.data, r22.ctypes.data, t13.ctypes.data,
                                   C.addressof(rec), n, C.byref(opt))
        assert bytes(a) == bytes(b)


@pytest.mark.parametrize("dt", DTS)
def test_ext_metrics_lasv2_oracle_vs_reference(ref, ora, dt):
    n = 1 << 13
    g = _gen.matrices(dt, 0xE1F00003, n)
    mask = (_gen.draws(5, n, 0) % np.uint64(16)).astype(np.int64)
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][(mask & bit) == 0] = 0
    a, b = refbind.records(capi.kog_extsvd, n), refbind.records(capi.kog_extsvd, n)
    fn(ref, "svd2_ext", dt)(C.byref(refbind.mat(g)), C.addressof(a), n)
    fn(ora, "svd2_ext", dt)(C.byref(refbind.mat(g)), C.addressof(b), n)
    assert bytes(a) == bytes(b)
    a, b = refbind.records(capi.kog_metrics, n), refbind.records(capi.kog_metrics, n)
    fn(ref, "metrics", dt)(C.byref(refbind.mat(g)), C.addressof(a), n, C.byref(capi.default_options()), 0)
    fn(ora, "metrics", dt)(C.byref(refbind.mat(g)), C.addressof(b), n, C.byref(capi.default_options()), 0)
    assert bytes(a) == bytes(b)
    f, gg, h = g[0].copy(), g[1].copy(), g[3].copy()
    wa, wb = np.empty((n, 6), dt), np.empty((n, 6), dt)
    fn(ref, "lasv2", dt)(f.ctypes.data, gg.ctypes.data, h.ctypes.data, wa.ctypes.data, n)
    fn(ora, "lasv2", dt)(f.ctypes.data, gg.ctypes.data, h.ctypes.data, wb.ctypes.data, n)
    _gen.assert_bits_equal(wb.ravel(), wa.ravel(), "lasv2")


def _rc(**kw) -> capi.kog_run_config:
    c = capi.kog_run_config()
    c.options = capi.default_options()
    c.threads = 0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@pytest.mark.parametrize("cfg", [
    dict(shape=capi.SHAPE_GEN, regime=capi.REGIME_CIRC, count=60000, seed=0xC0FFEE),
    dict(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=50000, seed=0x1234ABCD),
    dict(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=50000, seed=0x1234ABCD, routine=capi.ROUTINE_LASV2),
    dict(shape=capi.SHAPE_GEN, regime=capi.REGIME_SIGMA, varsigma=1024, count=30000, seed=0x0F1E2D3C),
    dict(single_precision=1, shape=capi.SHAPE_GEN, regime=capi.REGIME_CIRC, count=30000, seed=0xC0FFEE),
    dict(shape=capi.SHAPE_GEN, regime=capi.REGIME_RANGED, count=30000, seed=0x0F1E2D3C, elo=-500, ehi=500,
         zero_mask_rule=1),
    dict(single_precision=1, shape=capi.SHAPE_GEN, regime=capi.REGIME_RANGED, count=30000, seed=0xF32, elo=-60,
         ehi=60, tail_lo=-126, tail_hi=-100, tail_mod=100),
], ids=lambda d: f"{d.get('regime')}-{d.get('shape')}-{d.get('routine', 0)}-{d.get('single_precision', 0)}")
def test_run_batch_oracle_vs_reference(ref, ora, cfg):
    c = _rc(**cfg)
    rw, sw, _ = refbind.run_batch(ref, c)
    ro, so, _ = refbind.run_batch(ora, c)
    assert rw == ro == 0
    assert bytes(sw) == bytes(so)
    assert refbind.csv_row(ora, c, so) == refbind.csv_row(ref, c, sw)


def test_run_batch_validation(ora):
    assert refbind.run_batch(ora, _rc(shape=capi.SHAPE_GEN, routine=capi.ROUTINE_LASV2, count=10))[0] == -1
    assert refbind.run_batch(ora, _rc(regime=capi.REGIME_SIGMA, varsigma=0, count=10))[0] == -1
    assert refbind.run_batch(ora, _rc(regime=capi.REGIME_SIGMA, varsigma=5000, count=10))[0] == -1
    rc, st, _ = refbind.run_batch(ora, _rc(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=0, seed=1))
    assert rc == 0 and st.reG == 0 and st.max_kappa2.hi == 0
