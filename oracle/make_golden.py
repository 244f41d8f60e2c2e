"""TEST INFRASTRUCTURE ONLY: regenerate tests/golden/golden_v1.npz from the
reference compiled in place (oracle/_ref/libkogref.so, built by `make -C
oracle ref` from /root/reference/proj/include).

Every array is an input batch and the reference's own outputs for it:
  hypot_{f64,f32}_{a,b,out}     any-finite pairs, 3-4-5 midpoint ties, edge grid
  svd2_{f64,f32}_{set}_{g,<field>}  svd2 (compact layout of include/kog2.h) on
                                the first 2048 matrices of BASELINE configs 1-4
                                (on-device generator rule) and on
                                4096 any-finite matrices with zero patterns
  metrics_{f64,f32}_{g,rec}     kog_metrics records (svd2 vs svd2_ext)
  csv_rows                      csv_row of run_batch for 9 configurations
Run:  python oracle/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refbind  # noqa: E402
from paper_2407_13116_b200 import capi, configs  # noqa: E402
from tests import _gen  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")

CSV_CONFIGS = [  # (single, shape, regime, varsigma, count, seed, routine) + extension fields
    dict(shape=1, regime=0, count=1 << 20, seed=0xC0FFEE),
    dict(shape=0, regime=1, count=1 << 20, seed=0x05B1),
    dict(shape=1, regime=1, count=1 << 20, seed=0xFEEDBEEF),
    dict(shape=1, regime=2, varsigma=1024, count=1 << 20, seed=0x0F1E2D3C),
    dict(single_precision=1, shape=1, regime=0, count=1 << 20, seed=0xC0FFEE),
    dict(shape=0, regime=1, count=50000, seed=0x1234ABCD, routine=1),
    dict(shape=0, regime=3, count=1 << 16, seed=0x05B1, elo=-1000, ehi=1000),
    dict(shape=1, regime=3, count=1 << 16, seed=0x0F1E2D3C, elo=-500, ehi=500, zero_mask_rule=1),
    dict(single_precision=1, shape=1, regime=3, count=1 << 16, seed=0xF32, elo=-60, ehi=60, tail_lo=-126,
         tail_hi=-100, tail_mod=100),
]


def run_cfg(d: dict) -> capi.kog_run_config:
    c = capi.kog_run_config()
    c.options = capi.default_options()
    c.threads = 0
    for k, v in d.items():
        setattr(c, k, v)
    return c


def hypot_inputs(dt):
    n = 16384
    a = _gen.any_finite(dt, 0x60D0, n, 0)
    b = _gen.any_finite(dt, 0x60D0, n, 1)
    p = 53 if dt == np.float64 else 24
    rng = np.random.default_rng(7)
    q = rng.integers((1 << p) // 5 + 1, ((1 << (p + 1)) - 1) // 5, size=2048, dtype=np.int64) | 1
    x = rng.integers(-30, 31, size=q.size)
    ta = np.ldexp((3 * q).astype(np.float64), x).astype(dt)
    tb = np.ldexp((4 * q).astype(np.float64), x).astype(dt)
    fi = np.finfo(dt)
    edge = np.array([0, fi.smallest_subnormal, fi.tiny, fi.tiny / 2, 1, 1 + fi.eps, fi.max, fi.max / 2, 3, 4, 0.5],
                    dtype=dt)
    ea, eb = np.meshgrid(np.concatenate([edge, -edge]), np.concatenate([edge, -edge]))
    return (np.concatenate([a, ta, ea.ravel()]).astype(dt), np.concatenate([b, tb, eb.ravel()]).astype(dt))


def main():
    ref = refbind.ref()
    data = {}
    for dt in (np.float64, np.float32):
        suf = "f64" if dt == np.float64 else "f32"
        a, b = hypot_inputs(dt)
        o = np.empty_like(a)
        getattr(ref, f"hypot_{suf}")(a.ctypes.data, b.ctypes.data, o.ctypes.data, a.size)
        data[f"hypot_{suf}_a"], data[f"hypot_{suf}_b"], data[f"hypot_{suf}_out"] = a, b, o
        sets = {}
        for k in ((1, 2, 3) if dt == np.float64 else (4,)):
            sets[f"cfg{k}"] = refbind.generate(ref, configs.cfg(k, count=2048).c(), 0, 2048)
        if dt == np.float32:
            c1 = configs.cfg(1, count=2048)
            c1.single_precision = True
            sets["cfg1"] = refbind.generate(ref, c1.c(), 0, 2048)
        g = _gen.matrices(dt, 0x601D, 4096)
        mask = (_gen.draws(0x601E, 4096, 0) % np.uint64(16)).astype(np.int64)
        sel = (_gen.draws(0x601E, 4096, 1) % np.uint64(3)) == 0
        for kk, bit in enumerate((1, 4, 2, 8)):
            g[kk][sel & ((mask & bit) == 0)] = 0
        sets["any"] = g
        for name, gg in sets.items():
            out = refbind.svd2(ref, gg)
            data[f"svd2_{suf}_{name}_g"] = gg
            for f, v in out.items():
                data[f"svd2_{suf}_{name}_{f}"] = v
        gm = np.ascontiguousarray(g[:, :1024])
        rec = refbind.records(capi.kog_metrics, 1024)
        getattr(ref, f"metrics_{suf}")(C.byref(refbind.mat(gm)), C.addressof(rec), 1024,
                                       C.byref(capi.default_options()), 0)
        data[f"metrics_{suf}_g"] = gm
        data[f"metrics_{suf}_rec"] = np.frombuffer(bytes(rec), dtype=np.uint8).reshape(1024, -1).copy()
    rows = []
    for d in CSV_CONFIGS:
        c = run_cfg(d)
        rc, st, msg = refbind.run_batch(ref, c)
        assert rc == 0, msg
        rows.append(refbind.csv_row(ref, c, st))
    data["csv_rows"] = np.array(rows)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **data)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")
    for r in rows:
        print(r)


if __name__ == "__main__":
    main()
