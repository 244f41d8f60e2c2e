"""Golden fixtures (tests/golden/golden_v1.npz, made by oracle/make_golden.py
from the reference compiled in place) checked against the C oracle on the CPU
and against the CUDA path on the GPU.  These run where /root/reference and
even oracle/_ref are absent."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

from oracle import refbind
from paper_2407_13116_b200 import capi
from tests import _gen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")
APPENDIX_B = [  # SURVEY.md Appendix B, captured independently during the survey
    "double,gen,circ,0,1048576,0000000000c0ffee,kog,5.262556799095865e-16,4.469753940626907e-16,5.475477442600766e-16,4.740088882553483e-16,4.726642799363624e-16,14512464.951216837",
    "single,gen,circ,0,1048576,0000000000c0ffee,kog,2.8583080828580647e-07,2.3807519202657365e-07,3.222986020883533e-07,2.534061500807315e-07,2.5379602539148014e-07,12409701.427193983",
]


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def svd_sets(gold, suf):
    names = sorted({k.split("_")[2] for k in gold.files if k.startswith(f"svd2_{suf}_")})
    return names


def test_golden_contains_the_survey_rows(gold):
    rows = list(gold["csv_rows"])
    for r in APPENDIX_B:
        assert r in rows


@pytest.mark.parametrize("suf", ["f64", "f32"])
def test_oracle_matches_golden(ora, gold, suf):
    dt = np.float64 if suf == "f64" else np.float32
    a, b, want = gold[f"hypot_{suf}_a"], gold[f"hypot_{suf}_b"], gold[f"hypot_{suf}_out"]
    got = np.empty_like(a)
    getattr(ora, f"hypot_{suf}")(a.ctypes.data, b.ctypes.data, got.ctypes.data, a.size)
    _gen.assert_bits_equal(got, want, "oracle hypot vs golden")
    for name in svd_sets(gold, suf):
        g = np.ascontiguousarray(gold[f"svd2_{suf}_{name}_g"])
        out = refbind.svd2(ora, g)
        for f in refbind.OUT_DTYPES:
            _gen.assert_bits_equal(out[f], gold[f"svd2_{suf}_{name}_{f}"], f"oracle svd2 {name}.{f}")
    gm = np.ascontiguousarray(gold[f"metrics_{suf}_g"])
    rec = refbind.records(capi.kog_metrics, gm.shape[1])
    getattr(ora, f"metrics_{suf}")(C.byref(refbind.mat(gm)), C.addressof(rec), gm.shape[1],
                                   C.byref(capi.default_options()), 0)
    assert np.array_equal(np.frombuffer(bytes(rec), np.uint8).reshape(gm.shape[1], -1), gold[f"metrics_{suf}_rec"])
    assert dt  # noqa


def test_oracle_csv_rows_match_golden(ora, gold):
    from oracle.make_golden import CSV_CONFIGS, run_cfg

    for d, want in zip(CSV_CONFIGS, gold["csv_rows"]):
        if d["count"] > 70000:  # the 2^20 rows: 1-2 s each on 8 cores; keep two
            if not (d.get("regime") == 0 and d.get("shape") == 1):
                continue
        c = run_cfg(d)
        rc, st, msg = refbind.run_batch(ora, c)
        assert rc == 0, msg
        assert refbind.csv_row(ora, c, st) == str(want)


@pytest.mark.gpu
@pytest.mark.parametrize("suf", ["f64", "f32"])
def test_cuda_matches_golden(cuda, gold, suf):
    import torch

    from paper_2407_13116_b200 import kogsvd2 as K

    a, b, want = gold[f"hypot_{suf}_a"], gold[f"hypot_{suf}_b"], gold[f"hypot_{suf}_out"]
    got = K.hypot_cr(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    _gen.assert_bits_equal(got, want, "cuda hypot vs golden")
    for name in svd_sets(gold, suf):
        g = torch.from_numpy(np.ascontiguousarray(gold[f"svd2_{suf}_{name}_g"])).cuda()
        out = K.svd2(g)
        for f in refbind.OUT_DTYPES:
            v = out[f].cpu().numpy()
            if f == "flags":
                v = v.view(np.uint32)
            _gen.assert_bits_equal(v, gold[f"svd2_{suf}_{name}_{f}"], f"cuda svd2 {name}.{f}")
    gm = torch.from_numpy(np.ascontiguousarray(gold[f"metrics_{suf}_g"])).cuda()
    rec = K.metrics(gm)
    assert np.array_equal(np.frombuffer(bytes(rec), np.uint8).reshape(gm.shape[1], -1), gold[f"metrics_{suf}_rec"])


@pytest.mark.gpu
def test_cuda_csv_rows_match_golden(cuda, gold):
    from oracle.make_golden import CSV_CONFIGS
    from paper_2407_13116_b200 import kogsvd2 as K

    for d, want in zip(CSV_CONFIGS, gold["csv_rows"]):
        cfg = K.RunConfig(**{k: v for k, v in d.items()})
        assert K.csv_row(cfg, K.run_batch(cfg)) == str(want)
