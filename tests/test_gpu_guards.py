"""Guard-zone checks of every C-ABI entry point (the memory-safety part of
SURVEY.md §5; compute-sanitizer is closed on this GPU pool, see
profiles/sanitizer_r2.txt).

Each array an entry point reads or writes sits inside a larger device
allocation whose guard zones (64 KiB before and after) hold a byte pattern.
Every call runs on ragged sizes (1, 31, 33, 4097, 2^16 + 3 matrices) and on
inputs with many deferred lanes; afterwards every guard zone must still hold
its pattern (no out-of-bounds write, tail handling included) and every input
must be unchanged (const-correctness).  Outputs are also compared with a
second, un-guarded call so the guarded pointers (odd 8-byte offsets into the
allocation) do not change results.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2407_13116_b200 import capi, configs
from paper_2407_13116_b200 import kogsvd2 as K
from tests import _gen

pytestmark = pytest.mark.gpu

G = 1 << 16
PAT = 0xA5
SIZES = [1, 31, 33, 4097, (1 << 16) + 3]


class Arena:
    """Device arrays carved out of one allocation with a guard zone around each."""

    def __init__(self):
        self.bufs: list[tuple[torch.Tensor, int, int]] = []
        self.inputs: list[tuple[torch.Tensor, torch.Tensor]] = []

    def array(self, n: int, dtype, init: np.ndarray | None = None) -> torch.Tensor:
        es = torch.empty(0, dtype=dtype).element_size()
        nbytes = max(n * es, 1)
        raw = torch.full((G + nbytes + 8 + G,), PAT, dtype=torch.uint8, device="cuda")
        off = G + 8  # 8-byte aligned, not 256-byte aligned
        view = raw[off:off + n * es].view(dtype)
        if init is not None:
            view.copy_(torch.from_numpy(np.ascontiguousarray(init)).view(dtype).cuda())
            self.inputs.append((view, view.clone()))
        self.bufs.append((raw, off, n * es))
        return view

    def check(self, what: str) -> None:
        torch.cuda.synchronize()
        for raw, off, nb in self.bufs:
            lo, hi = raw[:off], raw[off + nb:]
            assert bool((lo == PAT).all()), f"{what}: write below an array"
            assert bool((hi == PAT).all()), f"{what}: write past the end of an array"
        for view, copy in self.inputs:
            assert torch.equal(view.view(torch.uint8), copy.view(torch.uint8)), f"{what}: an input array changed"


def _st() -> int:
    return torch.cuda.current_stream().cuda_stream


def _inputs(dt, n: int) -> np.ndarray:
    g = _gen.matrices(dt, 0x6A4D + n, n)
    mask = (_gen.draws(0x6A4E, n, 0) % np.uint64(16)).astype(np.int64)
    sel = (_gen.draws(0x6A4E, n, 1) % np.uint64(4)) == 0
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][sel & ((mask & bit) == 0)] = 0
    return g


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", SIZES)
def test_svd2_guards(cuda, dt, n):
    lib = capi.load()
    suf = "f64" if dt == np.float64 else "f32"
    tdt = torch.float64 if dt == np.float64 else torch.float32
    g = _inputs(dt, n)
    for opt in (capi.default_options(), capi.kog_options(0, 1, 1, 0)):
        A = Arena()
        ins = [A.array(n, tdt, g[k]) for k in range(4)]
        outs = {k: A.array(n, torch.int32 if k in ("sig1_e", "sig2_e", "s", "flags") else tdt) for k in K.SVD_FIELDS}
        m = capi.kog_mat(*[t.data_ptr() for t in ins])
        o = capi.kog_svd_out(*[outs[k].data_ptr() for k in K.SVD_FIELDS])
        capi.check(getattr(lib, f"kog_svd2_batch_{suf}")(C.byref(m), C.byref(o), n, C.byref(opt), _st()))
        A.check(f"svd2_{suf} n={n}")
        plain = K.svd2(torch.from_numpy(g).cuda(), K.Options(bool(opt.hypot_is_cr), bool(opt.ominus_for_d),
                                                             int(opt.wide_channel)))
        for k in K.SVD_FIELDS:
            assert torch.equal(outs[k].view(torch.uint8), plain[k].view(torch.uint8)), k


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_unit_routine_guards(cuda, dt):
    lib = capi.load()
    suf = "f64" if dt == np.float64 else "f32"
    tdt = torch.float64 if dt == np.float64 else torch.float32
    for n in SIZES:
        g = _inputs(dt, n)
        A = Arena()
        a, b = A.array(n, tdt, g[0]), A.array(n, tdt, g[1])
        out, out2 = A.array(n, tdt), A.array(n, tdt)
        e64, st8 = A.array(n, torch.int64), A.array(n, torch.uint8)
        capi.check(getattr(lib, f"kog_hypot_batch_{suf}")(a.data_ptr(), b.data_ptr(), out.data_ptr(), n, _st()))
        capi.check(getattr(lib, f"kog_div_batch_{suf}")(a.data_ptr(), b.data_ptr(), out.data_ptr(), n, _st()))
        capi.check(getattr(lib, f"kog_split_batch_{suf}")(a.data_ptr(), e64.data_ptr(), out.data_ptr(), n, _st()))
        ein = A.array(n, torch.int64, (np.arange(n) % 300 - 150).astype(np.int64))
        capi.check(getattr(lib, f"kog_assemble_batch_{suf}")(ein.data_ptr(), a.data_ptr(), out.data_ptr(), n, _st()))
        capi.check(getattr(lib, f"kog_tan_from_double_angle_batch_{suf}")(a.data_ptr(), out.data_ptr(), n, _st()))
        capi.check(getattr(lib, f"kog_sec_from_tan_batch_{suf}")(a.data_ptr(), out.data_ptr(), n, _st()))
        for op in range(7):
            capi.check(getattr(lib, f"kog_epair_batch_{suf}")(op, ein.data_ptr(), a.data_ptr(), ein.data_ptr(),
                                                              b.data_ptr(), e64.data_ptr(), out2.data_ptr(),
                                                              st8.data_ptr(), n, _st()))
        f = A.array(n, tdt, np.abs(g[0]) + 1)
        h = A.array(n, tdt, np.abs(g[3]) + 1)
        o6 = A.array(6 * n, tdt)
        capi.check(getattr(lib, f"kog_lasv2_batch_{suf}")(f.data_ptr(), b.data_ptr(), h.data_ptr(), o6.data_ptr(), n,
                                                          _st()))
        A.check(f"unit routines {suf} n={n}")


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_record_routine_guards(cuda, dt):
    """classify/prescale, urv15, tri_svd, compose_left, triangularize13,
    svd2_ext, metrics, generate: the record outputs and SoA outputs."""
    lib = capi.load()
    suf = "f64" if dt == np.float64 else "f32"
    tdt = torch.float64 if dt == np.float64 else torch.float32
    for n in SIZES[:4]:
        g = _inputs(dt, n)
        A = Arena()
        ins = [A.array(n, tdt, g[k]) for k in range(4)]
        m = capi.kog_mat(*[t.data_ptr() for t in ins])
        gp = [A.array(n, tdt) for _ in range(4)]
        mp = capi.kog_mat(*[t.data_ptr() for t in gp])
        co = capi.kog_classify_out(*(A.array(n, t).data_ptr() for t in (torch.uint8, torch.int32, torch.int64,
                                                                        torch.int64, torch.uint8, torch.uint8)))
        capi.check(getattr(lib, f"kog_classify_prescale_batch_{suf}")(C.byref(m), C.byref(co), C.byref(mp), n, _st()))
        rec = {"f64": (capi.kog_urv15_f64, capi.kog_trisvd_f64), "f32": (capi.kog_urv15_f32, capi.kog_trisvd_f32)}[suf]
        urv = A.array(n * C.sizeof(rec[0]), torch.uint8)
        capi.check(getattr(lib, f"kog_urv15_batch_{suf}")(C.byref(m), urv.data_ptr(), n, None, _st()))
        t13 = A.array(n, torch.uint8, (np.arange(n) % 2).astype(np.uint8))
        pos = [A.array(n, tdt, np.abs(g[k]) + 1) for k in range(3)]
        tri = A.array(n * C.sizeof(rec[1]), torch.uint8)
        capi.check(getattr(lib, f"kog_tri_svd_batch_{suf}")(pos[0].data_ptr(), pos[1].data_ptr(), pos[2].data_ptr(),
                                                            t13.data_ptr(), tri.data_ptr(), n, None, _st()))
        c, s = A.array(n, tdt), A.array(n, tdt)
        capi.check(getattr(lib, f"kog_compose_left_batch_{suf}")(ins[0].data_ptr(), ins[1].data_ptr(),
                                                                 t13.data_ptr(), c.data_ptr(), s.data_ptr(), n,
                                                                 _st()))
        tt = A.array(n, torch.uint8, np.array([13, 14, 7, 11] * n, dtype=np.uint8)[:n])
        r = [A.array(n, tdt) for _ in range(4)]
        mr = capi.kog_mat(*[t.data_ptr() for t in r])
        up, vp = A.array(4 * n, torch.int8), A.array(4 * n, torch.int8)
        capi.check(getattr(lib, f"kog_triangularize13_batch_{suf}")(C.byref(m), tt.data_ptr(), C.byref(mr),
                                                                    up.data_ptr(), vp.data_ptr(), n, _st()))
        ext = A.array(n * C.sizeof(capi.kog_extsvd), torch.uint8)
        capi.check(getattr(lib, f"kog_svd2_ext_batch_{suf}")(C.byref(m), ext.data_ptr(), n, _st()))
        met = A.array(n * C.sizeof(capi.kog_metrics), torch.uint8)
        capi.check(getattr(lib, f"kog_metrics_batch_{suf}")(C.byref(m), met.data_ptr(), n, None, _st()))
        gen = [A.array(n, tdt) for _ in range(4)]
        cfg = configs.cfg(4 if dt == np.float32 else 3, count=n).c()
        capi.check(getattr(lib, f"kog_generate_batch_{suf}")(C.byref(cfg), 12345, C.byref(capi.kog_mat(
            *[t.data_ptr() for t in gen])), n, _st()))
        A.check(f"record routines {suf} n={n}")


def test_study_stats_guard(cuda):
    """kog_study_batch writes exactly one kog_stats."""
    lib = capi.load()
    A = Arena()
    init = capi.kog_stats()
    lib.kog_stats_init(C.byref(init))
    st = A.array(C.sizeof(capi.kog_stats), torch.uint8, np.frombuffer(bytes(init), np.uint8))
    A.inputs.clear()  # it is an in/out argument
    for cfg in (configs.cfg(5, count=(1 << 22) + 5), configs.cfg(4, count=4097)):
        with _gen.study_chunk(22):  # (two chunks)
            capi.check(lib.kog_study_batch(C.byref(cfg.c()), 7, cfg.count, st.data_ptr(), _st()))
    A.check("kog_study_batch")
