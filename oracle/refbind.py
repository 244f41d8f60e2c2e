"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the oracles.

  ref()     -> oracle/_ref/libkogref.so   the reference headers compiled in place
  oracle()  -> oracle/_build/libkog_oracle.so   the plain-C restatement

Both expose host-array functions shaped like include/kog2.h (struct layouts
are shared with paper_2407_13116_b200.capi).  Only tests/, smoke() and
bench.py's CPU legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2407_13116_b200 import capi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libkogref.so")
ORACLE_PATH = os.path.join(HERE, "_build", "libkog_oracle.so")

P = C.c_void_p
u64 = C.c_uint64
i32 = C.c_int
PTR = C.POINTER

_COMMON = {
    "hypot_f64": (i32, [P, P, P, u64]),
    "hypot_f32": (i32, [P, P, P, u64]),
    "split_f64": (i32, [P, P, P, u64]),
    "split_f32": (i32, [P, P, P, u64]),
    "assemble_f64": (i32, [P, P, P, u64]),
    "assemble_f32": (i32, [P, P, P, u64]),
    "tan2_f64": (i32, [P, P, u64]),
    "tan2_f32": (i32, [P, P, u64]),
    "sec_f64": (i32, [P, P, u64]),
    "sec_f32": (i32, [P, P, u64]),
    "epair_f64": (i32, [i32, P, P, P, P, P, P, P, u64]),
    "epair_f32": (i32, [i32, P, P, P, P, P, P, P, u64]),
    "classify_prescale_f64": (i32, [PTR(capi.kog_mat), PTR(capi.kog_classify_out), PTR(capi.kog_mat), u64]),
    "classify_prescale_f32": (i32, [PTR(capi.kog_mat), PTR(capi.kog_classify_out), PTR(capi.kog_mat), u64]),
    "urv15_f64": (i32, [PTR(capi.kog_mat), P, u64, PTR(capi.kog_options)]),
    "urv15_f32": (i32, [PTR(capi.kog_mat), P, u64, PTR(capi.kog_options)]),
    "tri_svd_f64": (i32, [P, P, P, P, P, u64, PTR(capi.kog_options)]),
    "tri_svd_f32": (i32, [P, P, P, P, P, u64, PTR(capi.kog_options)]),
    "compose_left_f64": (i32, [P, P, P, P, P, u64]),
    "compose_left_f32": (i32, [P, P, P, P, P, u64]),
    "triangularize13_f64": (i32, [PTR(capi.kog_mat), P, PTR(capi.kog_mat), P, P, u64]),
    "triangularize13_f32": (i32, [PTR(capi.kog_mat), P, PTR(capi.kog_mat), P, P, u64]),
    "svd2_f64": (i32, [PTR(capi.kog_mat), PTR(capi.kog_svd_out), u64, PTR(capi.kog_options), i32]),
    "svd2_f32": (i32, [PTR(capi.kog_mat), PTR(capi.kog_svd_out), u64, PTR(capi.kog_options), i32]),
    "svd2_ext_f64": (i32, [PTR(capi.kog_mat), P, u64]),
    "svd2_ext_f32": (i32, [PTR(capi.kog_mat), P, u64]),
    "metrics_f64": (i32, [PTR(capi.kog_mat), P, u64, PTR(capi.kog_options), i32]),
    "metrics_f32": (i32, [PTR(capi.kog_mat), P, u64, PTR(capi.kog_options), i32]),
    "generate_f64": (i32, [PTR(capi.kog_run_config), u64, PTR(capi.kog_mat), u64, i32]),
    "generate_f32": (i32, [PTR(capi.kog_run_config), u64, PTR(capi.kog_mat), u64, i32]),
    "run_batch": (i32, [PTR(capi.kog_run_config), PTR(capi.kog_stats)]),
    "run_range": (i32, [PTR(capi.kog_run_config), u64, u64, PTR(capi.kog_stats)]),
    "csv_row": (i32, [PTR(capi.kog_run_config), PTR(capi.kog_stats), C.c_char_p, C.c_size_t]),
    "lasv2_f64": (i32, [P, P, P, P, u64]),
    "lasv2_f32": (i32, [P, P, P, P, u64]),
    "last_error": (C.c_char_p, []),
    "hardware_threads": (C.c_uint, []),
}


class Lib:
    """A loaded oracle library with the common surface (prefix kogref_/kogora_)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in _COMMON.items():
            fn = getattr(self.lib, prefix + name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)


_ref = None
_oracle = None


def ref() -> Lib:
    global _ref
    if _ref is None:
        _ref = Lib(REF_PATH, "kogref_")
    return _ref


def oracle() -> Lib:
    global _oracle
    if _oracle is None:
        _oracle = Lib(ORACLE_PATH, "kogora_")
    return _oracle


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


def have_oracle() -> bool:
    return os.path.exists(ORACLE_PATH)


# ----------------------------------------------------------- numpy helpers
def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def mat(g: np.ndarray) -> capi.kog_mat:
    """(4, n) C-contiguous numpy array -> kog_mat of row pointers."""
    assert g.flags.c_contiguous and g.shape[0] == 4
    return capi.kog_mat(*[g[k].ctypes.data for k in range(4)])


OUT_DTYPES = {"sig1_f": None, "sig2_f": None, "sig1_e": np.int32, "sig2_e": np.int32, "u11": None, "u12": None,
              "v11": None, "v12": None, "s": np.int32, "flags": np.uint32}


def svd2(lib: Lib, g: np.ndarray, opt: capi.kog_options | None = None, threads: int = 0) -> dict:
    n = g.shape[1]
    out = {k: np.empty(n, dtype=(dt or g.dtype)) for k, dt in OUT_DTYPES.items()}
    o = capi.kog_svd_out(*[out[k].ctypes.data for k in OUT_DTYPES])
    fn = lib.svd2_f64 if g.dtype == np.float64 else lib.svd2_f32
    fn(C.byref(mat(g)), C.byref(o), n, C.byref(opt or capi.default_options()), threads)
    return out


def generate(lib: Lib, cfg: capi.kog_run_config, index0: int, n: int, threads: int = 0) -> np.ndarray:
    dt = np.float32 if cfg.single_precision else np.float64
    g = np.empty((4, n), dtype=dt)
    fn = lib.generate_f32 if cfg.single_precision else lib.generate_f64
    fn(C.byref(cfg), index0, C.byref(mat(g)), n, threads)
    return g


def records(ctype, n: int):
    return (ctype * n)()


def run_batch(lib: Lib, cfg: capi.kog_run_config):
    st = capi.kog_stats()
    rc = lib.run_batch(C.byref(cfg), C.byref(st))
    return rc, st, lib.last_error().decode()


def run_range(lib: Lib, cfg: capi.kog_run_config, index0: int, n: int):
    """The reference's run_one over indices [index0, index0 + n): one shard."""
    st = capi.kog_stats()
    rc = lib.run_range(C.byref(cfg), index0, n, C.byref(st))
    return rc, st, lib.last_error().decode()


def csv_row(lib: Lib, cfg: capi.kog_run_config, st: capi.kog_stats) -> str:
    buf = C.create_string_buffer(512)
    lib.csv_row(C.byref(cfg), C.byref(st), buf, 512)
    return buf.value.decode()
