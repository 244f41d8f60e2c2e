"""ctypes mirror of include/kog2.h (the C-ABI of libkog2.so).

Only plumbing lives here: struct layouts, prototypes and the loader.  The
library must exist (built in-tree by paper_2407_13116_b200._build / the repo's
__graft_entry__.build()); there is no fallback when it does not.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KOG2_LIB") or os.path.join(HERE, "lib", "libkog2.so")

# ---------------------------------------------------------------- constants
KOG_OK, KOG_ERR_ARG, KOG_ERR_CUDA, KOG_ERR_NODEV, KOG_ERR_ABORT = 0, -1, -2, -3, -4
KOG_WIDE_WIDER_TYPE, KOG_WIDE_KAHAN_DET = 0, 1

F_SIGN_U21, F_SIGN_U22, F_SIGN_V21, F_SIGN_V22 = 1, 2, 4, 8
F_PATH_SHIFT, F_T2P_SHIFT = 4, 7
F_TANPSI_INF = 1 << 10
F_DIAG_SWAP = 1 << 11
F_SIGMA_SWAP = 1 << 12
F_COMPOSE_MINUS = 1 << 13
F_PRESCALE_INEXACT = 1 << 14
F_URV_COL_SWAP = 1 << 15
F_URV_ROW_SWAP = 1 << 16
F_TYPE_INIT_SHIFT, F_TYPE_SCALED_SHIFT = 17, 21
F_DOMAIN_ERROR = 1 << 31
M_NAN_METRIC = 1 << 30
M_NONFINITE_FACTOR = 1 << 29

PATHS = ["simple", "mono_col", "mono_row", "tri13", "urv15", "urv15_to_diag", "urv15_to_row"]
T2P = ["none", "diag_equal", "offdiag_equal", "small_ratio", "fallback", "general", "general_inf"]

EPAIR_OPLUS, EPAIR_OMINUS, EPAIR_MUL, EPAIR_DIV, EPAIR_LESS, EPAIR_RECIP, EPAIR_MAKE = range(7)
SHAPE_TRI, SHAPE_GEN = 0, 1
REGIME_CIRC, REGIME_BULLET, REGIME_SIGMA, REGIME_RANGED = 0, 1, 2, 3
ROUTINE_KOG, ROUTINE_LASV2 = 0, 1
FAIL_NONFINITE, FAIL_NAN_METRIC = 1, 2

P = C.c_void_p
u64 = C.c_uint64


class kog_options(C.Structure):
    _fields_ = [("hypot_is_cr", C.c_uint8), ("ominus_for_d", C.c_uint8),
                ("wide_channel", C.c_uint8), ("reserved", C.c_uint8)]


class kog_mat(C.Structure):  # kog_mat_f64 / kog_mat_f32: four pointers
    _fields_ = [("g11", P), ("g12", P), ("g21", P), ("g22", P)]


class kog_svd_out(C.Structure):  # kog_svd_out_f64 / _f32
    _fields_ = [("sig1_f", P), ("sig2_f", P), ("sig1_e", P), ("sig2_e", P),
                ("u11", P), ("u12", P), ("v11", P), ("v12", P), ("s", P), ("flags", P)]


class kog_classify_out(C.Structure):
    _fields_ = [("t", P), ("s_type", P), ("s", P), ("e_G", P), ("inexact_underflow", P), ("status", P)]


def _urv_fields(ft):
    return [("gppp", ft * 4), ("tan_theta", ft), ("sec_theta", ft), ("r11", ft), ("r12_raw", ft),
            ("r22_raw", ft), ("r", ft * 4), ("sr0", C.c_int32), ("sr1", C.c_int32), ("s12", C.c_int32),
            ("s22", C.c_int32), ("col_swap", C.c_uint8), ("row_swap", C.c_uint8), ("ext_is_r22", C.c_uint8),
            ("next", C.c_uint8)]


class kog_urv15_f64(C.Structure):
    _fields_ = _urv_fields(C.c_double)


class kog_urv15_f32(C.Structure):
    _fields_ = _urv_fields(C.c_float)


def _tri_fields(ft):
    return [(n, ft) for n in ("tan_phi", "sec_phi", "cos_phi", "sin_phi", "tan_psi", "sec_psi", "cos_psi",
                              "sin_psi", "sig1_f", "sig2_f", "t2f")] + \
           [("sig1_e", C.c_int64), ("sig2_e", C.c_int64), ("sigma_swapped", C.c_uint8),
            ("tanpsi_inf", C.c_uint8), ("t2p", C.c_uint8), ("status", C.c_uint8)]


class kog_trisvd_f64(C.Structure):
    _fields_ = _tri_fields(C.c_double)


class kog_trisvd_f32(C.Structure):
    _fields_ = _tri_fields(C.c_float)


class kog_extfloat(C.Structure):
    _fields_ = [("e", C.c_int64), ("hi", C.c_double), ("lo", C.c_double)]


class kog_extsvd(C.Structure):
    _fields_ = [("sigma1", kog_extfloat), ("sigma2", kog_extfloat), ("u", kog_extfloat * 4),
                ("v", kog_extfloat * 4)]


class kog_metrics(C.Structure):
    _fields_ = [("reG", C.c_double), ("reS1", C.c_double), ("reS2", C.c_double), ("reU", C.c_double),
                ("reV", C.c_double), ("kappa2", kog_extfloat), ("kappa_inf", C.c_uint32), ("flags", C.c_uint32)]


class kog_run_config(C.Structure):
    _fields_ = [("single_precision", C.c_uint8), ("shape", C.c_uint8), ("regime", C.c_uint8),
                ("routine", C.c_uint8), ("varsigma", C.c_int32), ("count", C.c_uint64), ("seed", C.c_uint64),
                ("threads", C.c_int32), ("options", kog_options), ("elo", C.c_int32), ("ehi", C.c_int32),
                ("tail_lo", C.c_int32), ("tail_hi", C.c_int32), ("tail_mod", C.c_uint32),
                ("zero_mask_rule", C.c_uint32)]


class kog_stats(C.Structure):
    _fields_ = [("reG", C.c_double), ("reS1", C.c_double), ("reS2", C.c_double), ("reU", C.c_double),
                ("reV", C.c_double), ("max_kappa2", kog_extfloat), ("max_kappa2_index", C.c_uint64),
                ("kappa_inf", C.c_uint64), ("t2p", C.c_uint64 * 7), ("path", C.c_uint64 * 7),
                ("tanpsi_inf", C.c_uint64), ("diag_swap", C.c_uint64), ("compose_minus", C.c_uint64),
                ("sigma_swap", C.c_uint64), ("prescale_inexact", C.c_uint64), ("fail_key", C.c_uint64)]


assert C.sizeof(kog_stats) == 240, C.sizeof(kog_stats)
assert C.sizeof(kog_metrics) == 72, C.sizeof(kog_metrics)
assert C.sizeof(kog_extsvd) == 240

PTR = C.POINTER
i32 = C.c_int
# name -> (restype, argtypes); every symbol include/kog2.h declares
PROTOTYPES: dict[str, tuple] = {
    "kog_last_error": (C.c_char_p, []),
    "kog_version": (C.c_char_p, []),
    "kog_set_device": (i32, [i32]),
    "kog_svd2_batch_f64": (i32, [PTR(kog_mat), PTR(kog_svd_out), u64, PTR(kog_options), P]),
    "kog_svd2_batch_f32": (i32, [PTR(kog_mat), PTR(kog_svd_out), u64, PTR(kog_options), P]),
    "kog_svd2_host_f64": (i32, [PTR(kog_mat), PTR(kog_svd_out), u64, PTR(kog_options)]),
    "kog_svd2_host_f32": (i32, [PTR(kog_mat), PTR(kog_svd_out), u64, PTR(kog_options)]),
    "kog_hypot_batch_f64": (i32, [P, P, P, u64, P]),
    "kog_hypot_batch_f32": (i32, [P, P, P, u64, P]),
    "kog_split_batch_f64": (i32, [P, P, P, u64, P]),
    "kog_split_batch_f32": (i32, [P, P, P, u64, P]),
    "kog_assemble_batch_f64": (i32, [P, P, P, u64, P]),
    "kog_assemble_batch_f32": (i32, [P, P, P, u64, P]),
    "kog_tan_from_double_angle_batch_f64": (i32, [P, P, u64, P]),
    "kog_tan_from_double_angle_batch_f32": (i32, [P, P, u64, P]),
    "kog_sec_from_tan_batch_f64": (i32, [P, P, u64, P]),
    "kog_sec_from_tan_batch_f32": (i32, [P, P, u64, P]),
    "kog_epair_batch_f64": (i32, [i32, P, P, P, P, P, P, P, u64, P]),
    "kog_epair_batch_f32": (i32, [i32, P, P, P, P, P, P, P, u64, P]),
    "kog_classify_prescale_batch_f64": (i32, [PTR(kog_mat), PTR(kog_classify_out), PTR(kog_mat), u64, P]),
    "kog_classify_prescale_batch_f32": (i32, [PTR(kog_mat), PTR(kog_classify_out), PTR(kog_mat), u64, P]),
    "kog_urv15_batch_f64": (i32, [PTR(kog_mat), P, u64, PTR(kog_options), P]),
    "kog_urv15_batch_f32": (i32, [PTR(kog_mat), P, u64, PTR(kog_options), P]),
    "kog_tri_svd_batch_f64": (i32, [P, P, P, P, P, u64, PTR(kog_options), P]),
    "kog_tri_svd_batch_f32": (i32, [P, P, P, P, P, u64, PTR(kog_options), P]),
    "kog_compose_left_batch_f64": (i32, [P, P, P, P, P, u64, P]),
    "kog_compose_left_batch_f32": (i32, [P, P, P, P, P, u64, P]),
    "kog_triangularize13_batch_f64": (i32, [PTR(kog_mat), P, PTR(kog_mat), P, P, u64, P]),
    "kog_triangularize13_batch_f32": (i32, [PTR(kog_mat), P, PTR(kog_mat), P, P, u64, P]),
    "kog_svd2_ext_batch_f64": (i32, [PTR(kog_mat), P, u64, P]),
    "kog_svd2_ext_batch_f32": (i32, [PTR(kog_mat), P, u64, P]),
    "kog_metrics_batch_f64": (i32, [PTR(kog_mat), P, u64, PTR(kog_options), P]),
    "kog_metrics_batch_f32": (i32, [PTR(kog_mat), P, u64, PTR(kog_options), P]),
    "kog_generate_batch_f64": (i32, [PTR(kog_run_config), u64, PTR(kog_mat), u64, P]),
    "kog_generate_batch_f32": (i32, [PTR(kog_run_config), u64, PTR(kog_mat), u64, P]),
    "kog_stats_init": (None, [PTR(kog_stats)]),
    "kog_stats_merge": (None, [PTR(kog_stats), PTR(kog_stats)]),
    "kog_study_stats_alloc": (i32, [PTR(P)]),
    "kog_study_stats_free": (i32, [P]),
    "kog_study_stats_reset": (i32, [P, P]),
    "kog_study_batch": (i32, [PTR(kog_run_config), u64, u64, P, P]),
    "kog_validate": (i32, [PTR(kog_run_config)]),
    "kog_run_batch": (i32, [PTR(kog_run_config), PTR(kog_stats)]),
    "kog_abort_message": (i32, [PTR(kog_run_config), u64, C.c_char_p, C.c_size_t]),
    "kog_csv_header": (i32, [C.c_char_p, C.c_size_t]),
    "kog_csv_row": (i32, [PTR(kog_run_config), PTR(kog_stats), C.c_char_p, C.c_size_t]),
    "kog_lasv2_batch_f64": (i32, [P, P, P, P, u64, P]),
    "kog_lasv2_batch_f32": (i32, [P, P, P, P, u64, P]),
    "kog_fp64_probe": (i32, [P, u64, C.c_uint32, P]),
    "kog_svd2_deferred_count": (C.c_int64, []),
    "kog_svd2_lean_count": (C.c_int64, []),
    "kog_svd2_set_lean_min": (C.c_uint64, [C.c_uint64]),
    "kog_study_set_chunk_log2": (C.c_int, [C.c_int]),
    "kog_div_batch_f64": (i32, [P, P, P, u64, P]),
    "kog_div_batch_f32": (i32, [P, P, P, u64, P]),
    "kog_launch_count": (C.c_uint64, []),
    # host-buffer forms (the C++ shim's surface)
    "kog_hypot_host_f64": (i32, [P, P, P, u64]),
    "kog_hypot_host_f32": (i32, [P, P, P, u64]),
    "kog_svd2_ext_host_f64": (i32, [PTR(kog_mat), P, u64]),
    "kog_svd2_ext_host_f32": (i32, [PTR(kog_mat), P, u64]),
    "kog_metrics_host_f64": (i32, [PTR(kog_mat), P, u64, PTR(kog_options)]),
    "kog_metrics_host_f32": (i32, [PTR(kog_mat), P, u64, PTR(kog_options)]),
    "kog_generate_host_f64": (i32, [PTR(kog_run_config), u64, PTR(kog_mat), u64]),
    "kog_generate_host_f32": (i32, [PTR(kog_run_config), u64, PTR(kog_mat), u64]),
    # multi-GPU study
    "kog_study_shard": (None, [u64, i32, i32, PTR(u64), PTR(u64)]),
    "kog_stats_slot_count": (C.c_size_t, [i32]),
    "kog_stats_pack": (i32, [PTR(kog_stats), i32, i32, P]),
    "kog_stats_unpack": (i32, [P, i32, PTR(kog_stats)]),
    "kog_nccl_available": (i32, []),
    "kog_nccl_unique_id": (i32, [P, C.c_size_t]),
    "kog_nccl_comm_init": (i32, [P, i32, i32, PTR(P)]),
    "kog_nccl_comm_destroy": (i32, [P]),
    "kog_study_allreduce": (i32, [P, i32, i32, PTR(kog_stats), P]),
    "kog_study_multi": (i32, [PTR(kog_run_config), P, i32, PTR(kog_stats), PTR(C.c_double)]),
}

_lib = None


class KogError(RuntimeError):
    """A non-zero status from the C-ABI (message from kog_last_error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"kog2 error {code}: {msg}")
        self.code = code
        self.msg = msg


def load(path: str | None = None) -> C.CDLL:
    """Load libkog2.so and bind every prototype.  Raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(p)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if os.environ.get("KOG2_LEAN_MIN_LOG2"):  # tuning runs (tools/lean_sizes.sh): the two-speed kernel's threshold
        lib.kog_svd2_set_lean_min(1 << int(os.environ["KOG2_LEAN_MIN_LOG2"]))
    if os.environ.get("KOG2_STUDY_CHUNK_LOG2"):  # tuning runs: the phased study's chunk
        lib.kog_study_set_chunk_log2(int(os.environ["KOG2_STUDY_CHUNK_LOG2"]))
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> int:
    if rc < 0:
        raise KogError(rc, load().kog_last_error().decode())
    return rc


def default_options() -> kog_options:
    return kog_options(1, 0, KOG_WIDE_WIDER_TYPE, 0)
