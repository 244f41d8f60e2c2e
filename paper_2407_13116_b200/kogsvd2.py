"""Host-side mirror of the reference's kogsvd2 API over the kog2 C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/kogsvd2 (cited per function); every call runs the
sm_100a kernels of libkog2.so.  torch supplies device memory and the current
CUDA stream only.  A matrix batch is a (4, n) tensor whose rows are
g11, g12, g21, g22 (structure of arrays, Matrix2 of classify.hpp:14-19).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import capi
from .capi import check

_F = {torch.float64: "f64", torch.float32: "f32"}


def _lib():
    return capi.load()


def _stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _suffix(t: torch.Tensor) -> str:
    try:
        return _F[t.dtype]
    except KeyError:
        raise TypeError(f"working precision must be float32 or float64, got {t.dtype}") from None


def _cuda(t: torch.Tensor) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError("kog2 batched entry points take CUDA tensors")
    return t.contiguous()


# ------------------------------------------------------------------ options
@dataclass
class Options:
    """Options (svd2.hpp:124-132)."""
    hypot_is_cr: bool = True
    ominus_for_d: bool = False
    wide_channel: int = capi.KOG_WIDE_WIDER_TYPE  # or capi.KOG_WIDE_KAHAN_DET

    def c(self) -> capi.kog_options:
        return capi.kog_options(int(self.hypot_is_cr), int(self.ominus_for_d), int(self.wide_channel), 0)


def _mat(g: torch.Tensor) -> capi.kog_mat:
    return capi.kog_mat(g[0].data_ptr(), g[1].data_ptr(), g[2].data_ptr(), g[3].data_ptr())


SVD_FIELDS = ("sig1_f", "sig2_f", "sig1_e", "sig2_e", "u11", "u12", "v11", "v12", "s", "flags")


def empty_result(n: int, dtype, device) -> dict[str, torch.Tensor]:
    out = {}
    for k in SVD_FIELDS:
        if k in ("sig1_e", "sig2_e", "s"):
            out[k] = torch.empty(n, dtype=torch.int32, device=device)
        elif k == "flags":
            out[k] = torch.empty(n, dtype=torch.int32, device=device)  # uint32 bit pattern
        else:
            out[k] = torch.empty(n, dtype=dtype, device=device)
    return out


def _out(o: dict[str, torch.Tensor]) -> capi.kog_svd_out:
    return capi.kog_svd_out(*[o[k].data_ptr() for k in SVD_FIELDS])


# ------------------------------------------------------------------- svd2
def svd2(g: torch.Tensor, opt: Options | None = None, out: dict | None = None) -> dict[str, torch.Tensor]:
    """svd2(G, opt) (svd2.hpp:603-687) on a (4, n) CUDA batch; compact result
    (include/kog2.h): sigma_i = 2^sig{i}_e * sig{i}_f, U/V from u11, u12, v11,
    v12 and the flag sign bits, s, BranchTrace bits."""
    g = _cuda(g)
    n = g.shape[1]
    suf = _suffix(g)
    if out is None:
        out = empty_result(n, g.dtype, g.device)
    o = (opt or Options()).c()
    check(getattr(_lib(), f"kog_svd2_batch_{suf}")(C.byref(_mat(g)), C.byref(_out(out)), n, C.byref(o),
                                                  _stream(g.device)))
    return out


def svd2_host(g, opt: Options | None = None, out: dict | None = None) -> dict[str, torch.Tensor]:
    """svd2 on HOST (ideally pinned) tensors through kog_svd2_host_*: chunked
    H2D -> kernel -> D2H pipeline on the current device."""
    assert not g.is_cuda
    g = g.contiguous()
    n = g.shape[1]
    suf = _suffix(g)
    if out is None:
        out = empty_result(n, g.dtype, "cpu")
    o = (opt or Options()).c()
    check(getattr(_lib(), f"kog_svd2_host_{suf}")(C.byref(_mat(g)), C.byref(_out(out)), n, C.byref(o)))
    return out


def expand_result(r: dict[str, torch.Tensor]) -> dict[str, torch.Tensor]:
    """Full U, V (each (4, n): x11, x12, x21, x22) from the compact layout."""
    fl = r["flags"].to(torch.int64) & 0xFFFFFFFF

    def signed(mag, bit):
        neg = (fl & bit) != 0
        a = mag.abs()
        return torch.where(neg, -a, a)

    u = torch.stack([r["u11"], r["u12"], signed(r["u12"], capi.F_SIGN_U21), signed(r["u11"], capi.F_SIGN_U22)])
    v = torch.stack([r["v11"], r["v12"], signed(r["v12"], capi.F_SIGN_V21), signed(r["v11"], capi.F_SIGN_V22)])
    return {"u": u, "v": v}


# ---------------------------------------------------------- unit routines
def hypot_cr(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """hypot_cr<T> (fpcore.hpp:140-188), correctly rounded."""
    a, b = _cuda(a), _cuda(b)
    out = torch.empty_like(a)
    check(getattr(_lib(), f"kog_hypot_batch_{_suffix(a)}")(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.numel(),
                                                             _stream(a.device)))
    return out


def split(x: torch.Tensor):
    """split (fpcore.hpp:41-47) -> (e int64, f)."""
    x = _cuda(x)
    e = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
    f = torch.empty_like(x)
    check(getattr(_lib(), f"kog_split_batch_{_suffix(x)}")(x.data_ptr(), e.data_ptr(), f.data_ptr(), x.numel(),
                                                             _stream(x.device)))
    return e, f


def assemble(e: torch.Tensor, f: torch.Tensor) -> torch.Tensor:
    """assemble (fpcore.hpp:51-55)."""
    e, f = _cuda(e.to(torch.int64)), _cuda(f)
    out = torch.empty_like(f)
    check(getattr(_lib(), f"kog_assemble_batch_{_suffix(f)}")(e.data_ptr(), f.data_ptr(), out.data_ptr(),
                                                                f.numel(), _stream(f.device)))
    return out


def tan_from_double_angle(t2: torch.Tensor) -> torch.Tensor:
    """tan_from_double_angle (fpcore.hpp:192-196)."""
    t2 = _cuda(t2)
    out = torch.empty_like(t2)
    check(getattr(_lib(), f"kog_tan_from_double_angle_batch_{_suffix(t2)}")(t2.data_ptr(), out.data_ptr(),
                                                                              t2.numel(), _stream(t2.device)))
    return out


def sec_from_tan(t: torch.Tensor) -> torch.Tensor:
    """sec_from_tan (fpcore.hpp:198-201)."""
    t = _cuda(t)
    out = torch.empty_like(t)
    check(getattr(_lib(), f"kog_sec_from_tan_batch_{_suffix(t)}")(t.data_ptr(), out.data_ptr(), t.numel(),
                                                                    _stream(t.device)))
    return out


def epair_op(op: int, xf: torch.Tensor, yf: torch.Tensor | None = None, xe: torch.Tensor | None = None,
             ye: torch.Tensor | None = None):
    """EPair operations (epair.hpp): returns (e, f, status); status 1 where the
    reference throws std::domain_error."""
    xf = _cuda(xf)
    n = xf.numel()
    dev = xf.device
    xe = None if xe is None else _cuda(xe.to(torch.int64))
    ye = None if ye is None else _cuda(ye.to(torch.int64))
    yf = None if yf is None else _cuda(yf)
    oe = torch.empty(n, dtype=torch.int64, device=dev)
    of = torch.empty_like(xf)
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    check(getattr(_lib(), f"kog_epair_batch_{_suffix(xf)}")(op, _p(xe), xf.data_ptr(), _p(ye), _p(yf),
                                                              oe.data_ptr(), of.data_ptr(), st.data_ptr(), n,
                                                              _stream(dev)))
    return oe, of, st


def classify_prescale(g: torch.Tensor):
    """classify (classify.hpp:44-58) + prescale (classify.hpp:67-78)."""
    g = _cuda(g)
    n = g.shape[1]
    dev = g.device
    o = {"t": torch.empty(n, dtype=torch.uint8, device=dev), "s_type": torch.empty(n, dtype=torch.int32, device=dev),
         "s": torch.empty(n, dtype=torch.int64, device=dev), "e_G": torch.empty(n, dtype=torch.int64, device=dev),
         "inexact_underflow": torch.empty(n, dtype=torch.uint8, device=dev),
         "status": torch.empty(n, dtype=torch.uint8, device=dev)}
    gp = torch.empty_like(g)
    co = capi.kog_classify_out(*[o[k].data_ptr() for k in ("t", "s_type", "s", "e_G", "inexact_underflow", "status")])
    check(getattr(_lib(), f"kog_classify_prescale_batch_{_suffix(g)}")(C.byref(_mat(g)), C.byref(co),
                                                                         C.byref(_mat(gp)), n, _stream(dev)))
    o["gp"] = gp
    return o


def _records(ctype, n: int, dev) -> torch.Tensor:
    return torch.empty(n * C.sizeof(ctype), dtype=torch.uint8, device=dev)


def records_to_host(buf: torch.Tensor, ctype, n: int):
    """Copy a device record array back as a ctypes array."""
    host = buf.cpu().numpy()
    arr = (ctype * n)()
    C.memmove(arr, host.ctypes.data, n * C.sizeof(ctype))
    return arr


def urv15(gp: torch.Tensor, opt: Options | None = None):
    """urv15 (svd2.hpp:339-384): ctypes array of kog_urv15_* records."""
    gp = _cuda(gp)
    n = gp.shape[1]
    suf = _suffix(gp)
    rt = capi.kog_urv15_f64 if suf == "f64" else capi.kog_urv15_f32
    buf = _records(rt, n, gp.device)
    check(getattr(_lib(), f"kog_urv15_batch_{suf}")(C.byref(_mat(gp)), buf.data_ptr(), n,
                                                      C.byref((opt or Options()).c()), _stream(gp.device)))
    return records_to_host(buf, rt, n)


def tri_svd(r11: torch.Tensor, r12: torch.Tensor, r22: torch.Tensor, t13, opt: Options | None = None):
    """tri_svd (svd2.hpp:438-474) incl. tan2phi's value (t2f) and branch."""
    r11, r12, r22 = _cuda(r11), _cuda(r12), _cuda(r22)
    n = r11.numel()
    suf = _suffix(r11)
    if isinstance(t13, bool):
        t13 = torch.full((n,), int(t13), dtype=torch.uint8, device=r11.device)
    t13 = _cuda(t13.to(torch.uint8))
    rt = capi.kog_trisvd_f64 if suf == "f64" else capi.kog_trisvd_f32
    buf = _records(rt, n, r11.device)
    check(getattr(_lib(), f"kog_tri_svd_batch_{suf}")(r11.data_ptr(), r12.data_ptr(), r22.data_ptr(),
                                                        t13.data_ptr(), buf.data_ptr(), n,
                                                        C.byref((opt or Options()).c()), _stream(r11.device)))
    return records_to_host(buf, rt, n)


def compose_left(tan_phi_bold: torch.Tensor, tan_theta: torch.Tensor, minus_form):
    """compose_left (svd2.hpp:485-515) -> (c, s)."""
    a, b = _cuda(tan_phi_bold), _cuda(tan_theta)
    n = a.numel()
    if isinstance(minus_form, bool):
        minus_form = torch.full((n,), int(minus_form), dtype=torch.uint8, device=a.device)
    m = _cuda(minus_form.to(torch.uint8))
    c, s = torch.empty_like(a), torch.empty_like(a)
    check(getattr(_lib(), f"kog_compose_left_batch_{_suffix(a)}")(a.data_ptr(), b.data_ptr(), m.data_ptr(),
                                                                    c.data_ptr(), s.data_ptr(), n,
                                                                    _stream(a.device)))
    return c, s


def triangularize13(gp: torch.Tensor, t: torch.Tensor):
    """triangularize13 (svd2.hpp:257-271) -> (R (4, n), Uplus int8 (n,4), Vplus int8 (n,4))."""
    gp = _cuda(gp)
    n = gp.shape[1]
    t = _cuda(t.to(torch.uint8))
    r = torch.empty_like(gp)
    up = torch.empty((n, 4), dtype=torch.int8, device=gp.device)
    vp = torch.empty((n, 4), dtype=torch.int8, device=gp.device)
    check(getattr(_lib(), f"kog_triangularize13_batch_{_suffix(gp)}")(C.byref(_mat(gp)), t.data_ptr(),
                                                                        C.byref(_mat(r)), up.data_ptr(),
                                                                        vp.data_ptr(), n, _stream(gp.device)))
    return r, up, vp


def svd2_ext(g: torch.Tensor):
    """svd2_ext (oracle.hpp:102-238): ctypes array of kog_extsvd."""
    g = _cuda(g)
    n = g.shape[1]
    buf = _records(capi.kog_extsvd, n, g.device)
    check(getattr(_lib(), f"kog_svd2_ext_batch_{_suffix(g)}")(C.byref(_mat(g)), buf.data_ptr(), n,
                                                                _stream(g.device)))
    return records_to_host(buf, capi.kog_extsvd, n)


def metrics(g: torch.Tensor, opt: Options | None = None):
    """metrics(g, svd2(g), svd2_ext(g)) (oracle.hpp:269-301): kog_metrics records."""
    g = _cuda(g)
    n = g.shape[1]
    buf = _records(capi.kog_metrics, n, g.device)
    check(getattr(_lib(), f"kog_metrics_batch_{_suffix(g)}")(C.byref(_mat(g)), buf.data_ptr(), n,
                                                               C.byref((opt or Options()).c()), _stream(g.device)))
    return records_to_host(buf, capi.kog_metrics, n)


def lasv2(f: torch.Tensor, g: torch.Tensor, h: torch.Tensor) -> torch.Tensor:
    """lasv2_ref (lasv2.hpp:22-127) -> (n, 6): ssmin, ssmax, snr, csr, snl, csl."""
    f, g, h = _cuda(f), _cuda(g), _cuda(h)
    out = torch.empty((f.numel(), 6), dtype=f.dtype, device=f.device)
    check(getattr(_lib(), f"kog_lasv2_batch_{_suffix(f)}")(f.data_ptr(), g.data_ptr(), h.data_ptr(),
                                                             out.data_ptr(), f.numel(), _stream(f.device)))
    return out


# ----------------------------------------------------------------- harness
@dataclass
class RunConfig:
    """RunConfig (harness.hpp:27-37) plus the kog2 generator extension
    (include/kog2.h, regime KOG_REGIME_RANGED)."""
    single_precision: bool = False
    shape: int = capi.SHAPE_TRI
    regime: int = capi.REGIME_CIRC
    varsigma: int = 0
    count: int = 0
    seed: int = 0
    routine: int = capi.ROUTINE_KOG
    threads: int = 1
    options: Options = field(default_factory=Options)
    elo: int = 0
    ehi: int = 0
    tail_lo: int = 0
    tail_hi: int = 0
    tail_mod: int = 0
    zero_mask_rule: int = 0

    def c(self) -> capi.kog_run_config:
        return capi.kog_run_config(int(self.single_precision), self.shape, self.regime, self.routine, self.varsigma,
                                   self.count, self.seed, self.threads, self.options.c(), self.elo, self.ehi,
                                   self.tail_lo, self.tail_hi, self.tail_mod, self.zero_mask_rule)

    @property
    def dtype(self):
        return torch.float32 if self.single_precision else torch.float64


class BatchAbort(RuntimeError):
    """BatchAbort (harness.hpp:108-110)."""


def validate(cfg: RunConfig) -> None:
    """validate<T> (harness.hpp:39-48): raises ValueError (std::invalid_argument)."""
    rc = _lib().kog_validate(C.byref(cfg.c()))
    if rc != capi.KOG_OK:
        raise ValueError(_lib().kog_last_error().decode())


def generate(cfg: RunConfig, index0: int, n: int, device=None) -> torch.Tensor:
    """generate<T>(cfg, index) (harness.hpp:139-186) for index0..index0+n-1."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    g = torch.empty((4, n), dtype=cfg.dtype, device=device)
    suf = "f32" if cfg.single_precision else "f64"
    rc = getattr(_lib(), f"kog_generate_batch_{suf}")(C.byref(cfg.c()), index0, C.byref(_mat(g)), n,
                                                       _stream(device))
    if rc == capi.KOG_ERR_ARG:
        raise ValueError(_lib().kog_last_error().decode())
    check(rc)
    return g


def new_stats() -> capi.kog_stats:
    st = capi.kog_stats()
    _lib().kog_stats_init(C.byref(st))
    return st


def merge_stats(st: capi.kog_stats, o: capi.kog_stats) -> capi.kog_stats:
    """ErrorStats::merge (harness.hpp:96-105), in place on st."""
    _lib().kog_stats_merge(C.byref(st), C.byref(o))
    return st


class StudyStats:
    """Device-resident ErrorStats accumulated by kog_study_batch."""

    def __init__(self):
        self.ptr = C.c_void_p()
        check(_lib().kog_study_stats_alloc(C.byref(self.ptr)))

    def reset(self):
        check(_lib().kog_study_stats_reset(self.ptr, _stream()))

    def add(self, cfg: RunConfig, index0: int, n: int):
        rc = _lib().kog_study_batch(C.byref(cfg.c()), index0, n, self.ptr, _stream())
        if rc == capi.KOG_ERR_ARG:
            raise ValueError(_lib().kog_last_error().decode())
        check(rc)

    def read(self) -> capi.kog_stats:
        torch.cuda.current_stream().synchronize()
        nbytes = C.sizeof(capi.kog_stats)
        host = _device_bytes(self.ptr.value, nbytes).cpu().numpy()
        st = capi.kog_stats()
        C.memmove(C.byref(st), host.ctypes.data, nbytes)
        return st

    def free(self):
        if self.ptr:
            _lib().kog_study_stats_free(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _device_bytes(ptr: int, nbytes: int) -> torch.Tensor:
    """A uint8 CUDA tensor aliasing raw device memory (no copy)."""
    class _Cai:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Cai(), device="cuda")


def run_batch(cfg: RunConfig) -> capi.kog_stats:
    """run_batch_any (harness.hpp:226-271, 319-321), GPU-backed.  Raises
    ValueError for an invalid config and BatchAbort with the reference's
    message when a matrix fails."""
    st = capi.kog_stats()
    rc = _lib().kog_run_batch(C.byref(cfg.c()), C.byref(st))
    if rc == capi.KOG_ERR_ARG:
        raise ValueError(_lib().kog_last_error().decode())
    if rc == capi.KOG_ERR_ABORT:
        raise BatchAbort(_lib().kog_last_error().decode())
    check(rc)
    return st


run_batch_any = run_batch


def csv_header() -> str:
    buf = C.create_string_buffer(256)
    check(_lib().kog_csv_header(buf, 256))
    return buf.value.decode()


def csv_row(cfg: RunConfig, st: capi.kog_stats) -> str:
    """csv_row (harness.hpp:290-317), byte-identical to the reference."""
    buf = C.create_string_buffer(512)
    check(_lib().kog_csv_row(C.byref(cfg.c()), C.byref(st), buf, 512))
    return buf.value.decode()


def launch_count() -> int:
    return int(_lib().kog_launch_count())
