"""Per-reason counts of matrices leaving the fast svd2 path and of rare-path
calls (needs the KOG2_FAST_STATS variant: KOG2_LIB=.../libkog2_stats.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_13116_b200 import capi, configs  # noqa: E402
from paper_2407_13116_b200 import kogsvd2 as K  # noqa: E402

NAMES = ["div", "hypot_arg", "hypot_ziv", "ep", "scal", "epval", "pattern", "subnormal_in", "s<0", "prescale",
         "t2p_equal", "general_inf", "oplus", "degenerate", "ilogb", "-",
         "rare:ilogb_sub", "rare:mant_sub", "rare:scalbn_slow", "rare:div_rare", "rare:hypot_rare", "rare:ep_make_rare",
         "-", "-", "div:y0", "div:inf", "div:nan", "div:x0_ysub", "div:sub_operand", "div:sub_result", "-",
         "div:x0_inline"]
lib = capi.load()
fn = lib.kog2_fast_stats
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 96)()
for k in (1, 2, 3, 4):
    c = configs.cfg(k, count=1 << 22)
    g = K.generate(c, 0, c.count)
    torch.cuda.synchronize()
    fn(buf, 1)
    d0 = lib.kog_svd2_deferred_count()
    K.svd2(g)
    torch.cuda.synchronize()
    fn(buf, 1)
    d = lib.kog_svd2_deferred_count() - d0
    print(f"cfg{k}: deferred {d / c.count:.4f}; events per matrix:",
          {NAMES[i]: round(buf[i] / c.count, 4) for i in range(32) if buf[i]})
    print("   div sites (zero numerator):", {i: round(buf[32 + i] / c.count, 4) for i in range(32) if buf[32 + i]})
    print("   div sites (off fast path):", {i: round(buf[64 + i] / c.count, 4) for i in range(32) if buf[64 + i]})
