"""Full-population parity at the bench sizes (SURVEY.md §8(d) parity row:
"cfg1-4 in full"): ONE kog_svd2_batch call over the whole on-device batch
(2^26 or 2^28 matrices, the bench workload itself), then EVERY field of EVERY
matrix compared bit-for-bit with the reference's svd2 (oracle/_ref, all host
threads; svd2.hpp:603-687 on the generator of harness.hpp:139-186 with the
§8(d) extensions) in 2^24-matrix chunks.  Config 5 (2^31 matrices, the study
stream) is checked on eight 2^24-matrix windows spread over [0, 2^31),
including the first and the last.  Each test asserts zero mismatches out of N.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import refbind
from paper_2407_13116_b200 import capi, configs
from paper_2407_13116_b200 import kogsvd2 as K

pytestmark = pytest.mark.gpu

CHUNK = 1 << 24


def _int_view(t: torch.Tensor) -> torch.Tensor:
    return t.view({8: torch.int64, 4: torch.int32}[t.element_size()])


def mismatches(got: dict, lo: int, want: dict) -> tuple[int, int]:
    """(number of matrices whose result differs in any field, first such index)
    between got[k][lo:lo+W] (device) and want[k] (host, the reference)."""
    w = next(iter(want.values())).size
    bad = torch.zeros(w, dtype=torch.bool, device="cuda")
    for k in refbind.OUT_DTYPES:
        g = _int_view(got[k][lo:lo + w])
        ref = torch.from_numpy(want[k]).cuda()
        bad |= g != _int_view(ref)
    nbad = int(bad.sum())
    first = int(torch.nonzero(bad)[0]) + lo if nbad else -1
    return nbad, first


def check_full(ref, cfg: K.RunConfig, count: int, index0: int = 0) -> int:
    g = K.generate(cfg, index0, count)
    r = K.svd2(g)
    torch.cuda.synchronize()
    assert int((r["flags"].view(torch.int32) < 0).sum()) == 0, "domain-error bit set on finite input"
    del g
    checked = 0
    for lo in range(0, count, CHUNK):
        w = min(CHUNK, count - lo)
        gh = refbind.generate(ref, cfg.c(), index0 + lo, w)
        want = refbind.svd2(ref, gh)
        nbad, first = mismatches(r, lo, want)
        assert nbad == 0, f"{nbad} of {w} matrices differ at indices [{index0 + lo}, +{w}); first {index0 + first}"
        checked += w
    del r
    torch.cuda.empty_cache()
    return checked


@pytest.mark.parametrize("k,count", [(2, 1 << 26), (3, 1 << 28), (4, 1 << 28)], ids=["cfg2", "cfg3", "cfg4"])
def test_svd2_full_population(cuda, ref, k, count):
    cfg = configs.cfg(k, count=count)
    assert check_full(ref, cfg, count) == count


def test_cfg5_windows(cuda, ref):
    """Config 5's 2^31-matrix stream: eight 2^24-matrix windows over the whole
    index range (first, last and six in between), each one svd2 call."""
    cfg = configs.cfg(5)
    total = cfg.count
    assert total == 1 << 31
    W = 1 << 24
    starts = [0, total - W] + [int(x) * W for x in np.linspace(1, total // W - 2, 6).round()]
    for s in sorted(set(starts)):
        assert check_full(ref, cfg, W, index0=s) == W


def test_mismatch_detector_fires(cuda, ref):
    """The comparison itself: a one-bit change in one field of one matrix is
    reported with its index."""
    cfg = configs.cfg(3, count=4096)
    g = K.generate(cfg, 0, cfg.count)
    r = K.svd2(g)
    want = refbind.svd2(ref, refbind.generate(ref, cfg.c(), 0, cfg.count))
    assert mismatches(r, 0, want) == (0, -1)
    r["v12"][1234] = torch.from_numpy(np.array([np.nextafter(want["v12"][1234], 2.0)])).cuda()[0]
    assert mismatches(r, 0, want) == (1, 1234)
