"""The two-speed binary64 decomposition kernel (k_svd2_lean, batches of 2^22
and more with the default Options): every route through its queues against the
reference's svd2 (svd2.hpp:603-687), bit for bit — mixed batches whose regions
change the class mix under the warps' feet (lean-friendly, triangular, narrow
range, sparse, deferring), ragged sizes, the sample's hand-back to
k_svd2_fast, several launches in flight."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import refbind
from paper_2407_13116_b200 import capi, configs
from paper_2407_13116_b200 import kogsvd2 as K
from tests import _gen
from tests.test_gpu_parity import compare_svd, dev, host
from tests.test_gpu_reentrancy import deferring_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def small_batches_on_the_lean_kernel():
    """the kernel normally takes batches of 2^24 and more; these tests run it on 2^22"""
    lib = capi.load()
    before = lib.kog_svd2_set_lean_min(1 << 22)
    yield
    lib.kog_svd2_set_lean_min(before)


def cfg_host(k: int, n: int, off: int = 0) -> np.ndarray:
    """(4, n) host matrices of a BASELINE config's generator"""
    return host(K.generate(configs.cfg(k, count=off + n), off, n))


def sparse(seed: int, n: int) -> np.ndarray:
    """config-3 entries with every zero pattern equally likely (the all-zero matrix included)"""
    g = cfg_host(3, n, 1 << 20)
    mask = (_gen.draws(seed, n, 0) % np.uint64(16)).astype(np.int64)
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][(mask & bit) == 0] = 0
    return g


def mixed_batch(n: int, order: int) -> np.ndarray:
    """about 70% lean-friendly matrices (so that the kernel's sample keeps the
    batch) cut by stretches of every other kind, in pieces of uneven lengths"""
    pieces = []
    left = n
    k = 0
    kinds = [3, "tri", 3, "circ", 3, "sparse", 3, "defer", 3, 3, "tri", 3][order:] + [3]
    sizes = {3: 311_111, "tri": 70_001, "circ": 65_537, "sparse": 50_021, "defer": 40_009}
    while left > 0:
        kind = kinds[k % len(kinds)]
        m = min(left, sizes[kind] + 977 * k)
        if kind == 3:
            pieces.append(cfg_host(3, m, 12345 * k))
        elif kind == "tri":
            pieces.append(cfg_host(2, m, 999 * k))
        elif kind == "circ":
            pieces.append(cfg_host(1, m, 77 * k))
        elif kind == "sparse":
            pieces.append(sparse(0x51 + k, m))
        else:
            pieces.append(deferring_batch(np.float64, 0xDE00 + k, m))
        left -= m
        k += 1
    return np.ascontiguousarray(np.concatenate(pieces, axis=1))


@pytest.mark.parametrize("n,order", [((1 << 22) + (1 << 20) + 37, 0), ((1 << 22) + 1, 3), (3 * (1 << 21) + 31, 1)])
def test_lean_kernel_mixed_batches(cuda, ref, n, order):
    g = mixed_batch(n, order)
    lib = capi.load()
    kept0, def0 = lib.kog_svd2_lean_count(), lib.kog_svd2_deferred_count()
    got = K.svd2(dev(g))
    torch.cuda.synchronize()
    assert lib.kog_svd2_lean_count() == kept0 + 1, "the sample handed the batch back: k_svd2_lean did not run"
    assert lib.kog_svd2_deferred_count() > def0, "no lane reached the general kernel"
    compare_svd(got, refbind.svd2(ref, g), f"mixed batch n={n}")


def test_lean_kernel_hands_unfriendly_batches_back(cuda, ref):
    """narrow-range, triangular and deferring batches of 2^22: the sample sends
    them to k_svd2_fast (same results either way)"""
    n = (1 << 22) + 5
    for what, g in (("circ", cfg_host(1, n)), ("tri", cfg_host(2, n)), ("defer", deferring_batch(np.float64, 0xAB, n))):
        kept0 = capi.load().kog_svd2_lean_count()
        got = K.svd2(dev(g))
        torch.cuda.synchronize()
        assert capi.load().kog_svd2_lean_count() == kept0, f"{what}: kept on the two-speed kernel"
        compare_svd(got, refbind.svd2(ref, g), what)


def test_lean_kernel_config3_window_and_streams(cuda, ref):
    """config 3 at 2^22 + a ragged tail on three streams at once (each launch
    its own queues and workspace), all equal to the reference"""
    n = (1 << 22) + 12345
    gs = [cfg_host(3, n, off) for off in (0, 1 << 24, (1 << 27) + 3)]
    ds = [dev(g) for g in gs]
    streams = [torch.cuda.Stream() for _ in ds]
    torch.cuda.synchronize()
    kept0 = capi.load().kog_svd2_lean_count()
    outs = []
    for d, s in zip(ds, streams):
        with torch.cuda.stream(s):
            outs.append(K.svd2(d))
    torch.cuda.synchronize()
    assert capi.load().kog_svd2_lean_count() == kept0 + 3
    for k, (g, r) in enumerate(zip(gs, outs)):
        compare_svd(r, refbind.svd2(ref, g), f"stream {k}")


def test_lean_kernel_guard_zones(cuda, ref):
    """the two-speed kernel on arrays carved out of larger allocations (64 KiB
    guard zones, 8-byte-aligned but not 16-byte-aligned pointers: its cp.async
    copies are 8 bytes wide) at a ragged size: no write outside the arrays, the
    inputs unchanged, results equal to the reference"""
    import ctypes as C

    from tests.test_gpu_guards import Arena, _st

    lib = capi.load()
    n = (1 << 22) + 4099
    g = mixed_batch(n, 2)
    A = Arena()
    ins = [A.array(n, torch.float64, g[k]) for k in range(4)]
    outs = {k: A.array(n, torch.int32 if k in ("sig1_e", "sig2_e", "s", "flags") else torch.float64)
            for k in K.SVD_FIELDS}
    m = capi.kog_mat(*[t.data_ptr() for t in ins])
    o = capi.kog_svd_out(*[outs[k].data_ptr() for k in K.SVD_FIELDS])
    kept0 = lib.kog_svd2_lean_count()
    opt = capi.default_options()
    capi.check(lib.kog_svd2_batch_f64(C.byref(m), C.byref(o), n, C.byref(opt), _st()))
    A.check("k_svd2_lean")
    assert lib.kog_svd2_lean_count() == kept0 + 1
    compare_svd(outs, refbind.svd2(ref, g), "guarded two-speed call")


def _edge_matrices(rng: np.random.Generator, reps: int) -> np.ndarray:
    """matrices that sit on svd2_lean's acceptance thresholds (kog2_lean.cuh):
    column entries 28 binades apart give or take a binade and an ulp of the
    high word, a near column whose larger entry is half the other column's
    give or take the same, r12 against r11 and tan(2 phi) around 2^-27 — each
    with random significands, signs and row/column arrangements"""
    out = []

    def rnd_m(k):  # significands in [1, 2), some at the ends of the range
        m = 1.0 + rng.random(k)
        pick = rng.integers(0, 8, k)
        m[pick == 0] = 1.0
        m[pick == 1] = np.nextafter(2.0, 1.0)
        m[pick == 2] = 1.0 + 2.0 ** -20
        m[pick == 3] = 1.0 + 2.0 ** -20 - 2.0 ** -52
        return m

    def emit(g11, g12, g21, g22):
        g = np.stack([g11, g12, g21, g22])
        k = g.shape[1]
        g = g * rng.choice([-1.0, 1.0], size=(4, k))
        # random row and column exchanges (rows: g11<->g21, g12<->g22; columns: g11<->g12, g21<->g22)
        rs, cs = rng.random(k) < 0.5, rng.random(k) < 0.5
        g[:, rs] = g[[2, 3, 0, 1]][:, rs]
        g[:, cs] = g[[1, 0, 3, 2]][:, cs]
        out.append(g)

    for _ in range(reps):
        k = 4096
        E = rng.integers(-300, 300, k).astype(np.float64)
        # 1. the pivot column's gap around 28 binades; the other column far below and separated
        d = rng.choice([26, 27, 28, 29, 30], k).astype(np.float64)
        x = rnd_m(k) * 2.0 ** E
        y = rnd_m(k) * 2.0 ** (E - d)
        p = rnd_m(k) * 2.0 ** (E - rng.integers(40, 200, k))
        q = rnd_m(k) * 2.0 ** (E - rng.integers(240, 400, k))
        emit(x, p, y, q)
        # 2. a near column (entries within a few binades) beside a separated one whose larger entry is about
        #    twice the near column's: the exchange decided with or without the norm
        a = rnd_m(k) * 2.0 ** E
        a2 = a * rng.choice([1.0, 0.9, 0.5, 0.75, 2.0 ** -5, 2.0 ** -27], k)
        ratio = rng.choice([1.0, 2.0 ** 0.5, 1.9999990463256836, 2.0, 2.0000019073486328, 4.0, 2.0 ** -1, 2.0 ** 20], k)
        b = np.maximum(np.abs(a), np.abs(a2)) * ratio * rng.choice([1.0, np.nextafter(1.0, 0.0), np.nextafter(1.0, 2.0)], k)
        b2 = b * 2.0 ** -rng.integers(29, 90, k).astype(np.float64) * rnd_m(k)
        emit(a, b, a2, b2)
        # 3. r12 against r11 around 2^-27 .. 2^-29 (tan psi and the hypot(r11, r12) early-out), r22 anywhere below
        x = rnd_m(k) * 2.0 ** E
        y = rnd_m(k) * 2.0 ** (E - rng.choice([26, 27, 28, 29], k))
        z = rnd_m(k) * 2.0 ** (E - rng.integers(0, 120, k))
        tiny = x * 2.0 ** -rng.integers(60, 300, k).astype(np.float64)
        emit(x, y, tiny, z)
        # 4. tan(2 phi) = 2 r12 r22 / (r11^2 - r22^2) around 2^-27
        x = rnd_m(k) * 2.0 ** E
        e12 = rng.integers(0, 28, k)
        y = rnd_m(k) * 2.0 ** (E - e12 - 29)
        z = rnd_m(k) * 2.0 ** (E - (28 - e12) + rng.integers(-1, 2, k))
        emit(x, y, x * 2.0 ** -200.0, np.minimum(z, x * 0.999))
    return np.ascontiguousarray(np.concatenate(out, axis=1))


def test_lean_kernel_threshold_edges(cuda, ref):
    """svd2_lean's acceptance tests at their thresholds (inside a config-3
    batch, so that the kernel's sample keeps it): every lane, accepted or
    queued, equals the reference"""
    rng = np.random.default_rng(0x1EA4)
    edges = _edge_matrices(rng, 8)
    assert np.isfinite(edges).all() and (edges != 0).all()
    n = 1 << 22
    g = cfg_host(3, n, 777)
    pos = rng.permutation(n)[:edges.shape[1]]  # scattered through the batch: every warp meets some
    g[:, pos] = edges
    lib = capi.load()
    kept0 = lib.kog_svd2_lean_count()
    got = K.svd2(dev(g))
    torch.cuda.synchronize()
    assert lib.kog_svd2_lean_count() == kept0 + 1
    compare_svd(got, refbind.svd2(ref, g), "threshold edges")
