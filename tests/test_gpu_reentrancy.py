"""Reentrancy of the C-ABI (SURVEY.md §8b "reentrant; stream-ordered"; the
reference's routines are pure and thread-safe, README.md:135-136).

Every entry point that needs device scratch takes it per call from the
stream-ordered workspace pool (csrc/kog2_ws.cpp).  These tests issue
overlapping calls — several streams from one host thread, several host
threads, the pinned host pipeline — on inputs with many deferred lanes (the
k_svd2_fast -> k_svd2_list hand-off whose list used to be shared), and require
every result to stay bit-exact against the reference (oracle/_ref).
"""
from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

from oracle import refbind
from paper_2407_13116_b200 import capi, configs
from paper_2407_13116_b200 import kogsvd2 as K
from tests import _gen
from tests.test_gpu_parity import compare_svd, dev

pytestmark = pytest.mark.gpu

DTS = [np.float64, np.float32]


def deferring_batch(dt, seed: int, n: int) -> np.ndarray:
    """any-finite matrices (subnormal, huge and tiny entries: many lanes leave
    the fast path) with a quarter of them given a random zero pattern."""
    g = _gen.matrices(dt, seed, n)
    mask = (_gen.draws(seed + 1, n, 0) % np.uint64(16)).astype(np.int64)
    sel = (_gen.draws(seed + 1, n, 1) % np.uint64(4)) == 0
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][sel & ((mask & bit) == 0)] = 0
    return g


@pytest.mark.parametrize("dt", DTS)
def test_svd2_interleaved_streams_one_thread(cuda, ref, dt):
    """Batches of different sizes issued alternately on two streams from one
    host thread with no synchronisation in between: every lane (deferred ones
    included) equals the reference."""
    sizes = [(1 << 20) + 7, 3 * (1 << 18) + 3, 4099, (1 << 19) + 1, 77, (1 << 20) - 5]
    hosts = [deferring_batch(dt, 0xAE00 + k, n) for k, n in enumerate(sizes)]
    devs = [dev(g) for g in hosts]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    before = capi.load().kog_svd2_deferred_count()
    outs = []
    for k, g in enumerate(devs):
        with torch.cuda.stream(streams[k % 2]):
            outs.append(K.svd2(g))
    torch.cuda.synchronize()
    deferred = capi.load().kog_svd2_deferred_count() - before
    assert deferred > sum(sizes) // 100, f"only {deferred} deferred lanes: the hand-off was not exercised"
    for k, (g, r) in enumerate(zip(hosts, outs)):
        compare_svd(r, refbind.svd2(ref, g), f"stream {k % 2} batch {k}")


@pytest.mark.parametrize("dt", DTS)
def test_svd2_concurrent_host_threads(cuda, ref, dt):
    """Four host threads, each with its own stream, calling kog_svd2_batch_*
    repeatedly at the same time (ctypes releases the GIL around the call)."""
    nthreads, reps = 4, 3
    hosts = [deferring_batch(dt, 0xBE00 + k, (1 << 18) + 13 * k) for k in range(nthreads)]
    devs = [dev(g) for g in hosts]
    torch.cuda.synchronize()
    results: list = [None] * nthreads
    errors: list = []
    barrier = threading.Barrier(nthreads)

    def worker(k: int) -> None:
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            barrier.wait()
            with torch.cuda.stream(s):
                rs = [K.svd2(devs[k]) for _ in range(reps)]
            s.synchronize()
            results[k] = rs
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(nthreads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for k in range(nthreads):
        want = refbind.svd2(ref, hosts[k])
        for j, r in enumerate(results[k]):
            compare_svd(r, want, f"thread {k} rep {j}")


@pytest.mark.parametrize("dt", DTS)
def test_svd2_host_pipeline_pinned_overlap(cuda, ref, dt):
    """kog_svd2_host_* with pinned inputs AND outputs (the three slot streams
    then really overlap) on deferring inputs, several chunks and a ragged
    tail."""
    n = 3 * (1 << 22) + 12345
    g = deferring_batch(dt, 0xCE01, n)
    gt = torch.from_numpy(g).pin_memory()
    out = {k: v.pin_memory() for k, v in K.empty_result(n, gt.dtype, "cpu").items()}
    before = capi.load().kog_svd2_deferred_count()
    got = K.svd2_host(gt, out=out)
    assert capi.load().kog_svd2_deferred_count() - before > n // 100
    compare_svd({k: v.numpy() for k, v in got.items()}, refbind.svd2(ref, g), "svd2_host pinned")


def test_studies_on_two_streams(cuda, ref):
    """Two kog_study_batch calls in flight at once on two streams (each with
    its own device ErrorStats): both equal the same studies run one at a time,
    and the smaller one equals the reference's run_batch."""
    cfg_a = configs.cfg(5, count=2 * (1 << 22) + 4099)   # three chunks of 2^22: both chunk buffers in use
    cfg_b = K.RunConfig(shape=capi.SHAPE_GEN, regime=capi.REGIME_BULLET, count=(1 << 18) + 5, seed=0x5E1)
    cfg_c = K.RunConfig(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=50000, seed=0x5E2,
                        routine=capi.ROUTINE_LASV2)
    cfgs = [cfg_a, cfg_b, cfg_c]
    with _gen.study_chunk(22):
        _studies_on_two_streams(ref, cfgs)


def _studies_on_two_streams(ref, cfgs):
    serial = []
    for cfg in cfgs:
        s = K.StudyStats()
        s.add(cfg, 0, cfg.count)
        serial.append(bytes(s.read()))
    streams = [torch.cuda.Stream() for _ in cfgs]
    stats = [K.StudyStats() for _ in cfgs]
    torch.cuda.synchronize()
    for _ in range(2):  # twice, so the second round reuses pooled scratch and side streams
        for s in stats:
            s.reset()
        for cfg, s, q in zip(cfgs, stats, streams):
            with torch.cuda.stream(q):
                s.add(cfg, 0, cfg.count)
        torch.cuda.synchronize()
        for cfg, s, want in zip(cfgs, stats, serial):
            assert bytes(s.read()) == want, f"concurrent study differs: {K.csv_row(cfg, s.read())}"
    for cfg, s in zip(cfgs[1:], stats[1:]):
        rc, want, msg = refbind.run_batch(ref, cfg.c())
        assert rc == 0, msg
        assert K.csv_row(cfg, s.read()) == refbind.csv_row(ref, cfg.c(), want)


def test_study_and_svd2_share_nothing(cuda, ref):
    """A study on one stream while svd2 batches run on another."""
    cfg = configs.cfg(5, count=(1 << 24) + 17)  # (two chunks at the default 2^24)
    s0 = K.StudyStats()
    s0.add(cfg, 0, cfg.count)
    want_st = bytes(s0.read())
    g = deferring_batch(np.float64, 0xDE01, (1 << 20) + 3)
    gd = dev(g)
    qa, qb = torch.cuda.Stream(), torch.cuda.Stream()
    s1 = K.StudyStats()
    torch.cuda.synchronize()
    with torch.cuda.stream(qa):
        s1.add(cfg, 0, cfg.count)
    with torch.cuda.stream(qb):
        rs = [K.svd2(gd) for _ in range(3)]
    torch.cuda.synchronize()
    assert bytes(s1.read()) == want_st
    want = refbind.svd2(ref, g)
    for r in rs:
        compare_svd(r, want, "svd2 beside a study")
