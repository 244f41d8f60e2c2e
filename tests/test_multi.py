"""The multi-GPU study from the C++ side: contiguous shards
(kog_study_shard), the packed int64 stats vector (kog_stats_pack/unpack) and
one MAX all-reduce, merged in rank order (ErrorStats::merge,
harness.hpp:96-105).

CPU (gloo, world size 2): each rank runs the REFERENCE's own run_one loop on
its real shard of a study (oracle/_ref run_range, harness.hpp:190-271), the
shard stats go through the library's pack -> MAX all-reduce -> unpack, and the
result equals the reference's single-process run_batch over the whole range.
GPU: kog_study_multi and the one-process-per-GPU NCCL path (kog_nccl_* +
kog_study_allreduce) give kog_run_batch's stats byte for byte."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

from oracle import refbind
from paper_2407_13116_b200 import capi, configs, dist
from paper_2407_13116_b200 import kogsvd2 as K

STUDIES = [configs.cfg(5, count=3 * (1 << 13) + 77),
           K.RunConfig(shape=capi.SHAPE_GEN, regime=capi.REGIME_BULLET, count=20000, seed=0x77),
           K.RunConfig(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=9000, seed=0x1234ABCD,
                       routine=capi.ROUTINE_LASV2, single_precision=True)]


def _csv(lib, cfg, st) -> str:
    return refbind.csv_row(lib, cfg.c(), st)


def test_pack_unpack_roundtrip_and_fail_key():
    st = K.new_stats()
    st.reG, st.reV = 3e-16, 0.0
    st.max_kappa2 = capi.kog_extfloat(-5000, 1.25, -1e-17)
    st.max_kappa2_index = (1 << 40) + 3
    st.path[4], st.t2p[5], st.prescale_inexact = (1 << 35) + 1, 7, 9
    st.fail_key = 4 * 12345 + 2
    for world in (1, 3):
        for rank in range(world):
            buf = dist.pack(st, rank, world)
            assert buf.size == 7 + 46 * world and (buf >= -1).all()
            assert bytes(dist.unpack(buf, world)) == bytes(st)
    # MAX over ranks picks the lowest failure key; no failure is UINT64_MAX
    a, b = K.new_stats(), K.new_stats()
    a.fail_key, b.fail_key = 4 * 99 + 1, 0xFFFFFFFFFFFFFFFF
    red = np.maximum(dist.pack(a, 0, 2), dist.pack(b, 1, 2))
    assert dist.unpack(red, 2).fail_key == 4 * 99 + 1
    assert dist.unpack(dist.pack(b, 0, 1), 1).fail_key == 0xFFFFFFFFFFFFFFFF


def _worker(rank, world, port, q):
    import torch.distributed as tdist

    from oracle import refbind as rb
    from paper_2407_13116_b200 import dist as kd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    lib = rb.ref()
    rows = []
    for cfg in STUDIES:
        lo, hi = kd.shard(cfg.count, rank, world)
        rc, st, msg = rb.run_range(lib, cfg.c(), lo, hi - lo)
        assert rc == 0, msg
        out = kd.allreduce_stats(st)
        rows.append((bytes(out), rb.csv_row(lib, cfg.c(), out)))
    q.put((rank, rows))
    tdist.destroy_process_group()


@pytest.mark.skipif(not refbind.have_ref(), reason="oracle/_ref not built")
def test_gloo_world2_real_shards_equal_whole_study():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == res[1]
    lib = refbind.ref()
    for cfg, (raw, row) in zip(STUDIES, res[0]):
        rc, whole, msg = refbind.run_batch(lib, cfg.c())
        assert rc == 0, msg
        assert row == _csv(lib, cfg, whole)
        got = capi.kog_stats.from_buffer_copy(raw)
        assert list(got.path) == list(whole.path) and list(got.t2p) == list(whole.t2p)
        assert (got.max_kappa2.e, got.max_kappa2.hi, got.max_kappa2.lo) == \
               (whole.max_kappa2.e, whole.max_kappa2.hi, whole.max_kappa2.lo)


@pytest.mark.gpu
def test_study_multi_equals_run_batch(cuda):
    """kog_study_multi over every visible device (shards + one NCCL
    all-reduce) == kog_run_batch, for several studies."""
    import torch
    lib = capi.load()
    if not lib.kog_nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    n = torch.cuda.device_count()
    for cfg in STUDIES + [configs.cfg(5, count=(1 << 23) + 4099)]:
        want = K.run_batch(cfg)
        for ndev in sorted({1, n}):
            got = capi.kog_stats()
            secs = C.c_double()
            capi.check(lib.kog_study_multi(C.byref(cfg.c()), None, ndev, C.byref(got), C.byref(secs)))
            assert K.csv_row(cfg, got) == K.csv_row(cfg, want)
            got.max_kappa2_index = want.max_kappa2_index = 0
            assert bytes(got) == bytes(want)
            assert secs.value > 0


@pytest.mark.gpu
def test_study_multi_abort_message(cuda):
    """A failing matrix aborts the multi-device study with run_batch's text."""
    lib = capi.load()
    if not lib.kog_nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    cfg = K.RunConfig(regime=capi.REGIME_SIGMA, varsigma=0, count=10)
    assert lib.kog_study_multi(C.byref(cfg.c()), None, 1, C.byref(capi.kog_stats()), None) == capi.KOG_ERR_ARG


@pytest.mark.gpu
def test_nccl_per_process_path_world1(cuda):
    """The one-process-per-GPU path bench.py uses under torchrun: id through
    torch.distributed, communicator and MAX all-reduce from the C++ side."""
    import socket

    import torch
    import torch.distributed as tdist
    lib = capi.load()
    if not lib.kog_nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        torch.cuda.set_device(0)
        nc = dist.NcclStats()
        cfg = configs.cfg(5, count=1 << 20)
        st = K.run_batch(cfg)
        out = nc.allreduce(st)
        nc.close()
        assert bytes(out) == bytes(st)
    finally:
        tdist.destroy_process_group()
