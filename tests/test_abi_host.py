"""CPU: the C-ABI library loads without a GPU and exports every symbol that
include/kog2.h declares; host-side logic (stats merge, CSV formatting,
validation, the multi-GPU stats all-reduce) is exercised without a device."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2407_13116_b200 import capi, dist
from paper_2407_13116_b200 import kogsvd2 as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols() -> list[str]:
    src = open(os.path.join(ROOT, "include", "kog2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kog_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(capi.PROTOTYPES), set(names) - set(capi.PROTOTYPES)


def test_version_and_no_device_error(lib):
    assert b"sm_100a" in lib.kog_version()
    assert lib.kog_launch_count() == 0 or lib.kog_launch_count() > 0


def test_csv_header_and_validation(lib):
    assert K.csv_header() == "precision,shape,regime,varsigma,count,seed,routine,reG,reS1,reS2,reU,reV,maxKappa2"
    K.validate(K.RunConfig(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=10))
    for bad in (K.RunConfig(shape=capi.SHAPE_GEN, routine=capi.ROUTINE_LASV2, count=10),
                K.RunConfig(regime=capi.REGIME_SIGMA, varsigma=0),
                K.RunConfig(regime=capi.REGIME_SIGMA, varsigma=5000),
                K.RunConfig(regime=capi.REGIME_RANGED, elo=5, ehi=1)):
        with pytest.raises(ValueError):
            K.validate(bad)


def _stats(**kw) -> capi.kog_stats:
    st = K.new_stats()
    for k, v in kw.items():
        if k == "kappa":
            st.max_kappa2 = capi.kog_extfloat(*v[:3])
            st.max_kappa2_index = v[3]
        elif k in ("t2p", "path"):
            for i, x in enumerate(v):
                getattr(st, k)[i] = x
        else:
            setattr(st, k, v)
    return st


def test_csv_row_formatting_matches_reference_conventions():
    """csv_row (harness.hpp:290-317): shortest round-trip doubles, the
    extended decimal for kappa outside the double range, 'inf'."""
    cfg = K.RunConfig(shape=capi.SHAPE_GEN, regime=capi.REGIME_CIRC, count=1048576, seed=0xC0FFEE)
    st = _stats(reG=5.262556799095865e-16, reS1=4.469753940626907e-16, reS2=5.475477442600766e-16,
                reU=4.740088882553483e-16, reV=4.726642799363624e-16, kappa=(23, 1.730020198378564, 0.0, 5))
    row = K.csv_row(cfg, st)
    assert row.startswith("double,gen,circ,0,1048576,0000000000c0ffee,kog,5.262556799095865e-16,")
    assert row.split(",")[-1] == repr(1.730020198378564 * 2 ** 23)
    st2 = _stats(reS2=1.0, kappa=(4042, 1.5, 0.0, 1))
    last = K.csv_row(cfg, st2).split(",")
    assert last[9] == "1" and last[-1] == "8.6962843710554552e+1216"  # 1.5 * 2^4042
    st3 = _stats(kappa_inf=1)
    assert K.csv_row(cfg, st3).endswith(",inf")
    from oracle import refbind
    if refbind.have_ref():  # byte-identical to the reference's csv_row on the same stats
        for st in (st, st2, st3, _stats(kappa=(-1500, 1.25, 1e-30, 0)), _stats(reG=float("inf"))):
            assert K.csv_row(cfg, st) == refbind.csv_row(refbind.ref(), cfg.c(), st)


def test_stats_merge_semantics():
    """ErrorStats::merge (harness.hpp:96-105): fmax, OR, ext_cmp max with the
    earlier index winning ties, counter sums, lowest failure key."""
    a = _stats(reG=1e-16, reS1=3e-16, kappa=(10, 1.5, 0.0, 7), t2p=[1, 2, 3, 0, 0, 5, 0], fail_key=2**64 - 1)
    b = _stats(reG=2e-16, reS1=1e-16, kappa=(10, 1.5, 0.0, 3), t2p=[1, 1, 1, 1, 1, 1, 1], kappa_inf=1, fail_key=41)
    m = K.merge_stats(K.merge_stats(K.new_stats(), a), b)
    assert (m.reG, m.reS1) == (2e-16, 3e-16)
    assert m.max_kappa2_index == 3 and m.kappa_inf == 1 and m.fail_key == 41
    assert list(m.t2p) == [2, 3, 4, 1, 1, 6, 1]
    c = _stats(kappa=(11, 1.0, 0.0, 99))
    assert K.merge_stats(m, c).max_kappa2_index == 99


def test_dist_pack_unpack_roundtrip():
    parts = [_stats(reG=1e-16 * (r + 1), reV=5e-17, kappa=(20 + r, 1.25, -1e-20, 100 * r), path=[r, 1, 2, 3, 4, 5, 6],
                    tanpsi_inf=r, fail_key=(2**64 - 1) if r != 2 else 4 * 77 + 1) for r in range(4)]
    bufs = [dist.pack(p, r, 4) for r, p in enumerate(parts)]
    red = np.maximum.reduce(bufs)  # what the MAX all-reduce computes
    got = dist.unpack(red, 4)
    want = K.new_stats()
    for p in parts:
        K.merge_stats(want, p)
    assert bytes(got) == bytes(want)


def _worker(rank, world, port, q):
    import torch.distributed as tdist

    from paper_2407_13116_b200 import dist as kd
    from paper_2407_13116_b200 import kogsvd2 as KK

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    st = KK.new_stats()
    st.reG = 1e-16 * (rank + 1)
    st.max_kappa2 = capi.kog_extfloat(30 - rank, 1.5, 0.0)
    st.max_kappa2_index = 1000 + rank
    st.path[4] = 10 + rank
    out = kd.allreduce_stats(st)
    q.put((rank, bytes(out)))
    tdist.destroy_process_group()


def test_gloo_world2_stats_allreduce():
    """The N>1 path: per-rank stats combined by one MAX all-reduce (gloo on
    CPU here; NCCL on the GPU box) equal the single-process merge."""
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
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == res[1]
    st = capi.kog_stats.from_buffer_copy(res[0])
    assert st.reG == 2e-16 and st.max_kappa2.e == 30 and st.max_kappa2_index == 1000 and st.path[4] == 21


def test_shard_partition_covers_range():
    for count in (0, 1, 7, 2**31):
        for world in (1, 2, 3, 8):
            spans = [dist.shard(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
