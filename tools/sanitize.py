"""Driver for compute-sanitizer (memcheck / racecheck / synccheck): one small
invocation of every kernel family of libkog2.so — the unit kernels, the
svd2 fast/list pair on inputs with many deferred lanes, the general kernel
(non-default Options), svd2_ext / metrics, the generator, a phased study over
two chunks, a lasv2 study, the host pipeline, and two svd2 batches plus two
studies in flight on two streams at once.  Sizes are small: the sanitizer
slows kernels down 10-100x.

  compute-sanitizer --tool memcheck --leak-check full python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_13116_b200 import capi, configs  # noqa: E402
from paper_2407_13116_b200 import kogsvd2 as K  # noqa: E402
from tests import _gen  # noqa: E402


def deferring(dt, seed, n):
    g = _gen.matrices(dt, seed, n)
    mask = (_gen.draws(seed + 1, n, 0) % np.uint64(16)).astype(np.int64)
    sel = (_gen.draws(seed + 1, n, 1) % np.uint64(4)) == 0
    for k, bit in enumerate((1, 4, 2, 8)):
        g[k][sel & ((mask & bit) == 0)] = 0
    return torch.from_numpy(g).cuda()


def main():
    torch.cuda.set_device(0)
    n = 1 << 14
    for dt in (np.float64, np.float32):
        g = deferring(dt, 0x5A1, n)
        K.svd2(g)
        K.svd2(g, K.Options(hypot_is_cr=False, ominus_for_d=True, wide_channel=1))
        K.hypot_cr(g[0], g[1])
        K.split(g[0])
        K.tan_from_double_angle(g[0])
        K.sec_from_tan(g[1])
        K.classify_prescale(g)
        K.urv15(g)
        K.svd2_ext(g[:, :2048].contiguous())
        K.metrics(g[:, :2048].contiguous())
        K.lasv2(g[0].abs() + 1, g[1], g[3].abs() + 1)
        K.svd2_host(g.cpu().pin_memory())
    # studies: phased kog (two chunks + tail would be 2^22+; a small count runs one chunk), lasv2
    for cfg in (configs.cfg(5, count=40000), configs.cfg(4, count=20000),
                K.RunConfig(shape=capi.SHAPE_TRI, regime=capi.REGIME_BULLET, count=20000, seed=3,
                            routine=capi.ROUTINE_LASV2)):
        st = K.run_batch(cfg)
        print(K.csv_row(cfg, st))
    # concurrency: two svd2 batches and two studies in flight on two streams
    qa, qb = torch.cuda.Stream(), torch.cuda.Stream()
    ga, gb = deferring(np.float64, 0x5A2, n), deferring(np.float64, 0x5A3, n + 77)
    sa, sb = K.StudyStats(), K.StudyStats()
    torch.cuda.synchronize()
    with torch.cuda.stream(qa):
        ra = K.svd2(ga)
        sa.add(configs.cfg(5, count=30000), 0, 30000)
    with torch.cuda.stream(qb):
        rb = K.svd2(gb)
        sb.add(configs.cfg(3, count=30000), 1000, 30000)
    torch.cuda.synchronize()
    print("deferred lanes so far:", capi.load().kog_svd2_deferred_count(), int(ra["flags"].numel() + rb["flags"].numel()))
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
