"""Small driver for ncu: generate one config on device and run svd2 `iters`
times (the kernel under profile is k_svd2)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2407_13116_b200 import configs  # noqa: E402
from paper_2407_13116_b200 import kogsvd2 as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--count", type=int, default=1 << 24)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--study", action="store_true", help="profile the fused study kernel instead")
a = ap.parse_args()
cfg = configs.cfg(a.config, count=a.count)
if a.study:
    s = K.StudyStats()
    for _ in range(a.iters):
        s.reset()
        s.add(configs.cfg(5, count=a.count), 0, a.count)
    print(K.csv_row(configs.cfg(5, count=a.count), s.read()))
else:
    g = K.generate(cfg, 0, a.count)
    out = K.empty_result(a.count, g.dtype, g.device)
    for _ in range(a.iters):
        K.svd2(g, out=out)
    torch.cuda.synchronize()
    print("ok", a.count)
