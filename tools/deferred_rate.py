"""Fraction of matrices the fast path defers (recomputed by k_svd2_list) per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_13116_b200 import capi, configs  # noqa: E402
from paper_2407_13116_b200 import kogsvd2 as K  # noqa: E402

lib = capi.load()
for k in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
    c = configs.cfg(k, count=min(configs.FULL_SIZE[k], 1 << 26))
    g = K.generate(c, 0, c.count)
    torch.cuda.synchronize()
    d0 = lib.kog_svd2_deferred_count()
    K.svd2(g)
    torch.cuda.synchronize()
    print(f"cfg{k}: {lib.kog_svd2_deferred_count() - d0} of {c.count} deferred")
