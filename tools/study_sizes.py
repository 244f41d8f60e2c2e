"""Time one kog_study_batch call per size (config-5 rule) to check that the
chunk pipeline's throughput does not depend on the number of chunks."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_13116_b200 import configs, kogsvd2 as K  # noqa: E402

cfg = configs.cfg(5, count=1 << 31)
ss = K.StudyStats()
for a in (sys.argv[1:] or ["26", "28", "29", "30", "31"]):
    n = int(float(a)) if "." in a or int(a) > 64 else 1 << int(a)
    lg = a
    ss.reset(); ss.add(cfg, 0, 1 << 22); ss.read()
    torch.cuda.synchronize(); t = time.perf_counter()
    ss.reset(); ss.add(cfg, 0, n); ss.read()
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(os.environ.get("KOG2_LIB", "main")[-12:], f"2^{lg}", round(n / dt / 1e6, 1), "M/s", flush=True)
