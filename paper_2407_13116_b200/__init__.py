"""kog2 — B200-native batched enhanced 2x2 Kogbetliantz SVD (arxiv 2407.13116).

The product is libkog2.so (sm_100a kernels behind the C-ABI in include/kog2.h);
`kogsvd2` mirrors the reference's kogsvd2 API over it for Python callers and
`configs` names the BASELINE workloads.
"""
from . import capi  # noqa: F401

__all__ = ["capi", "kogsvd2", "configs"]
