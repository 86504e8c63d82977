"""B200-native (sm_100a) per-Newton linear-solve hot path of StiffGIPC
(arXiv 2411.06224): Hessian assembly (sort + segmented / two-level
reduction), MAS preconditioner construction and the fused PCG loop, behind
the C-ABI in include/adipc_gpu.h and the reference's interface in api.py."""
from .api import *  # noqa: F401,F403
from .context import Context, PcgResult, default_context  # noqa: F401

__version__ = "0.1.0"
