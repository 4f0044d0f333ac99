"""B200-native (sm_100a) random-tree Monte Carlo for u_t = DΔu + f(u)
(arXiv:2402.06491, Strategy A + order binning + [L/M] Padé).

The product is the C-ABI library ``librt.so`` (include/rt.h); ``rt`` is its
ctypes binding.  Build with ``python -m paper_2402_06491_b200.build``.
"""
from . import rt  # noqa: F401
from .rt import Estimator, finalize, pade, pade_host, pdd_nodes, philox  # noqa: F401

__all__ = ["rt", "Estimator", "finalize", "pade", "pade_host", "pdd_nodes", "philox"]
