"""B200-native batched LDPC belief-propagation decoder (arXiv 2507.03509 hot path).

Public API mirrors the reference ``etdec`` decoder; see ``decoder.py``.
"""
from .decoder import *  # noqa: F401,F403
from .decoder import __all__ as _dec_all
from .configs import WORKLOADS, Workload, CODE_SEED, FRAME_SEED  # noqa: F401

__all__ = list(_dec_all) + ["WORKLOADS", "Workload", "CODE_SEED", "FRAME_SEED"]
