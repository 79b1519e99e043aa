"""paper_2602_15917_b200 -- B200-native (sm_100a) ROI extraction hot path of ROIX-Comp (arXiv 2602.15917).

Public API:
  * ``_lib``     the ctypes binding of libroix (same names as include/roix.h)
  * ``Pipeline`` / ``run``   the whole path on one GPU
  * ``sharded``  the z-slab sharded path over torch.distributed (NCCL)
"""
from . import _lib  # noqa: F401
from .pipeline import Pipeline, Result, run, unpack_bits  # noqa: F401
