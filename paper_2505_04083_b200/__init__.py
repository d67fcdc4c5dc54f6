"""B200-native Plexus 3D-parallel GCN hot path (arXiv 2505.04083).

The product is libplexus_b200.so (paper_2505_04083_b200/csrc, sm_100a
kernels behind the C ABI in include/plexus_b200.h). This package is the
host-side mirror of the reference's plexuskit API over CUDA tensors.
"""

from . import layout  # noqa: F401  (pure host logic; importable without the .so)
from ._capi import LIB_PATH, ContractError, TrainingError, lib  # noqa: F401

__all__ = ["lib", "LIB_PATH", "ContractError", "TrainingError", "layout"]
