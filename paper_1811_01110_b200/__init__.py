"""gigaqbx-b200: B200-native target-specific QBX (TSQBX) near-field evaluation.

Drop-in for the TSQBX path of the reference package ``gigaqbx``
(/root/reference/pkg/src/gigaqbx): same entry points (``TsConfig``,
``ts_accumulate``, ``ts_eval``, ``KernelSpec``, geometry/center setup, the
backend protocol) evaluated by hand-written sm_100a CUDA kernels behind a
C ABI (``include/tsqbx.h``), plus the batched ``ts_accumulate_batch`` and the
device near-list builder ``build_near_lists``.
"""

from ._backend import BACKEND_NAME, available_backends, get_backend
from .kernels import Equation, KernelSpec, Variant
from .nearlist import NearLists, build_near_lists
from .p2p import P2PProblem, direct_sum, kernel_value, p2p_rows
from .tsqbx import (PendingPotentials, TsConfig, TsqbxProblem, near_field_potentials,
                    ts_accumulate, ts_accumulate_batch, ts_eval)

__version__ = "0.1.0"

__all__ = [
    "BACKEND_NAME", "available_backends", "get_backend", "Equation", "KernelSpec", "Variant",
    "NearLists", "build_near_lists", "TsConfig", "TsqbxProblem", "ts_accumulate",
    "ts_accumulate_batch", "ts_eval", "near_field_potentials", "PendingPotentials", "P2PProblem", "direct_sum",
    "kernel_value", "p2p_rows", "__version__",
]
