"""Kernel specification types for the TSQBX path.

Mirrors the reference's ``gigaqbx.kernels`` configuration surface
(/root/reference/pkg/src/gigaqbx/kernels.py:26-71): ``Equation``, ``Variant``,
``KernelSpec`` with the same validation and the same variant codes
(``_backend/common.py:27-29``: 0 = S, 1 = S', 2 = D).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

VARIANT_S = 0        # single layer
VARIANT_SPRIME = 1   # target-normal derivative
VARIANT_D = 2        # source-normal derivative (double layer)


class Equation(enum.Enum):
    LAPLACE = "laplace"
    HELMHOLTZ = "helmholtz"


class Variant(enum.Enum):
    SINGLE_LAYER = "s"
    TARGET_NORMAL_DERIV = "sprime"
    SOURCE_NORMAL_DERIV = "d"


_VARIANT_CODE = {
    Variant.SINGLE_LAYER: VARIANT_S,
    Variant.TARGET_NORMAL_DERIV: VARIANT_SPRIME,
    Variant.SOURCE_NORMAL_DERIV: VARIANT_D,
}


@dataclass(frozen=True)
class KernelSpec:
    """Same fields and validation as kernels.py:44-71."""

    equation: Equation = Equation.LAPLACE
    variant: Variant = Variant.SINGLE_LAYER
    helmholtz_k: float | None = None

    def __post_init__(self):
        if self.equation is Equation.HELMHOLTZ:
            if self.helmholtz_k is None or self.helmholtz_k <= 0:
                raise ValueError("Helmholtz requires helmholtz_k > 0")
        elif self.helmholtz_k is not None:
            raise ValueError("helmholtz_k only valid for the Helmholtz equation")

    @classmethod
    def coerce(cls, spec) -> "KernelSpec":
        """This type from any spec with the reference's fields (e.g. a
        ``gigaqbx.kernels.KernelSpec`` handed over by the reference's driver):
        equal enum values, the same ``helmholtz_k``."""
        if isinstance(spec, cls):
            return spec
        return cls(equation=Equation(spec.equation.value), variant=Variant(spec.variant.value),
                   helmholtz_k=spec.helmholtz_k)

    @property
    def is_laplace(self) -> bool:
        return self.equation is Equation.LAPLACE

    @property
    def variant_code(self) -> int:
        return _VARIANT_CODE[self.variant]

    @property
    def needs_source_normals(self) -> bool:
        return self.variant is Variant.SOURCE_NORMAL_DERIV

    @property
    def needs_target_normals(self) -> bool:
        return self.variant is Variant.TARGET_NORMAL_DERIV
