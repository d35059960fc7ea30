"""Host-side behaviour of the public API that needs no GPU: argument checks in
the reference's order (tsqbx.py:38-65, kernels.py:44-71)."""

import numpy as np
import pytest

from paper_1811_01110_b200 import KernelSpec, TsConfig, ts_accumulate
from paper_1811_01110_b200.kernels import Equation, Variant

D = KernelSpec(variant=Variant.SOURCE_NORMAL_DERIV)
SP = KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=2.0, variant=Variant.TARGET_NORMAL_DERIV)


def test_geometry_errors_precede_missing_normals():
    # _prep checks coincidence, then separation, then the normals
    with pytest.raises(ValueError, match="source 1 coincides"):
        ts_accumulate(TsConfig(D, 4), [[1.0, 0, 0], [0, 0, 0]], [1, 1], np.zeros(3),
                      [0.1, 0, 0])
    with pytest.raises(ValueError, match="separation violation for source 0"):
        ts_accumulate(TsConfig(SP, 4), [[0.1, 0, 0]], [1], np.zeros(3), [0.5, 0, 0])


def test_missing_normals_and_empty_batches():
    with pytest.raises(ValueError, match="double-layer variant requires source normals"):
        ts_accumulate(TsConfig(D, 4), np.zeros((0, 3)), [], np.zeros(3), np.zeros(3))
    with pytest.raises(ValueError, match="S' variant requires a target normal"):
        ts_accumulate(TsConfig(SP, 4), [[0, 0, 2.0]], [1], np.zeros(3), [0.1, 0, 0])
    assert ts_accumulate(TsConfig(KernelSpec(), 4), np.zeros((0, 3)), [], np.zeros(3),
                         np.zeros(3)) == 0


def test_kernelspec_validation():
    # kernels.py:50-55
    with pytest.raises(ValueError, match="Helmholtz requires"):
        KernelSpec(equation=Equation.HELMHOLTZ)
    with pytest.raises(ValueError, match="only valid for the Helmholtz"):
        KernelSpec(helmholtz_k=1.0)
    with pytest.raises(ValueError, match="nonnegative"):
        TsConfig(KernelSpec(), -1)


def test_row_split_choice(monkeypatch):
    from paper_1811_01110_b200.tsqbx import pick_split
    monkeypatch.delenv("GIGAQBX_SPLIT", raising=False)
    assert pick_split(12.0, 262144, False) == 1          # literal rows: never split
    assert pick_split(201.0, 262144, False) == 2         # dense, several waves
    assert pick_split(201.0, 4096, True) == 4            # dense, under one wave
    # 200 k rows: 1.76 waves of 3 CTAs/SM, 1.32 waves of 4 (uniform target runs)
    assert pick_split(201.0, 200000, False) == 2
    assert pick_split(201.0, 200000, False, uniform=True) == 4
    monkeypatch.setenv("GIGAQBX_SPLIT", "1")
    assert pick_split(201.0, 262144, False) == 1


def test_kernel_value_checks_before_the_gpu():
    """kernel_value (kernels.py:83-111) raises the reference's errors from the
    host-side checks, before any device work (so these run without a GPU)."""
    from paper_1811_01110_b200 import Equation, KernelSpec, Variant, kernel_value
    with pytest.raises(ValueError, match="singular point: target coincides with source"):
        kernel_value(KernelSpec(), np.ones(3), np.ones(3))
    with pytest.raises(ValueError, match="requires a source normal"):
        kernel_value(KernelSpec(variant=Variant.SOURCE_NORMAL_DERIV), np.zeros(3), np.ones(3))
    with pytest.raises(ValueError, match="requires a target normal"):
        kernel_value(KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=1.0,
                                variant=Variant.TARGET_NORMAL_DERIV), np.zeros(3), np.ones(3))
    with pytest.raises(ValueError, match="source normal must be unit length"):
        kernel_value(KernelSpec(variant=Variant.SOURCE_NORMAL_DERIV), np.array([1.0, 0, 0]),
                     np.zeros(3), source_normal=np.array([0.0, 0, 2.0]))


def test_kernel_spec_coerce_from_foreign_spec():
    # the reference driver hands its own KernelSpec type to DirectStage / TsConfig
    import enum
    from types import SimpleNamespace

    from paper_1811_01110_b200.kernels import Equation, KernelSpec, Variant

    class Eq(enum.Enum):
        HELMHOLTZ = "helmholtz"

    class Va(enum.Enum):
        D = "d"

    foreign = SimpleNamespace(equation=Eq.HELMHOLTZ, variant=Va.D, helmholtz_k=2.5)
    spec = KernelSpec.coerce(foreign)
    assert spec == KernelSpec(Equation.HELMHOLTZ, Variant.SOURCE_NORMAL_DERIV, 2.5)
    assert KernelSpec.coerce(spec) is spec
    from paper_1811_01110_b200 import TsConfig
    assert TsConfig(foreign, 4).spec == spec
