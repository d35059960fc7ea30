"""near_field_potentials into a pinned host buffer written directly by the
evaluation kernel (zero-copy through unified addressing, ``_direct_out``):
same potentials as the device-buffer path, validation still raises."""

import numpy as np
import pytest
import torch

from paper_1811_01110_b200 import configs, near_field_potentials

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,preset", [("c1", "dense"), ("c3", "literal"), ("c5", "literal")])
def test_direct_pinned_output(monkeypatch, name, preset):
    kw = {"n": 32768, "spheres": 2} if name == "c5" else ({"n": 32768} if name == "c3" else {})
    case = configs.make_case(name, preset, **kw)
    args = (case.cfg, case.sources, case.weights, case.centers, case.near_radii, case.targets)
    monkeypatch.setenv("GIGAQBX_DIRECT_OUT", "0")
    ref = near_field_potentials(*args, tgt_ptr=case.tgt_ptr)
    out = torch.full((case.n_targets,), complex("nan"), dtype=torch.complex128).pin_memory()
    monkeypatch.setenv("GIGAQBX_DIRECT_OUT", "1")
    got = near_field_potentials(*args, tgt_ptr=case.tgt_ptr, out=out)
    assert got is out
    assert np.array_equal(out.numpy(), ref)


def test_direct_pinned_output_validation(monkeypatch):
    case = configs.make_case("c1", "literal")
    tgt = case.targets.copy()
    tgt[10] = case.centers[10] + 10.0 * (tgt[10] - case.centers[10])
    out = torch.empty(case.n_targets, dtype=torch.complex128).pin_memory()
    monkeypatch.setenv("GIGAQBX_DIRECT_OUT", "1")
    with pytest.raises(ValueError, match="separation violation"):
        near_field_potentials(case.cfg, case.sources, case.weights, case.centers,
                              case.near_radii, tgt, out=out)
