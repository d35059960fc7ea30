"""The reference's own test suite, run against this repository's CUDA backend.

``__graft_entry__.build()`` installs the unmodified reference package (compiled
core included) and its tests into the git-ignored ``baseline/_ref``; the
plugin ``tests/refswap/gq_cuda_swap.py`` makes ``paper_1811_01110_b200``'s
CUDA backend serve every TSQBX and P2P call of the reference
(``tsqbx.ts_accumulate``/``ts_eval`` through the reference's own ``_prep``,
``kernels.direct_sum``, the driver's ``_ts_accum`` and p2p, and the
cross-backend checks of test_backends.py against the NumPy backend).  With
``GQ_GPU_DIRECT=1`` the driver's TS direct stages run as one
``DirectStage.run`` per list instead, which is
what test_driver.py's mode-equivalence pin (test_driver.py:38-48) then checks.

Pins: test_tsqbx.py:28-157, test_backends.py:47-59,106-137,
test_driver.py:38-48, test_kernels.py.
"""

import json
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
HAVE_REF = os.path.isdir(os.path.join(REF, "gigaqbx")) and os.path.isdir(os.path.join(REF, "tests"))


def _run(files, tmp_path, gpu_direct):
    counts = tmp_path / "counts.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(REPO, "tests", "refswap"), REPO,
                                         env.get("PYTHONPATH", "")])
    env["GQ_SWAP_COUNTS"] = str(counts)
    env["GQ_GPU_DIRECT"] = "1" if gpu_direct else "0"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "gq_cuda_swap", "-p", "no:cacheprovider",
           "--rootdir", REF, "-c", os.devnull] + [os.path.join(REF, "tests", f) for f in files]
    res = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=1500)
    print(res.stdout[-3000:], res.stderr[-2000:])
    assert res.returncode == 0, res.stdout[-3000:]
    m = re.search(r"(\d+) passed", res.stdout)
    return int(m.group(1)) if m else 0, json.loads(counts.read_text())


@pytest.mark.skipif(not HAVE_REF, reason="baseline/_ref not installed (run __graft_entry__.build())")
def test_reference_tsqbx_backends_kernels_through_cuda_backend(tmp_path):
    passed, counts = _run(["test_tsqbx.py", "test_backends.py", "test_kernels.py"], tmp_path,
                          gpu_direct=False)
    print("calls into the CUDA backend:", counts)
    assert passed >= 40
    for k in ("ts_accum_laplace", "ts_accum_helmholtz", "laplace_p2p", "helmholtz_p2p"):
        assert counts.get(k, 0) > 0, k


@pytest.mark.skipif(not HAVE_REF, reason="baseline/_ref not installed (run __graft_entry__.build())")
def test_reference_driver_with_gpu_direct_stages(tmp_path):
    passed, counts = _run(["test_driver.py", "test_backends.py::test_full_pipeline_agreement"],
                          tmp_path, gpu_direct=True)
    print("calls into the CUDA backend:", counts)
    assert passed >= 15
    assert counts.get("DirectStage.run", 0) > 0
