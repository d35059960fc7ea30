"""pytest plugin: run the reference's own test suite (``gigaqbx``, installed
into the git-ignored ``baseline/_ref`` by ``__graft_entry__.build()``) with
its TSQBX and P2P entry points served by this repository's CUDA backend.

This is INTEGRATION.md sections 1 and 3 in executable form:

* a ``cuda`` backend module = the reference's compiled backend with
  ``ts_accum_laplace``, ``ts_accum_helmholtz``, ``laplace_p2p`` and
  ``helmholtz_p2p`` replaced by ``paper_1811_01110_b200._backend.cuda``
  (the far-field entry points p2m, m2l, ... stay on the CPU core: out of
  scope); it becomes ``gigaqbx._backend.impl`` and every consumer's bound
  ``_impl`` (``tsqbx.py:22``, ``kernels.py:19``, ``driver.py:28``,
  ``expansion.py:22``), and ``get_backend("compiled")`` returns it, so the
  reference's cross-backend tests (test_backends.py) compare it with the
  NumPy backend;
* with ``GQ_GPU_DIRECT=1`` the driver's TS-mode ``direct_stage``
  (driver.py:197-228, a closure inside ``evaluate``) is replaced by one
  ``DirectStage.run`` per list (``paper_1811_01110_b200.direct_stage``): the
  driver module is re-executed from its own source with that function's body
  swapped, nothing on disk is modified.

Calls into the CUDA backend are counted and written to ``$GQ_SWAP_COUNTS``
(JSON) at the end of the session, so the caller can check the GPU path ran.
"""

import json
import os
import sys
import types
from collections import Counter

_COUNTS = Counter()

_GPU_DIRECT_SRC = '''    def direct_stage(stage_name, list_csr):
        if is_ts and _impl is _GQ_CUDA:
            with clock.stage(stage_name):
                if not _gpu_stage:
                    _gpu_stage.append(_GQ_DirectStage(
                        spec, p_qbx, tree, lists.target_boxes, w,
                        source_normals=sn_or_none, qtargets=qtargets,
                        qnormals=qnormals, conv_normals=conv_normals))
                conv_add, qbx_add, n_ts = _gpu_stage[0].run(list_csr)
                _GQ_COUNTS["DirectStage.run"] += 1
                if n_conv:
                    conv_near[:] += conv_add.cpu().numpy()
                qbx_near_val[:] += qbx_add.cpu().numpy()
                counts["ts"] += n_ts
            return
        _cpu_direct_stage(stage_name, list_csr)

    def _cpu_direct_stage(stage_name, list_csr):
'''


def _counted(name, fn):
    def wrapper(*args, **kwargs):
        _COUNTS[name] += 1
        return fn(*args, **kwargs)
    wrapper.__name__ = getattr(fn, "__name__", name)
    return wrapper


def _cuda_backend():
    from gigaqbx._backend import compiled
    from paper_1811_01110_b200._backend import cuda as ours

    mod = types.ModuleType("gigaqbx._backend.cuda")
    for k in dir(compiled):
        if not k.startswith("__"):
            setattr(mod, k, getattr(compiled, k))
    for k in ("ts_accum_laplace", "ts_accum_helmholtz", "laplace_p2p", "helmholtz_p2p"):
        setattr(mod, k, _counted(k, getattr(ours, k)))
    mod.BACKEND_NAME = "cuda"
    return mod


def _patch_driver(drv, cuda):
    import torch  # noqa: F401  (DirectStage needs the CUDA runtime)
    from paper_1811_01110_b200.direct_stage import DirectStage

    src = open(drv.__file__).read()
    head = "    def direct_stage(stage_name, list_csr):\n"
    if src.count(head) != 1:
        raise RuntimeError("driver.direct_stage not found: reference layout changed")
    src = src.replace(head, "    _gpu_stage = []\n" + _GPU_DIRECT_SRC, 1)
    code = compile(src, drv.__file__, "exec")
    drv.__dict__.update(_GQ_DirectStage=DirectStage, _GQ_COUNTS=_COUNTS, _GQ_CUDA=cuda)
    exec(code, drv.__dict__)
    drv._impl = cuda


def pytest_configure(config):
    import gigaqbx._backend as bk

    cuda = _cuda_backend()
    sys.modules["gigaqbx._backend.cuda"] = cuda
    bk.cuda = cuda
    bk.impl = cuda
    bk.BACKEND_NAME = "cuda"
    orig_get = bk.get_backend

    def get_backend(name=None):
        if name in (None, "cuda", "compiled"):
            return cuda
        return orig_get(name)

    bk.get_backend = get_backend
    bk.available_backends = lambda: ["python", "compiled", "cuda"]
    import gigaqbx
    import gigaqbx.driver as drv
    import gigaqbx.expansion as ex
    import gigaqbx.kernels as kn
    import gigaqbx.tsqbx as ts
    for m in (drv, ex, kn, ts):
        m._impl = cuda
    if hasattr(gigaqbx, "BACKEND_NAME"):
        gigaqbx.BACKEND_NAME = "cuda"
    if os.environ.get("GQ_GPU_DIRECT", "0") == "1":
        _patch_driver(drv, cuda)


def pytest_unconfigure(config):
    path = os.environ.get("GQ_SWAP_COUNTS")
    if path:
        with open(path, "w") as f:
            json.dump(dict(_COUNTS), f)
