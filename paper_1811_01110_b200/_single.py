"""The reference's per-call protocol on the GPU: one (center, target) over a
source batch per call (``_core.ts_accum_*``, _core.pyx:205, :310, and
``tsqbx.ts_accumulate``, tsqbx.py:68-80).

A batch of one would pay for device allocations, several launches and
several synchronisations (~0.27 ms per call).  This path keeps one pinned
staging buffer and one device buffer per device: the inputs are packed on the
host straight into the layout the kernel reads, and ``tsqbx_eval_one`` does
one H2D copy, one launch (``one_kernel``: reference operation order, exact
``_prep`` predicate when validating), one D2H copy of {Re, Im, key} and a
stream synchronisation.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _device as dv
from . import _lib

_ctx: dict = {}
_ctx_lock = threading.Lock()


class _OneCall:
    def __init__(self, dev: torch.device):
        self.dev = dev
        self.cap = 0
        self.lock = threading.Lock()
        # a private stream: the inputs come from the host and the call
        # synchronises it, so no ordering with the caller's streams is needed,
        # and its handle is looked up once instead of per call
        self.stream = torch.cuda.Stream(dev)
        self.stream_ptr = self.stream.cuda_stream
        self.fn = _lib.load().tsqbx_eval_one
        self.staging = _lib.load().tsqbx_one_staging_doubles
        self.res = torch.zeros(4, dtype=torch.float64).pin_memory()
        self.res_np = self.res.numpy()
        self.res_ptr = self.res.data_ptr()
        self._grow(4096)

    def _grow(self, nd: int) -> None:
        cap = max(nd, 2 * self.cap)
        self.host = torch.zeros(cap, dtype=torch.float64).pin_memory()
        self.host_np = self.host.numpy()
        self.host_ptr = self.host.data_ptr()
        self.devbuf = torch.empty(cap + 8, dtype=torch.float64, device=self.dev)
        self.devbuf_ptr = self.devbuf.data_ptr()
        self.devbuf_len = int(self.devbuf.numel())
        self.cap = cap

    def run(self, equation: int, variant: int, k: float, p: int, sources, weights, snormals,
            center, target, tnormal, validate: bool, r_ref: float = 0.0):
        """(value, key): key = _lib.ERR_KEY_NONE or (kind << 31) | position."""
        n = sources.shape[0]
        with_nrm = variant == 2
        nd = int(self.staging(n, int(with_nrm)))
        with self.lock:
            if nd > self.cap:
                self._grow(nd)
            h = self.host_np
            h[:16] = 0.0
            h[0:3] = center
            h[3:6] = target
            if tnormal is not None:
                h[6:9] = tnormal
            h[9] = r_ref
            sp = h[16:16 + 4 * n].reshape(n, 4)
            sp[:, :3] = sources
            sp[:, 3] = weights.real
            h[16 + 4 * n:16 + 5 * n] = weights.imag
            off = 16 + 4 * n + ((n + 3) & ~3)
            h[16 + 5 * n:off] = 0.0
            if with_nrm:
                sn = h[off:off + 4 * n].reshape(n, 4)
                sn[:, :3] = snormals
                sn[:, 3] = 0.0
            rc = self.fn(equation, variant, float(k), int(p), self.host_ptr, n,
                         _lib.FLAG_VALIDATE if validate else 0, self.devbuf_ptr,
                         self.devbuf_len, self.res_ptr, self.stream_ptr)
            if rc:
                _lib.check(rc, "tsqbx_eval_one")
            value = complex(self.res_np[0], self.res_np[1])
            key = int(self.res_np[2:3].view(np.int64)[0])
        return value, key


def one_call(equation: int, variant: int, k: float, p: int, sources, weights, snormals, center,
             target, tnormal, validate: bool = False, r_ref: float = 0.0):
    idx = torch.cuda.current_device() if torch.cuda.is_available() else -1
    ctx = _ctx.get(idx)
    if ctx is None:
        dev = dv.require_cuda()
        with _ctx_lock:
            ctx = _ctx.get(idx)
            if ctx is None:
                ctx = _ctx[idx] = _OneCall(dev)
    return ctx.run(equation, variant, k, p, sources, weights, snormals, center, target, tnormal,
                   validate, r_ref)
