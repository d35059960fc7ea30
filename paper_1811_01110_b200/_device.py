"""Device-buffer plumbing (PyTorch is used only for allocation and streams)."""

from __future__ import annotations

import functools
import inspect

import numpy as np
import torch


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("TSQBX evaluation needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda",
                                                                       torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def on_device(fn):
    """Run ``fn`` with its ``device`` argument as the current CUDA device.

    The C ABI launches on the current device (a stream handle does not name
    one), so every public entry point that takes ``device=`` makes that device
    current for the call; ``device=None`` keeps the current one."""
    sig = inspect.signature(fn)

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        bound = sig.bind(*args, **kwargs)
        dev = require_cuda(bound.arguments.get("device"))
        bound.arguments["device"] = dev
        with torch.cuda.device(dev):
            return fn(*bound.args, **bound.kwargs)

    return wrapper


def on_own_device(fn):
    """Method form of :func:`on_device`: the device is the object's ``dev``."""

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        if self.dev.type != "cuda":          # host-side bookkeeping only (tests)
            return fn(self, *args, **kwargs)
        with torch.cuda.device(self.dev):
            return fn(self, *args, **kwargs)

    return wrapper


@functools.lru_cache(maxsize=None)
def sm_count(index: int) -> int:
    """Multiprocessors of CUDA device ``index`` (cached: the query is not free)."""
    return torch.cuda.get_device_properties(index).multi_processor_count


@functools.lru_cache(maxsize=None)
def _side_stream(index: int) -> torch.cuda.Stream:
    return torch.cuda.Stream(torch.device("cuda", index))


def side_stream(dev: torch.device) -> torch.cuda.Stream:
    """A second stream per device for copies that overlap work on the current one."""
    return _side_stream(dev.index if dev.index is not None else torch.cuda.current_device())


def stream_handle(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def to_device(a, dtype: torch.dtype, dev: torch.device, shape=None) -> torch.Tensor:
    """Contiguous device tensor of `dtype` (copies host arrays; no-op for matching tensors)."""
    if isinstance(a, torch.Tensor):
        # pinned host tensors are copied asynchronously (stream-ordered DMA)
        nb = bool(a.device.type == "cpu" and a.is_pinned() and a.dtype == dtype)
        t = a.to(device=dev, dtype=dtype, non_blocking=nb)
    else:
        np_dtype = {torch.float64: np.float64, torch.int64: np.int64, torch.int32: np.int32,
                    torch.complex128: np.complex128}[dtype]
        arr = np.ascontiguousarray(np.asarray(a, dtype=np_dtype))
        if not arr.flags.writeable:          # e.g. np.broadcast_to views
            arr = arr.copy()
        t = torch.from_numpy(arr).to(device=dev, non_blocking=False)
    t = t.contiguous()
    if shape is not None:
        t = t.reshape(shape)
    return t


def complex_as_f64(w: torch.Tensor) -> torch.Tensor:
    """complex128 (n,) tensor -> interleaved float64 (n, 2) view."""
    return torch.view_as_real(w.contiguous())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
