"""Backend selection, mirroring the reference protocol (_backend/__init__.py:7-41).

The reference chooses between a compiled Cython core and a NumPy twin.  Here
there is exactly one backend -- ``cuda``, the sm_100a C-ABI library -- and no
CPU fallback: importing works anywhere, calling it needs a B200.
"""

from . import cuda as impl

BACKEND_NAME = impl.BACKEND_NAME


def get_backend(name=None):
    """Return a backend module by name (only 'cuda' exists)."""
    if name in (None, BACKEND_NAME):
        return impl
    raise ValueError(f"unknown backend {name!r} (available: {available_backends()})")


def available_backends():
    return [BACKEND_NAME]
