"""Backend seam: the B200 "cuda" backend registered where the reference registers
"numba" and "numpy" (reference _backend.py:24-66).

There is exactly one backend. It runs the hand-written sm_100a kernels in
liblwb200.so and has no CPU fallback: when the library or a CUDA device is
missing, calls raise :class:`BackendUnavailable` instead of computing on the
host. ``LWB200_BACKEND`` (or ``LANEWORK_BACKEND=cuda``) may name it explicitly.
"""

from __future__ import annotations

import os
from contextlib import contextmanager

from ._lib import BackendUnavailable

ENV_VAR = "LWB200_BACKEND"
_BACKENDS = ("cuda",)
# reference name (_backend.py:17-22): there is no numba CPU backend in this package
NUMBA_AVAILABLE = False


def _resolve_default() -> str:
    value = os.environ.get(ENV_VAR, "").strip().lower()
    if value in ("", "auto", "cuda"):
        return "cuda"
    raise ValueError(f"unrecognized {ENV_VAR}={value!r}; the only backend is 'cuda'")


_active = _resolve_default()


def backend_name() -> str:
    return _active


def cuda_active() -> bool:
    return _active == "cuda"


def numba_active() -> bool:
    """Reference-compatible query; the numba CPU backend does not exist here."""
    return False


def cuda_available() -> bool:
    """True when liblwb200.so loads and a CUDA device is visible."""
    try:
        import torch

        if not torch.cuda.is_available():
            return False
        from . import _lib

        _lib.load()
        return True
    except (ImportError, BackendUnavailable):
        return False


_ready = False


def require_cuda() -> None:
    """Raise BackendUnavailable unless the library and a CUDA device are usable
    (checked once; later calls are a flag test on the hot path)."""
    global _ready
    if _ready:
        return
    if _active != "cuda":  # pragma: no cover - only one backend exists
        raise BackendUnavailable(f"backend {_active!r} is not the cuda backend")
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("the cuda backend needs a visible CUDA device; there is no CPU fallback")
    from . import _lib

    _lib.load()
    _ready = True


@contextmanager
def use_backend(name: str):
    """Run a block under an explicit backend (only "cuda" exists)."""
    global _active
    if name not in _BACKENDS:
        raise ValueError(f"unknown backend {name!r}; expected one of {_BACKENDS}")
    previous = _active
    _active = name
    try:
        yield
    finally:
        _active = previous
