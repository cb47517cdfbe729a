"""Backend selection for the per-pixel kernels.

Mirrors ``floodstream.backends`` (/root/reference/pkg/src/floodstream/backends.py:21-47):
``select_backend(name)``, the import-time module global ``kernels`` and
``available_backends()``, driven by the same ``FLOODSTREAM_BACKEND`` variable.

The only product backend is ``"cuda"`` (libfloodstream, sm_100a); ``"auto"`` resolves
to it.  The reference's CPU backends (``"numpy"``, ``"cython"``) are deliberately not
part of this framework — asking for one raises instead of silently running on the
host, exactly like the reference raises when a forced backend is missing
(backends.py:27-32).  The CPU restatement used to check results lives in ``oracle/``
and is test infrastructure only.
"""

from __future__ import annotations

import os

_CPU_BACKENDS = ("numpy", "cython")


def _load_cuda():
    from . import _kernels_cuda

    return _kernels_cuda


def select_backend(name: str | None = None):
    """Return the kernel module for ``name`` (default: env var, then auto)."""
    if name is None:
        name = os.environ.get("FLOODSTREAM_BACKEND", "auto")
    if name in ("cuda", "auto"):
        return _load_cuda()
    if name in _CPU_BACKENDS:
        raise RuntimeError(
            f"backend {name!r} is a CPU implementation of the reference package; this "
            "framework runs the overlap path on the GPU only (use backend 'cuda')"
        )
    raise ValueError(f"unknown backend {name!r}")


kernels = select_backend()


def available_backends() -> dict:
    """Importable kernel backends, keyed by name."""
    return {"cuda": _load_cuda()}
