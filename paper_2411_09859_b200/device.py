"""Device-memory plumbing (torch is used only for allocation and streams).

Matrices cross the C ABI as (device pointer, leading dimension) of a
column-major buffer.  A column-major torch tensor is one whose ``stride(0)``
is 1 (e.g. ``buf.t()`` of a row-major ``buf``).
"""

from __future__ import annotations

import numpy as np

from . import _capi

_WS = {}


def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise _capi.NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    _capi.load()
    return t


def stream_ptr(stream=None):
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return s.cuda_stream


def workspace(nbytes, device=None, stream=None):
    """Grow-only scratch buffer (uint8 tensor), one per (device, stream).

    Calls enqueued on different streams never share scratch.  When a buffer
    grows, the old one is handed back to the caching allocator only after the
    work already queued on its stream has finished (``record_stream``).
    """
    t = torch()
    if stream is not None:
        dev = stream.device
    else:
        dev = t.device("cuda", t.cuda.current_device() if device is None else device)
    with t.cuda.device(dev):
        st = stream if stream is not None else t.cuda.current_stream(dev)
        key = (dev, st.cuda_stream)
        buf = _WS.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                buf.record_stream(st)
            buf = t.empty(max(int(nbytes), 1), dtype=t.uint8, device=dev)
            _WS[key] = buf
    return buf


def is_colmajor_cuda(x):
    return (type(x).__module__.startswith("torch") and x.is_cuda and x.dim() == 2
            and (x.stride(0) == 1 or x.shape[0] <= 1) and x.stride(1) >= max(x.shape[0], 1))


def to_device_colmajor(a, dtype=None):
    """numpy (any order) -> column-major CUDA tensor (ld = rows)."""
    t = require_cuda()
    a = np.asarray(a)
    if dtype is not None:
        a = a.astype(dtype, copy=False)
    host = t.from_numpy(np.ascontiguousarray(a.T))  # (cols, rows) row-major == column-major a
    return host.to("cuda", non_blocking=False).t()


def empty_colmajor(rows, cols, dtype):
    t = require_cuda()
    return t.empty((cols, rows), dtype=dtype, device="cuda").t()


def to_host_colmajor(x):
    """column-major CUDA tensor -> F-ordered numpy array."""
    return np.asfortranarray(x.t().contiguous().cpu().numpy().T)


def ld_of(x):
    return max(int(x.stride(1)), int(x.shape[0]), 1)


def vec_to_device(v, dtype):
    t = require_cuda()
    return t.as_tensor(np.ascontiguousarray(np.asarray(v)), device="cuda").to(dtype)


def _is_cuda_tensor(x):
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)
