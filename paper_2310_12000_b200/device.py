"""Per-device library context and host<->device plumbing (torch tensors carry
device memory; the library runs on torch's current stream)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import DeviceError

_CTX = {}


def torch():
    import torch as _t
    return _t


class Context:
    """One library context per CUDA device (vl_ctx)."""

    def __init__(self, device):
        T = torch()
        if not T.cuda.is_available():
            raise DeviceError("no CUDA device available: the Vecchia-Laplace path runs only on B200 (sm_100a)")
        self.device = int(device)
        self.tdev = T.device("cuda", self.device)
        with T.cuda.device(self.device):
            T.cuda.init()
            stream = T.cuda.current_stream(self.device).cuda_stream
        h = C.c_void_p()
        _lib.call("vl_ctx_create", self.device, C.c_void_p(stream), C.byref(h))
        self.h = h
        info = (C.c_int64 * 2)()
        _lib.call("vl_ctx_info", self.h, info)
        self.num_sms = int(info[1])

    def sync(self):
        _lib.call("vl_ctx_sync", self.h)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().vl_ctx_destroy(self.h)
        except Exception:
            pass


def context(device=None):
    T = torch()
    if device is None:
        device = T.cuda.current_device() if T.cuda.is_available() else 0
    ctx = _CTX.get(device)
    if ctx is None:
        ctx = Context(device)
        _CTX[device] = ctx
    return ctx


def empty(ctx, *shape):
    T = torch()
    return T.empty(shape, dtype=T.float64, device=ctx.tdev)


def zeros(ctx, *shape):
    T = torch()
    return T.zeros(shape, dtype=T.float64, device=ctx.tdev)


def upload(ctx, a, dtype=None):
    """numpy -> contiguous device tensor."""
    T = torch()
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return T.from_numpy(a).to(ctx.tdev)


def download(x):
    return x.detach().cpu().numpy()
