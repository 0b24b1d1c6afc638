"""Array plumbing between the reference's numpy API and device tensors.

The reference functions take and return numpy arrays.  The drop-in keeps that
contract: numpy in -> numpy out (host<->device copies included), while torch
CUDA tensors stay on the device (no copies).  CPU torch tensors are returned as
CPU torch tensors.  Compute always happens on the GPU; without one, calls fail
loudly after argument validation.
"""

from __future__ import annotations

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2305_10553_b200 computes on a CUDA (sm_100a) device; none is visible "
                           "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class Carrier:
    """Remembers how an input arrived so the output goes back the same way."""

    __slots__ = ("kind", "device")

    def __init__(self, kind, device):
        self.kind = kind
        self.device = device

    def back(self, t: torch.Tensor):
        if self.kind == "cuda":
            return t
        if self.kind == "torch":
            return t.cpu()
        return t.cpu().numpy()


def shape_of(a):
    return tuple(a.shape) if hasattr(a, "shape") else np.shape(a)


def to_device(a, dtype: torch.dtype, device=None):
    """Return (contiguous tensor on the GPU, Carrier)."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            # a CUDA tensor stays where it is unless a device is requested
            t = a.to(device=device, dtype=dtype) if device is not None else a.to(dtype=dtype)
            return t.contiguous(), Carrier("cuda", t.device)
        dev = device or require_cuda()
        return a.to(dtype=dtype).contiguous().to(dev), Carrier("torch", dev)
    dev = device or require_cuda()
    npdt = {torch.complex128: np.complex128, torch.float64: np.float64, torch.int32: np.int32,
            torch.int64: np.int64}[dtype]
    host = np.ascontiguousarray(np.asarray(a, dtype=npdt))
    return torch.from_numpy(host).to(dev), Carrier("numpy", dev)


def as_host_numpy(a, dtype=None):
    """Host copy of a small auxiliary input (shifts, stencils, weights for validation)."""
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, dtype=dtype)


def on_device(device):
    """The CUDA device context for libgk calls (the library allocates and launches
    on the current device); a no-op for None / CPU devices."""
    import contextlib
    if device is None:
        return contextlib.nullcontext()
    d = torch.device(device)
    return torch.cuda.device(d) if d.type == "cuda" else contextlib.nullcontext()


def device_method(fn):
    """Run a Stepper / DistStepper method with ``self.device`` current."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        with on_device(getattr(self, "device", None)):
            return fn(self, *args, **kwargs)
    return wrapper


def on_input_device(fn):
    """Run a kernel entry point with the device of its first CUDA tensor argument
    current (numpy / host inputs go to the current device anyway)."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        for a in list(args) + list(kwargs.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                with torch.cuda.device(a.device):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)
    return wrapper

