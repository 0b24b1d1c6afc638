"""The five proxy kernels on B200 -- drop-in for the reference's
``gyroproxy.kernels`` (kernels.py).

Same names, signatures, constants and ValueError conditions as the reference;
the arithmetic runs in libgk (csrc/*.cu) through the C-ABI of include/gk.h.
numpy inputs give numpy outputs; torch CUDA tensors stay on the device.

Variant semantics (kernels.py:9-20): ``shear`` variants are bitwise equal (pure
data movement); ``stream`` "original" reproduces the reference's roll-accumulate
rounding exactly, "optimized" is a fused FMA pass (agreement to rounding, as in
the reference); ``field``, ``collision`` and ``nonlinear`` have one
implementation run under both labels.
"""

from __future__ import annotations

import hashlib
import statistics
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_host_numpy, shape_of, to_device, on_input_device
from .grid import GridShape, random_complex, random_state, substream
from .spectral import _plan_size, _validate_bracket, bracket_plans, get_plan

KERNEL_NAMES = ("field", "stream", "shear", "collision", "nonlinear")
VARIANTS = ("original", "optimized")

#: fourth-order centred first derivative (kernels.py:40-42)
DEFAULT_STENCIL = (1.0 / 12.0, -8.0 / 12.0, 0.0, 8.0 / 12.0, -1.0 / 12.0)

_VARIANT_CODE = {"original": 0, "optimized": 1}


def _check_variant(variant: str):
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")


def _stream(device) -> int:
    return _lib.stream_of(device)


@on_input_device
def field_kernel(h, weights):
    """out[theta, ky, kx] = sum_{s,e,xi} w[s,e,xi] h[s,e,xi,theta,ky,kx] (kernels.py:45-52)."""
    hs, ws = shape_of(h), shape_of(weights)
    if tuple(ws) != tuple(hs[:3]):
        raise ValueError(f"weights shape {tuple(ws)} != velocity dims {tuple(hs[:3])}")
    ht, carrier = to_device(h, torch.complex128)
    wt, _ = to_device(weights, torch.float64, ht.device)
    n_vel = int(np.prod(hs[:3]))
    n_theta, n_cells = hs[3], hs[4] * hs[5]
    out = torch.empty(tuple(hs[3:]), dtype=torch.complex128, device=ht.device)
    if out.numel():
        if n_vel == 0:
            out.zero_()
        else:
            _lib.check(_lib.load().gk_field(ht.data_ptr(), wt.data_ptr(), out.data_ptr(), n_vel, n_theta,
                                            n_cells, _stream(ht.device)), "gk_field")
    return carrier.back(out)


@on_input_device
def stream_kernel(h, stencil, variant: str = "optimized"):
    """Periodic odd-width stencil along theta (kernels.py:55-77)."""
    _check_variant(variant)
    c = as_host_numpy(stencil, dtype=float)
    w = c.shape[0]
    hs = shape_of(h)
    n_theta = hs[3]
    if w % 2 == 0:
        raise ValueError(f"stencil width must be odd, got {w}")
    if w > n_theta:
        raise ValueError(f"stencil width {w} exceeds n_theta {n_theta}")
    ht, carrier = to_device(h, torch.complex128)
    out = torch.empty_like(ht)
    if out.numel():
        n_vel = int(np.prod(hs[:3]))
        if w <= 31:  # coefficients travel in the kernel parameters
            _lib.check(_lib.load().gk_stream(ht.data_ptr(), _lib.doubles(c), w, _VARIANT_CODE[variant],
                                             out.data_ptr(), n_vel, n_theta, hs[4] * hs[5], _stream(ht.device)),
                       "gk_stream")
        else:  # any wider odd stencil: coefficients from device memory
            cd = torch.from_numpy(np.ascontiguousarray(c)).to(ht.device)
            _lib.check(_lib.load().gk_stream_wide(ht.data_ptr(), cd.data_ptr(), w, _VARIANT_CODE[variant],
                                                  out.data_ptr(), n_vel, n_theta, hs[4] * hs[5],
                                                  _stream(ht.device)), "gk_stream_wide")
    return carrier.back(out)


@on_input_device
def shear_kernel(h, shifts, variant: str = "optimized"):
    """Per-toroidal-mode radial gather with zero fill (kernels.py:80-106)."""
    _check_variant(variant)
    s = as_host_numpy(shifts).astype(int)
    hs = shape_of(h)
    n_ky, n_kx = hs[-2:]
    if s.shape != (n_ky,):
        raise ValueError(f"need one shift per toroidal mode, got shape {s.shape}")
    if np.any(np.abs(s) > n_kx):
        raise ValueError("shifts exceed the radial extent")
    ht, carrier = to_device(h, torch.complex128)
    st = torch.from_numpy(s.astype(np.int32)).to(ht.device)
    out = torch.empty_like(ht)
    if out.numel():
        rows = int(np.prod(hs[:-2]))
        _lib.check(_lib.load().gk_shear(ht.data_ptr(), st.data_ptr(), out.data_ptr(), rows, n_ky, n_kx,
                                        _stream(ht.device)), "gk_shear")
    return carrier.back(out)


@on_input_device
def collision_kernel(h, matrices):
    """Per-theta real (M x M) matvec over flattened velocity space (kernels.py:109-123)."""
    hs = shape_of(h)
    ns, ne, nxi, n_theta = hs[:4]
    m = ns * ne * nxi
    if tuple(shape_of(matrices)) != (n_theta, m, m):
        raise ValueError(f"need matrices of shape {(n_theta, m, m)}, got {tuple(shape_of(matrices))}")
    ht, carrier = to_device(h, torch.complex128)
    at, _ = to_device(matrices, torch.float64, ht.device)
    out = torch.empty_like(ht)
    if out.numel():
        _lib.check(_lib.load().gk_collision(at.data_ptr(), ht.data_ptr(), out.data_ptr(), m, n_theta,
                                            hs[4] * hs[5], _stream(ht.device)), "gk_collision")
    return carrier.back(out)


@on_input_device
def nonlinear_device(h: torch.Tensor, phi: torch.Tensor, n_x: int, n_y: int) -> torch.Tensor:
    """Device-resident nonlinear term (validated inputs)."""
    n_theta, n_ky, n_kx = h.shape[3:]
    n_vel = int(np.prod(h.shape[:3]))
    out = torch.empty_like(h)
    if out.numel() == 0:
        return out
    plan = get_plan(n_kx, n_ky, n_x, n_y, h.device)
    lib = plan._lib
    nbytes = lib.gk_bracket_workspace_bytes(plan.handle, n_vel * n_theta, n_theta)
    ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=h.device)
    _lib.check(lib.gk_nonlinear(plan.handle, h.data_ptr(), phi.data_ptr(), out.data_ptr(), n_vel, n_theta,
                                ws.data_ptr(), ws.numel(), _stream(h.device)), "gk_nonlinear")
    return out


@on_input_device
def nonlinear_kernel(h, phi, plans, threads: int = 1):
    """Dealiased bracket of every (s, e, xi, theta) slice with phi[theta] (kernels.py:126-150).

    ``threads`` is accepted for API compatibility; the result never depends on it.
    """
    hs = shape_of(h)
    n_theta, n_ky, n_kx = hs[3:]
    if tuple(shape_of(phi)) != (n_theta, n_ky, n_kx):
        raise ValueError(f"phi shape {tuple(shape_of(phi))} != field dims {(n_theta, n_ky, n_kx)}")
    plan_x, plan_y = plans
    _, _, n_x, n_y = _validate_bracket(hs, shape_of(phi), plan_x, plan_y)
    ht, carrier = to_device(h, torch.complex128)
    pt, _ = to_device(phi, torch.complex128, ht.device)
    return carrier.back(nonlinear_device(ht, pt, n_x, n_y))


def make_kernel_inputs(shape: GridShape, seed: int) -> dict:
    """Seeded auxiliary inputs, substreams 1-4 (kernels.py:158-173); host numpy arrays."""
    m = shape.velocity_size
    return {
        "weights": substream(seed, 1).uniform(-1.0, 1.0, (shape.n_species, shape.n_energy, shape.n_xi)),
        "stencil": np.asarray(DEFAULT_STENCIL),
        "shifts": substream(seed, 2).integers(-3, 4, shape.n_toroidal),
        "matrices": substream(seed, 3).uniform(-1.0, 1.0, (shape.n_theta, m, m)),
        "phi": random_complex(substream(seed, 4), shape.field_dims),
        "plans": bracket_plans(shape.n_radial, shape.n_toroidal),
    }


def run_kernel(kernel: str, h, inputs: dict, variant: str = "optimized", threads: int = 1):
    """Dispatch one kernel by name (kernels.py:176-189)."""
    _check_variant(variant)
    if kernel == "field":
        return field_kernel(h, inputs["weights"])
    if kernel == "stream":
        return stream_kernel(h, inputs["stencil"], variant)
    if kernel == "shear":
        return shear_kernel(h, inputs["shifts"], variant)
    if kernel == "collision":
        return collision_kernel(h, inputs["matrices"])
    if kernel == "nonlinear":
        return nonlinear_kernel(h, inputs["phi"], inputs["plans"], threads)
    raise ValueError(f"unknown kernel {kernel!r}; expected one of {KERNEL_NAMES}")


def checksum(values) -> str:
    """First 16 hex of sha256(repr((shape, dtype.str)) + bytes) (kernels.py:192-198)."""
    if isinstance(values, torch.Tensor):
        values = values.detach().cpu().numpy()
    a = np.ascontiguousarray(values)
    digest = hashlib.sha256()
    digest.update(repr((a.shape, a.dtype.str)).encode())
    digest.update(a.tobytes())
    return digest.hexdigest()[:16]


@dataclass(frozen=True)
class KernelTiming:
    kernel: str
    variant: str
    reps: int
    median_s: float
    min_s: float
    checksum: str


def time_kernel(kernel: str, variant: str, shape: GridShape, reps: int, seed: int, threads: int = 1) -> KernelTiming:
    """Median/min device wallclock of a kernel on seeded data (kernels.py:211-235).

    Inputs are moved to the GPU once; each repetition is bracketed by device
    synchronisation, so the times are the kernel's, not the PCIe copies'.  The
    checksum is of the final output, as in the reference.
    """
    if reps < 3:
        raise ValueError(f"reps must be >= 3, got {reps}")
    _check_variant(variant)
    h, _ = to_device(random_state(shape, seed), torch.complex128)
    host_inputs = make_kernel_inputs(shape, seed)
    inputs = dict(host_inputs)
    for key in ("weights", "matrices"):
        inputs[key] = to_device(host_inputs[key], torch.float64, h.device)[0]
    inputs["phi"] = to_device(host_inputs["phi"], torch.complex128, h.device)[0]
    out = run_kernel(kernel, h, inputs, variant, threads)
    times = []
    for _ in range(reps):
        torch.cuda.synchronize(h.device)
        start = time.perf_counter()
        out = run_kernel(kernel, h, inputs, variant, threads)
        torch.cuda.synchronize(h.device)
        times.append(time.perf_counter() - start)
    return KernelTiming(kernel=kernel, variant=variant, reps=reps, median_s=statistics.median(times),
                        min_s=min(times), checksum=checksum(out))


__all__ = [
    "DEFAULT_STENCIL", "KERNEL_NAMES", "VARIANTS", "KernelTiming", "checksum", "collision_kernel",
    "field_kernel", "make_kernel_inputs", "nonlinear_kernel", "random_state", "run_kernel",
    "shear_kernel", "stream_kernel", "time_kernel", "_plan_size",
]
