"""Half-spectrum transforms and the dealiased Poisson bracket -- GPU drop-in for
the reference's ``gyroproxy.spectral`` (spectral.py).

Conventions are the reference's (spectral.py:1-37): spectra are complex
``[..., ky, kx]`` with ky = 0..n_ky-1 and kx in FFT wrap order; real fields are
``[..., y, x]``; synthesis is the unscaled mode sum, analysis divides by the
grid point count; the unpaired radial Nyquist column is zeroed whenever a
spectrum changes size.  The arithmetic runs in libgk (csrc/spectral.cu); this
module keeps the reference's signatures and ValueError conditions, validating
before any device work.
"""

from __future__ import annotations

import math
import threading

import numpy as np
import torch

from . import _lib
from ._device import require_cuda, shape_of, to_device, on_input_device
from .padding import DEFAULT_PRIMES, DEFAULT_RULE, PaddedPlan, dealias_minimum, plan_padded_size

# --------------------------------------------------------------------------
# wavenumber tables (spectral.py:46-62) -- host integers, bit-exact


def kx_values(n_kx: int) -> np.ndarray:
    """Signed radial wavenumbers in FFT wrap order."""
    k = np.arange(n_kx)
    return np.where(k < (n_kx + 1) // 2, k, k - n_kx)


def kx_derivative_values(n_kx: int) -> np.ndarray:
    """kx_values as float with the even-size Nyquist entry zeroed."""
    k = kx_values(n_kx).astype(float)
    if n_kx % 2 == 0:
        k[n_kx // 2] = 0.0
    return k


def min_padded_x(n_kx: int) -> int:
    """3/2-rule radial grid bound (spectral.py:203-206)."""
    return dealias_minimum(n_kx, DEFAULT_RULE)


def min_padded_y(n_ky: int) -> int:
    """Toroidal bound 3*n_ky - 2 for a half spectrum (spectral.py:209-214)."""
    return 3 * n_ky - 2


def bracket_plans(n_kx: int, n_ky: int, rule=DEFAULT_RULE, allowed_primes=DEFAULT_PRIMES):
    """(plan_x, plan_y): y planned on the signed extent 2*n_ky - 1 (spectral.py:217-225)."""
    return (plan_padded_size(n_kx, rule, allowed_primes),
            plan_padded_size(2 * n_ky - 1, rule, allowed_primes))


def _plan_size(plan) -> int:
    return plan.n_padded if isinstance(plan, PaddedPlan) else int(plan)


# --------------------------------------------------------------------------
# host-side spectrum helpers (inputs / checks; spectral.py:164-200)


def hermitian_ky0(spec):
    """Copy with the ky=0 row projected onto its Hermitian part."""
    spec = np.array(spec, dtype=complex)
    rev = (-np.arange(spec.shape[-1])) % spec.shape[-1]
    row = spec[..., 0, :]
    spec[..., 0, :] = 0.5 * (row + np.conj(row[..., rev]))
    return spec


def is_hermitian(spec, tol: float = 1e-12) -> bool:
    spec = spec.detach().cpu().numpy() if isinstance(spec, torch.Tensor) else np.asarray(spec)
    rev = (-np.arange(spec.shape[-1])) % spec.shape[-1]
    row = spec[..., 0, :]
    return bool(np.max(np.abs(row - np.conj(row[..., rev]))) <= tol)


def random_spectrum(n_kx: int, n_ky: int, gen: np.random.Generator) -> np.ndarray:
    """Random representable spectrum: Hermitian ky=0 row, empty Nyquist column."""
    re = gen.uniform(-1.0, 1.0, (n_ky, n_kx))
    im = gen.uniform(-1.0, 1.0, (n_ky, n_kx))
    spec = hermitian_ky0(re + 1j * im)
    if n_kx % 2 == 0:
        spec[..., n_kx // 2] = 0.0
    return spec


# --------------------------------------------------------------------------
# device plans


class SpectralPlan:
    """Owns a gk_spectral_plan (twiddle tables on one device)."""

    def __init__(self, n_kx: int, n_ky: int, n_x: int, n_y: int, device: torch.device):
        self.sizes = (n_kx, n_ky, n_x, n_y)
        self.device = device
        lib = _lib.load()
        handle = _lib._p()
        with torch.cuda.device(device):
            _lib.check(lib.gk_spectral_plan_create(n_kx, n_ky, n_x, n_y, _lib.C.byref(handle)),
                       "gk_spectral_plan_create")
        self.handle = handle
        self._lib = lib

    def __del__(self):
        try:
            if self.handle:
                with torch.cuda.device(self.device):
                    self._lib.gk_spectral_plan_destroy(self.handle)
        except Exception:
            pass


_plans: dict = {}
_plans_lock = threading.Lock()


def get_plan(n_kx: int, n_ky: int, n_x: int, n_y: int, device: torch.device) -> SpectralPlan:
    key = (device.index, n_kx, n_ky, n_x, n_y)
    with _plans_lock:
        plan = _plans.get(key)
        if plan is None:
            plan = SpectralPlan(n_kx, n_ky, n_x, n_y, device)
            _plans[key] = plan
        return plan


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def _check_sizes(n_kx, n_ky, n_x, n_y):
    if n_kx > n_x:
        raise ValueError(f"{n_kx} radial modes do not fit a grid of {n_x} points")
    if n_ky > n_y // 2 + 1:
        raise ValueError(f"{n_ky} toroidal modes do not fit a grid of {n_y} points")


# --------------------------------------------------------------------------
# transforms (spectral.py:116-161)


@on_input_device
def to_real(spec, n_x: int, n_y: int):
    """Real field (..., n_y, n_x) synthesised from retained modes (spectral.py:116-138)."""
    shp = shape_of(spec)
    n_ky, n_kx = shp[-2:]
    _check_sizes(n_kx, n_ky, n_x, n_y)
    t, carrier = to_device(spec, torch.complex128)
    batch = math.prod(shp[:-2])
    out = torch.empty(tuple(shp[:-2]) + (n_y, n_x), dtype=torch.float64, device=t.device)
    if batch:
        plan = get_plan(n_kx, n_ky, n_x, n_y, t.device)
        lib = plan._lib
        ws = _workspace(lib.gk_transform_workspace_bytes(plan.handle, batch), t.device)
        _lib.check(lib.gk_to_real(plan.handle, t.data_ptr(), out.data_ptr(), batch, ws.data_ptr(),
                                  ws.numel(), _lib.stream_of(t.device)), "gk_to_real")
    return carrier.back(out)


@on_input_device
def to_spectrum(field, n_kx: int, n_ky: int):
    """Retained modes (..., n_ky, n_kx) of a real field (spectral.py:141-161)."""
    shp = shape_of(field)
    n_y, n_x = shp[-2:]
    _check_sizes(n_kx, n_ky, n_x, n_y)
    if np.iscomplexobj(field) if not isinstance(field, torch.Tensor) else field.is_complex():
        field = field.real  # np.asarray(field, dtype=float) would warn and drop it too
    t, carrier = to_device(field, torch.float64)
    batch = math.prod(shp[:-2])
    out = torch.empty(tuple(shp[:-2]) + (n_ky, n_kx), dtype=torch.complex128, device=t.device)
    if batch:
        plan = get_plan(n_kx, n_ky, n_x, n_y, t.device)
        lib = plan._lib
        ws = _workspace(lib.gk_transform_workspace_bytes(plan.handle, batch), t.device)
        _lib.check(lib.gk_to_spectrum(plan.handle, t.data_ptr(), out.data_ptr(), batch, ws.data_ptr(),
                                      ws.numel(), _lib.stream_of(t.device)), "gk_to_spectrum")
    return carrier.back(out)


# --------------------------------------------------------------------------
# bracket (spectral.py:232-268)

#: bound on the per-call g-field cache (n_g * n_x * n_y * 16 bytes); larger
#: broadcast-free batches are processed in sub-batches.
G_FIELD_BUDGET = 4 << 30


def _validate_bracket(fshape, gshape, plan_x, plan_y):
    if tuple(fshape[-2:]) != tuple(gshape[-2:]):
        raise ValueError(f"logical shapes differ: {tuple(fshape[-2:])} vs {tuple(gshape[-2:])}")
    n_ky, n_kx = fshape[-2:]
    n_x, n_y = _plan_size(plan_x), _plan_size(plan_y)
    if n_x < min_padded_x(n_kx):
        raise ValueError(f"plan_x size {n_x} below dealias bound {min_padded_x(n_kx)}")
    if n_y < min_padded_y(n_ky):
        raise ValueError(f"plan_y size {n_y} below dealias bound {min_padded_y(n_ky)}")
    return n_kx, n_ky, n_x, n_y


@on_input_device
def bracket_device(f: torch.Tensor, g: torch.Tensor, n_x: int, n_y: int, out_batch=None) -> torch.Tensor:
    """Bracket of device tensors (complex128, contiguous), broadcasting batch axes."""
    n_ky, n_kx = f.shape[-2:]
    bf, bg = tuple(f.shape[:-2]), tuple(g.shape[:-2])
    ob = tuple(np.broadcast_shapes(bf, bg)) if out_batch is None else out_batch
    n_out = math.prod(ob)
    out = torch.empty(ob + (n_ky, n_kx), dtype=torch.complex128, device=f.device)
    if n_out == 0:
        return out
    nf, ng = math.prod(bf), math.prod(bg)
    plan = get_plan(n_kx, n_ky, n_x, n_y, f.device)
    lib = plan._lib
    fmap = None
    if bf != ob:
        fmap = torch.from_numpy(np.ascontiguousarray(
            np.broadcast_to(np.arange(nf).reshape(bf), ob).reshape(-1))).to(f.device)
    gidx = np.broadcast_to(np.arange(ng).reshape(bg), ob).reshape(-1)
    gmod = ng
    gmap = None
    if not np.array_equal(gidx, np.arange(n_out) % ng):
        gmap = torch.from_numpy(np.ascontiguousarray(gidx)).to(f.device)
    g_bytes = ng * n_x * n_y * 16
    if g_bytes > G_FIELD_BUDGET and gmap is None and fmap is None and ng == n_out:
        # one-to-one pairs: process in sub-batches so the g-field cache stays bounded
        step = max(1, G_FIELD_BUDGET // (n_x * n_y * 16))
        ff, gg, oo = f.reshape(-1, n_ky, n_kx), g.reshape(-1, n_ky, n_kx), out.view(-1, n_ky, n_kx)
        for s in range(0, n_out, step):
            e = min(n_out, s + step)
            oo[s:e] = bracket_device(ff[s:e], gg[s:e], n_x, n_y)
        return out
    ws = _workspace(lib.gk_bracket_workspace_bytes(plan.handle, n_out, ng), f.device)
    _lib.check(lib.gk_bracket(plan.handle, f.data_ptr(), g.data_ptr(), out.data_ptr(), n_out,
                              _lib.ptr(fmap), _lib.ptr(gmap), ng, gmod, ws.data_ptr(), ws.numel(),
                              _lib.stream_of(f.device)), "gk_bracket")
    return out


@on_input_device
def bracket(f, g, plan_x, plan_y):
    """Dealiased Poisson bracket {f, g} = (dx f)(dy g) - (dy f)(dx g) (spectral.py:232-268).

    Leading batch axes broadcast; plans are PaddedPlan or plain ints at or above
    the dealias bounds.  Same ValueErrors as the reference, raised before any
    device work.
    """
    fs, gs = shape_of(f), shape_of(g)
    _, _, n_x, n_y = _validate_bracket(fs, gs, plan_x, plan_y)
    ob = tuple(np.broadcast_shapes(tuple(fs[:-2]), tuple(gs[:-2])))
    ft, carrier = to_device(f, torch.complex128)
    gt, _ = to_device(g, torch.complex128, ft.device)
    return carrier.back(bracket_device(ft, gt, n_x, n_y, ob))
