"""numpy restatement of the reference's CPU hot path -- TEST INFRASTRUCTURE ONLY.

This is the "port" oracle: the same algorithm, the same numpy calls (pocketfft
for the transforms, BLAS for the contractions) and the same association order
as the reference's production functions, restated here so that the GPU box
(where ``/root/reference`` does not exist) can (a) check parity and (b) time
the reference's CPU algorithm for ``bench.py --impl reference`` and the
``cpu_baseline`` object.  Every function cites the reference file:line it
restates (paths relative to ``/root/reference/pkg/src/gyroproxy``).

It is pinned against the reference itself by ``tests/test_oracle_golden.py``
(golden vectors produced by importing the reference in the build container,
``tests/golden/make_golden.py``).  Nothing in ``paper_2305_10553_b200`` may
import this module.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from fractions import Fraction

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

DEFAULT_STENCIL = (1.0 / 12.0, -8.0 / 12.0, 0.0, 8.0 / 12.0, -1.0 / 12.0)  # kernels.py:40-42


# --------------------------------------------------------------------------
# plan sizes (padding.py:83-128, spectral.py:203-225)

def _smooth(n, primes=(2, 3, 5, 7)):
    for p in primes:
        while n % p == 0:
            n //= p
    return n == 1


def padded_size(n_logical, rule=Fraction(3, 2)):
    n = math.ceil(n_logical * Fraction(rule))
    while not _smooth(n):
        n += 1
    return n


def plan_sizes(n_kx, n_ky):
    """(n_x, n_y) of spectral.bracket_plans (spectral.py:217-225)."""
    return padded_size(n_kx), padded_size(2 * n_ky - 1)


# --------------------------------------------------------------------------
# spectral conventions (spectral.py:46-62)

def kx_signed(n_kx):
    k = np.arange(n_kx)
    return np.where(k < (n_kx + 1) // 2, k, k - n_kx)


def kx_deriv(n_kx):
    k = kx_signed(n_kx).astype(float)
    if n_kx % 2 == 0:
        k[n_kx // 2] = 0.0
    return k


def synth(spec, n_x, n_y):
    """to_real (spectral.py:116-138): embed, ifft over x, irfft over y, x n_x*n_y."""
    spec = np.asarray(spec, dtype=complex)
    n_ky, n_kx = spec.shape[-2:]
    if n_kx > n_x or n_ky > n_y // 2 + 1:
        raise ValueError("spectrum does not fit the grid")
    grid = np.zeros(spec.shape[:-2] + (n_y // 2 + 1, n_x), dtype=complex)
    grid[..., :n_ky, kx_signed(n_kx) % n_x] = spec
    if n_kx % 2 == 0 and n_x > n_kx:
        grid[..., :n_ky, (-(n_kx // 2)) % n_x] = 0.0
    return np.fft.irfft(np.fft.ifft(grid, axis=-1), n=n_y, axis=-2) * (n_x * n_y)


def analyse(field, n_kx, n_ky):
    """to_spectrum (spectral.py:141-161): rfft over y, fft over x, truncate, / n_x*n_y."""
    field = np.asarray(field, dtype=float)
    n_y, n_x = field.shape[-2:]
    if n_kx > n_x or n_ky > n_y // 2 + 1:
        raise ValueError("more modes than the field resolves")
    full = np.fft.fft(np.fft.rfft(field, axis=-2), axis=-1)
    out = full[..., :n_ky, kx_signed(n_kx) % n_x] / (n_x * n_y)
    if n_kx % 2 == 0 and n_x > n_kx:
        out[..., n_kx // 2] = 0.0
    return out


def poisson_bracket(f, g, n_x, n_y):
    """bracket (spectral.py:232-268) with validated integer plan sizes."""
    f = np.asarray(f, dtype=complex)
    g = np.asarray(g, dtype=complex)
    n_ky, n_kx = f.shape[-2:]
    dx = 1j * kx_deriv(n_kx)
    dy = 1j * np.arange(n_ky, dtype=float)[:, None]
    fx, fy = synth(f * dx, n_x, n_y), synth(f * dy, n_x, n_y)
    gx, gy = synth(g * dx, n_x, n_y), synth(g * dy, n_x, n_y)
    return analyse(fx * gy - fy * gx, n_kx, n_ky)


# --------------------------------------------------------------------------
# the five kernels (kernels.py:45-150)

def field(h, weights):
    """kernels.py:45-52 -- tensordot over the three velocity axes."""
    return np.tensordot(weights, h, axes=3)


def stream(h, stencil, variant="optimized"):
    """kernels.py:55-77 -- periodic theta stencil, both association orders."""
    c = np.asarray(stencil, dtype=float)
    w = c.shape[0]
    half = w // 2
    nt = h.shape[3]
    if variant == "original":
        acc = np.zeros_like(h)
        for i, ci in enumerate(c):
            acc += ci * np.roll(h, half - i, axis=3)
        return acc
    ext = np.concatenate([h[:, :, :, nt - half:], h, h[:, :, :, :half]], axis=3)
    return sliding_window_view(ext, w, axis=3) @ c


def shear(h, shifts):
    """kernels.py:80-106 -- per-ky radial gather with zero fill."""
    shifts = np.asarray(shifts, dtype=int)
    n_kx = h.shape[-1]
    out = np.zeros_like(h)
    for iy, s in enumerate(shifts):
        if s >= 0:
            out[..., iy, : n_kx - s] = h[..., iy, s:]
        else:
            out[..., iy, -s:] = h[..., iy, : n_kx + s]
    return out


def collision(h, matrices):
    """kernels.py:109-123 -- per-theta (M x M) @ (M x Y*R) over flattened velocity."""
    m = h.shape[0] * h.shape[1] * h.shape[2]
    nt = h.shape[3]
    hs = h.reshape(m, nt, -1)
    out = np.empty_like(hs)
    for t in range(nt):
        out[:, t] = matrices[t] @ hs[:, t]
    return out.reshape(h.shape)


def nonlinear(h, phi, n_x, n_y, threads=1):
    """kernels.py:126-150 -- bracket of every (v, theta) slice with phi[theta]."""
    nt, nky, nkx = h.shape[3:]
    batch = h.reshape(-1, nt, nky, nkx)
    if threads <= 1 or batch.shape[0] < 2 * threads:
        out = poisson_bracket(batch, phi, n_x, n_y)
    else:
        parts = np.array_split(batch, threads)
        with ThreadPoolExecutor(max_workers=threads) as pool:
            out = np.concatenate(list(pool.map(lambda c: poisson_bracket(c, phi, n_x, n_y), parts)))
    return out.reshape(h.shape)


# --------------------------------------------------------------------------
# builder-defined step: only reference functions composed

def step(h, weights, stencil, matrices, shifts, dt, n_x, n_y, nonlinear_on=True, threads=1):
    """phi = field(h); rhs = stream + nonlinear + collision; h' = shear(h + dt*rhs)."""
    phi = field(h, weights)
    rhs = stream(h, stencil)
    if nonlinear_on:
        rhs = rhs + nonlinear(h, phi, n_x, n_y, threads)
    rhs = rhs + collision(h, matrices)
    return shear(h + dt * rhs, shifts), phi
