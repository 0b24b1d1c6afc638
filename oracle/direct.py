"""Transform-free and loop oracles -- TEST INFRASTRUCTURE ONLY.

Restatement of the reference's independent checkers (gyroproxy/oracles.py and
the direct-summation DFT pair in gyroproxy/spectral.py:65-106, 164-200).  They
share no code with the FFT path, so agreement with them is evidence.  Desk
sizes only.
"""

from __future__ import annotations

import numpy as np

from .port import kx_deriv, kx_signed


def hermitian_ky0(spec):
    """Hermitian part of the ky=0 row (spectral.py:164-175)."""
    spec = np.array(spec, dtype=complex)
    rev = (-np.arange(spec.shape[-1])) % spec.shape[-1]
    row = spec[..., 0, :]
    spec[..., 0, :] = 0.5 * (row + np.conj(row[..., rev]))
    return spec


def is_hermitian(spec, tol=1e-12):
    """spectral.py:178-184."""
    spec = np.asarray(spec)
    rev = (-np.arange(spec.shape[-1])) % spec.shape[-1]
    row = spec[..., 0, :]
    return bool(np.max(np.abs(row - np.conj(row[..., rev]))) <= tol)


def random_spectrum(n_kx, n_ky, gen):
    """Representable random spectrum (spectral.py:187-200)."""
    re = gen.uniform(-1.0, 1.0, (n_ky, n_kx))
    im = gen.uniform(-1.0, 1.0, (n_ky, n_kx))
    spec = hermitian_ky0(re + 1j * im)
    if n_kx % 2 == 0:
        spec[..., n_kx // 2] = 0.0
    return spec


def dft2(field):
    """Unscaled forward half-spectrum by dense sums (spectral.py:65-80)."""
    field = np.asarray(field, dtype=float)
    n_y, n_x = field.shape
    ey = np.exp(-2j * np.pi * np.outer(np.arange(n_y // 2 + 1), np.arange(n_y)) / n_y)
    ex = np.exp(-2j * np.pi * np.outer(np.arange(n_x), np.arange(n_x)) / n_x)
    return ey @ field.astype(complex) @ ex.T


def idft2(spec, n_y):
    """Inverse of dft2 divided by n_x*n_y (spectral.py:83-106)."""
    spec = np.asarray(spec, dtype=complex)
    m, n_x = spec.shape
    if m > n_y // 2 + 1:
        raise ValueError("too many spectral rows")
    neg = (-np.arange(n_x)) % n_x
    full = np.zeros((n_y, n_x), dtype=complex)
    full[:m] = spec
    for row in range(m, n_y):
        mirror = n_y - row
        if 1 <= mirror < m:
            full[row] = np.conj(spec[mirror][neg])
    ey = np.exp(2j * np.pi * np.outer(np.arange(n_y), np.arange(n_y)) / n_y)
    ex = np.exp(2j * np.pi * np.outer(np.arange(n_x), np.arange(n_x)) / n_x)
    return (ey @ full @ ex.T / (n_x * n_y)).real


def field_loop(h, weights):
    """oracles.py:17-25."""
    out = np.zeros(h.shape[3:], dtype=h.dtype)
    for idx in np.ndindex(h.shape[:3]):
        out = out + weights[idx] * h[idx]
    return out


def stream_loop(h, stencil):
    """oracles.py:28-39."""
    c = np.asarray(stencil, dtype=float)
    half = len(c) // 2
    nt = h.shape[3]
    out = np.zeros_like(h)
    for t in range(nt):
        acc = np.zeros_like(h[:, :, :, 0])
        for i, ci in enumerate(c):
            acc = acc + ci * h[:, :, :, (t + i - half) % nt]
        out[:, :, :, t] = acc
    return out


def shear_loop(h, shifts):
    """oracles.py:42-52."""
    n_ky, n_kx = h.shape[-2:]
    out = np.zeros_like(h)
    for iy in range(n_ky):
        s = int(shifts[iy])
        for ix in range(n_kx):
            if 0 <= ix + s < n_kx:
                out[..., iy, ix] = h[..., iy, ix + s]
    return out


def collision_loop(h, matrices):
    """oracles.py:55-67 (scalar accumulation per velocity row)."""
    m = h.shape[0] * h.shape[1] * h.shape[2]
    nt = h.shape[3]
    hs = h.reshape(m, nt, -1)
    out = np.zeros_like(hs)
    for t in range(nt):
        for i in range(m):
            acc = np.zeros(hs.shape[2], dtype=hs.dtype)
            for j in range(m):
                acc = acc + matrices[t, i, j] * hs[j, t]
            out[i, t] = acc
    return out.reshape(h.shape)


def bracket_convolution(f, g):
    """Direct quadratic mode-sum bracket, no transforms (oracles.py:70-135).

    {f,g}(k) = -sum_{k1+k2=k} (k1x' k2y - k1y k2x') f(k1) g(k2), both inputs
    first projected onto what a c2r synthesis represents.
    """
    def representable(s):
        s = hermitian_ky0(np.asarray(s, dtype=complex))
        if s.shape[-1] % 2 == 0:
            s[..., s.shape[-1] // 2] = 0.0
        return s

    def full_plane(s):
        n_ky, n_kx = s.shape
        neg = (-np.arange(n_kx)) % n_kx
        kys = np.arange(-(n_ky - 1), n_ky)
        rows = np.stack([s[k] if k >= 0 else np.conj(s[-k][neg]) for k in kys])
        return rows, kys

    f = representable(f)
    g = representable(g)
    n_ky, n_kx = f.shape
    kxv = kx_signed(n_kx)
    kxd = kx_deriv(n_kx)
    ff, kys = full_plane(f)
    gf, _ = full_plane(g)
    ylo, yhi = 2 * kys.min(), 2 * kys.max()
    xlo, xhi = 2 * int(kxv.min()), 2 * int(kxv.max())
    acc = np.zeros((yhi - ylo + 1, xhi - xlo + 1), dtype=complex)
    g_dy = gf * kys[:, None]
    g_dx = gf * kxd[None, :]
    for i1, k1y in enumerate(kys):
        for j1, k1x in enumerate(kxv):
            c = ff[i1, j1]
            if c == 0:
                continue
            acc[np.ix_(k1y + kys - ylo, k1x + kxv - xlo)] += -(kxd[j1] * g_dy - k1y * g_dx) * c
    out = np.zeros((n_ky, n_kx), dtype=complex)
    for iy in range(n_ky):
        out[iy] = acc[iy - ylo, kxv - xlo]
    if n_kx % 2 == 0:
        out[:, n_kx // 2] = 0.0
    return out
