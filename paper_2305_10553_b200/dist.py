"""Multi-GPU step: toroidal-home layout with all-to-all transposes around the
nonlinear term (SURVEY.md §8 e; no reference code -- the reference only models
this decomposition analytically, commsim.py:1-32, 213-219).

One process per GPU, ``torch.distributed`` (NCCL) for the collectives.

Home ("linear") layout: rank g holds h[:, :, :, :, Y_g, :] -- a contiguous block
of Y/G toroidal modes, stored [M][T][Y/G][R].  field (full velocity sum, so no
all-reduce and bitwise G-invariant), stream, shear and collision are local.

Nonlinear layout: rank g holds velocity rows M_g (M/G of them) x all (T, Y, R).

Per step:
  1. all-gather phi blocks -> full phi[T][Y][R] (small).
  2. per velocity chunk k (pipelined, see DistStepper): all-to-all of the home
     rows (per-peer contiguous views of the home shard) -> [src][M/G/K][T][Y/G][R],
     permuted to [M/G/K][T][Y][R] (gk_permute_blocks); bracket; permute to
     [dst][M/G/K][T][Y/G][R]; all-to-all back straight into the home layout.
  5. h' = shear(h + dt * ((stream + nl) + collision)) locally.
Bytes per rank per all-to-all: S/G * (G-1)/G (commsim.alltoall_volume with n1=G).

The collectives move complex128 data viewed as float64.  The compute goes
through an ``ops`` object: ``CudaOps`` (libgk) in production; the gloo tests
pass a CPU oracle implementation of the same interface to check the exchange
logic without a GPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from .grid import GridShape


def _real(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t).reshape(-1)


def shard_bounds(n: int, world: int, rank: int):
    if n % world:
        raise ValueError(f"{n} is not divisible by {world} ranks")
    k = n // world
    return rank * k, (rank + 1) * k


class CudaOps:
    """libgk kernels on device tensors (contiguous complex128)."""

    def __init__(self, shape: GridShape, inputs: dict, dt: float, device, y_block: slice, nonlinear=True):
        import numpy as np

        from .kernels import DEFAULT_STENCIL
        from .spectral import _plan_size, get_plan

        self.lib = _lib.load()
        self.shape, self.dt, self.device = shape, float(dt), device
        self.w = torch.from_numpy(np.asarray(inputs["weights"], dtype=float)).to(device)
        self.A = torch.from_numpy(np.asarray(inputs["matrices"], dtype=float)).to(device)
        self.stencil = np.asarray(inputs.get("stencil", DEFAULT_STENCIL), dtype=float)
        self._st = _lib.doubles(self.stencil)
        sh = np.asarray(inputs["shifts"], dtype=np.int32)[y_block]
        self.shifts = torch.from_numpy(np.ascontiguousarray(sh)).to(device)
        self.plan = None
        if nonlinear:
            px, py = inputs["plans"]
            self.plan = get_plan(shape.n_radial, shape.n_toroidal, _plan_size(px), _plan_size(py), device)

    def _s(self):
        return _lib.stream_of(self.device)

    def field(self, h, out):  # h [M][T][Yl][R] -> out [T][Yl][R]
        M, T = h.shape[0], h.shape[1]
        _lib.check(self.lib.gk_field(h.data_ptr(), self.w.data_ptr(), out.data_ptr(), M, T,
                                     h.shape[2] * h.shape[3], self._s()), "gk_field")

    def stream(self, h, out):
        _lib.check(self.lib.gk_stream(h.data_ptr(), self._st, len(self.stencil), 1, out.data_ptr(), h.shape[0],
                                      h.shape[1], h.shape[2] * h.shape[3], self._s()), "gk_stream")

    def collision(self, h, out):
        _lib.check(self.lib.gk_collision(self.A.data_ptr(), h.data_ptr(), out.data_ptr(), h.shape[0], h.shape[1],
                                         h.shape[2] * h.shape[3], self._s()), "gk_collision")

    def nonlinear(self, hv, phi, out, ws):
        _lib.check(self.lib.gk_nonlinear(self.plan.handle, hv.data_ptr(), phi.data_ptr(), out.data_ptr(),
                                         hv.shape[0], hv.shape[1], ws.data_ptr(), ws.numel(), self._s()),
                   "gk_nonlinear")

    def nonlinear_workspace(self, m_local: int) -> torch.Tensor:
        n = self.lib.gk_bracket_workspace_bytes(self.plan.handle, m_local * self.shape.n_theta, self.shape.n_theta)
        return torch.empty(max(n, 16), dtype=torch.uint8, device=self.device)

    def finish(self, h, nl, c, out):
        """out = shear(h + dt * ((stream(h) + nl) + c)) in one pass (gk_step_finish)."""
        _lib.check(self.lib.gk_step_finish(h.data_ptr(), nl.data_ptr() if nl is not None else None, c.data_ptr(),
                                           self._st, len(self.stencil), self.shifts.data_ptr(), self.dt,
                                           out.data_ptr(), h.shape[0], h.shape[1], h.shape[2], h.shape[3],
                                           self._s()), "gk_step_finish")

    def axpy_shear(self, h, s, nl, c, tmp, out):
        n = h.numel()
        _lib.check(self.lib.gk_axpy3(h.data_ptr(), s.data_ptr(), nl.data_ptr() if nl is not None else None,
                                     c.data_ptr(), self.dt, tmp.data_ptr(), n, self._s()), "gk_axpy3")
        _lib.check(self.lib.gk_shear(tmp.data_ptr(), self.shifts.data_ptr(), out.data_ptr(),
                                     h.shape[0] * h.shape[1], h.shape[2], h.shape[3], self._s()), "gk_shear")

    def permute(self, src, dst, n_a, n_b, inner):
        _lib.check(self.lib.gk_permute_blocks(src.data_ptr(), dst.data_ptr(), n_a, n_b, inner, self._s()),
                   "gk_permute_blocks")


class DistStepper:
    """One rank's share of the distributed step (toroidal-home layout).

    The bracket's velocity rows are dealt out block-cyclically: chunk k is the
    contiguous home block of G*Mk rows, rank q brackets its q-th sub-block.  So
    each chunk's exchange is one contiguous all_to_all_single in both directions
    (no pack kernel on the send side, any backend), and the chunks pipeline:
    the all-to-all bringing chunk k+1 runs on the communication stream while
    chunk k is permuted and bracketed, and chunk k's result travels home while
    chunk k+1 computes.
    """

    def __init__(self, shape: GridShape, ops, device, group=None, nonlinear=True, chunks: int = 4):
        self.shape, self.ops, self.device, self.group = shape, ops, device, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nonlinear = nonlinear
        M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
        self.y0, self.y1 = shard_bounds(Y, self.world, self.rank)
        self.m0, self.m1 = shard_bounds(M, self.world, self.rank) if nonlinear else (0, M)
        self.Yl, self.Ml = self.y1 - self.y0, self.m1 - self.m0
        k = max(1, min(int(chunks), self.Ml))
        while self.Ml % k:
            k -= 1
        self.chunks, self.Mk = k, self.Ml // k
        c128 = dict(dtype=torch.complex128, device=device)
        home = (M, T, self.Yl, R)
        self.buf_c = torch.empty(home, **c128)
        self.phi_l = torch.empty((T, self.Yl, R), **c128)
        if nonlinear:
            G = self.world
            self.phi_g = torch.empty((G, T, self.Yl, R), **c128)
            self.phi = torch.empty((T, Y, R), **c128)
            self.recv = torch.empty((k, G, self.Mk, T, self.Yl, R), **c128)
            self.hv = torch.empty((self.Ml, T, Y, R), **c128)
            self.nlv = torch.empty((self.Ml, T, Y, R), **c128)
            self.send = torch.empty((k, G, self.Mk, T, self.Yl, R), **c128)
            self.nl = torch.empty(home, **c128)
            self.ws = ops.nonlinear_workspace(self.Mk)
        self.comm_bytes_per_step = 0
        if nonlinear and self.world > 1:
            self.comm_bytes_per_step = 2 * self.buf_c.numel() * 16 * (self.world - 1) // self.world

    def home_slice(self, h_full: torch.Tensor) -> torch.Tensor:
        """This rank's home shard of a full state (..., T, Y, R) -> [M][T][Y/G][R]."""
        M, T = self.shape.velocity_size, self.shape.n_theta
        return h_full.reshape(M, T, self.shape.n_toroidal, self.shape.n_radial)[:, :, self.y0:self.y1].contiguous()

    def _block(self, home: torch.Tensor, k: int) -> torch.Tensor:
        """Home rows of chunk k: a contiguous block of G*Mk velocity rows, split
        evenly across the ranks (rank q brackets rows k*G*Mk + q*Mk + [0, Mk))."""
        n = self.world * self.Mk
        return home[k * n:(k + 1) * n]

    def _fwd(self, h: torch.Tensor, k: int):
        """Start the all-to-all bringing chunk k of every rank's home rows here."""
        return dist.all_to_all_single(_real(self.recv[k]), _real(self._block(h, k)), group=self.group,
                                      async_op=True)

    def _back(self, k: int):
        """Start the all-to-all returning chunk k's bracket to its home ranks."""
        return dist.all_to_all_single(_real(self._block(self.nl, k)), _real(self.send[k]), group=self.group,
                                      async_op=True)

    def _nonlinear(self, h: torch.Tensor):
        G, T, Y, R = self.world, self.shape.n_theta, self.shape.n_toroidal, self.shape.n_radial
        ops, K, Mk = self.ops, self.chunks, self.Mk
        if G == 1:
            self.hv.copy_(h)
            ops.nonlinear(self.hv, self.phi, self.nlv, self.ws_full())
            self.nl.copy_(self.nlv)
            return
        pending = self._fwd(h, 0)
        backs = []
        for k in range(K):
            nxt = self._fwd(h, k + 1) if k + 1 < K else None
            pending.wait()  # the compute stream waits for chunk k's arrival
            rows = slice(k * Mk, (k + 1) * Mk)
            ops.permute(self.recv[k], self.hv[rows], G, Mk * T, self.Yl * R)
            ops.nonlinear(self.hv[rows], self.phi, self.nlv[rows], self.ws)
            ops.permute(self.nlv[rows], self.send[k], Mk * T, G, self.Yl * R)
            backs.append(self._back(k))
            pending = nxt
        for w in backs:
            w.wait()

    def ws_full(self):
        if not hasattr(self, "_ws_full"):
            self._ws_full = self.ops.nonlinear_workspace(self.Ml)
        return self._ws_full

    # kept for callers that time the transposes separately (bench split)
    def to_nonlinear_layout(self, h: torch.Tensor):
        G, T, R = self.world, self.shape.n_theta, self.shape.n_radial
        if G == 1:
            self.hv.copy_(h)
            return
        for k in range(self.chunks):
            self._fwd(h, k).wait()
            rows = slice(k * self.Mk, (k + 1) * self.Mk)
            self.ops.permute(self.recv[k], self.hv[rows], G, self.Mk * T, self.Yl * R)

    def to_home_layout(self, nlv: torch.Tensor, out: torch.Tensor):
        G, T, R = self.world, self.shape.n_theta, self.shape.n_radial
        if G == 1:
            out.copy_(nlv)
            return
        assert out is self.nl
        for k in range(self.chunks):
            rows = slice(k * self.Mk, (k + 1) * self.Mk)
            self.ops.permute(nlv[rows], self.send[k], self.Mk * T, G, self.Yl * R)
            self._back(k).wait()

    def step(self, h: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """h, out: home shards [M][T][Y/G][R] (contiguous complex128)."""
        ops = self.ops
        ops.field(h, self.phi_l)
        nl = None
        if self.nonlinear:
            G, T, R = self.world, self.shape.n_theta, self.shape.n_radial
            if G > 1:
                dist.all_gather_into_tensor(_real(self.phi_g), _real(self.phi_l), group=self.group)
                ops.permute(self.phi_g, self.phi, G, T, self.Yl * R)
            else:
                self.phi.copy_(self.phi_l)
            self._nonlinear(h)
            nl = self.nl
        ops.collision(h, self.buf_c)
        ops.finish(h, nl, self.buf_c, out)
        return out
