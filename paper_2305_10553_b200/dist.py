"""Multi-GPU step: toroidal-home layout with all-to-all transposes around the
nonlinear term (SURVEY.md §8 e; no reference code -- the reference only models
this decomposition analytically, commsim.py:1-32, 213-219).

One process per GPU.  Home ("linear") layout: rank g holds h[:, :, :, :, Y_g, :] --
a contiguous block of Y/G toroidal modes, stored [M][T][Y/G][R].  field (full
velocity sum, so no all-reduce and bitwise G-invariant), stream, shear and
collision are local.  The bracket needs every (ky, kx) of a slice, so the
velocity rows travel: the home rows are cut into K chunks of G*Mk rows and rank q
brackets sub-block q of every chunk.  Per chunk k:

  fwd(k)    all-to-all of the chunk's home rows -> recv[G src][Mk][T][Y/G][R]
  bracket   gk_nonlinear_blocked reads that blocked layout in place and writes
            send[G dst][Mk][T][Y/G][R] (no pack / unpack pass)
  back(k)   all-to-all of send -> the chunk's nl rows in home layout
  finish(k) h' = shear(h + dt*((stream + nl) + coll)) of the chunk's rows

with the phi blocks all-gathered once.  Bytes per rank per step: 2 transposes of
S/G*(G-1)/G (= commsim.alltoall_volume with n1=G) plus the phi gather.

``DistStepper`` runs the whole rank step as ONE C-ABI call (gk_dist_step):
NCCL (gk_comm_init, loaded by libgk) on a communication stream pipelined with the
compute by events.  ``DistStepper(..., backend="torch")`` runs the same schedule
in Python over ``torch.distributed`` with the kernels of an ``ops`` object -- the
gloo tests drive it on CPU with the oracle's kernels to check the geometry, the
blocked layouts and the chunk order without a GPU.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._device import on_device
from .grid import GridShape

HBM_BYTES_B200 = 180e9


def _real(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t).reshape(-1)


def shard_bounds(n: int, world: int, rank: int):
    if n % world:
        raise ValueError(f"{n} is not divisible by {world} ranks")
    k = n // world
    return rank * k, (rank + 1) * k


def choose_chunks(n_vel: int, world: int, want: int, nonlinear: bool = True) -> int:
    """Velocity chunks per step: the largest k <= want with n_vel % (world k) == 0."""
    if not nonlinear:
        return 1
    if n_vel % world:
        raise ValueError(f"n_vel {n_vel} is not divisible by {world} ranks")
    k = max(1, min(int(want), n_vel // world))
    while (n_vel // world) % k:
        k -= 1
    return k




def default_backend() -> str:
    """Transport of the multi-GPU step: GK_TRANSPORT=p2p (default: CUDA IPC
    windows, copy-engine pushes, the return transpose fused into the bracket) or
    nccl (NCCL all-to-alls behind the C-ABI)."""
    import os
    return os.environ.get("GK_TRANSPORT", "p2p")


def rank_memory_bytes(shape: GridShape, world: int, chunks: int | None = None, nonlinear: bool = True,
                      backend: str = "p2p") -> dict:
    """Per-rank device memory of DistStepper: the home shard h, the new state h'
    and the rank step's workspace (coll, the collision's int8 slices, the bracket
    workspace, and the 2-deep chunk rings: recv/send/nl in the workspace for NCCL,
    recv/nl + phi blocks in the IPC window for P2P), in bytes."""
    from .spectral import bracket_plans

    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    if chunks is None:
        chunks = auto_chunks(shape, world, nonlinear, backend)
    k = choose_chunks(M, world, chunks, nonlinear)
    nx, ny = ((p.n_padded for p in bracket_plans(R, Y)) if nonlinear else (0, 0))
    lib = _lib.load()
    p2p = backend == "p2p" and nonlinear
    ws = (lib.gk_dist_p2p_workspace_bytes if p2p else lib.gk_dist_workspace_bytes)(nx, ny, M, T, Y, R, world, k)
    shard = shape.state_bytes // world
    window = 0
    if p2p:  # gk_p2p_create: 2 recv + 2 nl chunk slots, 2 phi sets, flags
        a256 = lambda b: (b + 255) // 256 * 256  # noqa: E731
        chunk = (M // k) * T * (Y // world) * R * 16
        window = 2 * a256(2 * chunk) + a256(2 * world * T * (Y // world) * R * 16) + a256(5 * 16 * 4)
    total = 2 * shard + ws + window
    return {"world": world, "chunks": k, "backend": "p2p" if p2p else "nccl", "shard_bytes": shard,
            "workspace_bytes": ws, "window_bytes": window, "total_bytes": total,
            "states_per_rank": total / shard, "fits_180GB": total <= HBM_BYTES_B200}


CHUNK_SLICES = 1536  # target (velocity row, theta) slices per bracket chunk (sh03b, 1 rank: 24 chunks of 768 cost 33.9 ms/step, 12 of 1536 33.0)


def auto_chunks(shape: GridShape, world: int, nonlinear: bool = True, backend: str = "p2p") -> int:
    """Velocity chunks per step: each chunk's bracket should cover ~CHUNK_SLICES
    slices (smaller chunks pay per-launch ramp and tail, larger ones expose more
    of the first and last transfer), as few as the memory budget allows -- more
    chunks shrink the rings: the states that fill a GPU (em04b at 2 ranks, C5b at
    8) take the smallest chunk count that keeps a rank within 4 state shards."""
    if not nonlinear:
        return 1
    per = shape.velocity_size // world
    divisors = [k for k in range(1, per + 1) if per % k == 0]
    target = per * shape.n_theta / CHUNK_SLICES
    cands = [k for k in divisors if k >= target] or [divisors[-1]]
    for k in cands:
        m = rank_memory_bytes(shape, world, k, nonlinear, backend)
        big = shape.state_bytes / world > 16e9
        if m["total_bytes"] <= 0.8 * HBM_BYTES_B200 and (not big or m["states_per_rank"] <= 4.0):
            return k
    return cands[-1]


class NcclComm:
    """A libgk communicator (gk_comm_init: ncclCommInitRank on the current device);
    the 128-byte unique id travels over the torch.distributed group."""

    def __init__(self, group=None):
        self.lib = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = (C.c_char * 128)()
        if self.rank == 0:
            _lib.check(self.lib.gk_comm_unique_id(uid), "gk_comm_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _lib.check(self.lib.gk_comm_init(self.world, self.rank, uid, C.byref(h)), "gk_comm_init")
        self.handle = h

    def info(self):
        n, r, v = C.c_int(), C.c_int(), C.c_int()
        _lib.check(self.lib.gk_comm_info(self.handle, C.byref(n), C.byref(r), C.byref(v)), "gk_comm_info")
        return {"nranks": n.value, "rank": r.value, "nccl_version": v.value}

    def close(self):
        if self.handle:
            self.lib.gk_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class P2PUnavailable(RuntimeError):
    """Some rank could not set up the P2P transport (all ranks raise together)."""


SELFTEST_TIMEOUT_MS = 20000  # generous: the first P2P mapping of a peer window can take a while


class P2PComm:
    """A libgk P2P exchange window (gk_p2p_create: device memory shared by CUDA
    IPC) mapped by every rank; the IPC handles travel over the torch.distributed
    group.  The transposes then need no collective library: copy-engine pushes and
    P2P stores from the FFT kernel, ordered by stream memory operations.

    Set-up failures (no IPC, no peer access, no stream memory operations) are
    agreed on collectively: every rank raises P2PUnavailable, so a caller can fall
    back to another transport without a rank hanging in a collective."""

    def __init__(self, shape: GridShape, chunks: int, group=None):
        self.lib = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.handle = None
        M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
        h = C.c_void_p()
        mine = (C.c_char * 64)()
        err = None
        try:
            _lib.check(self.lib.gk_p2p_create(self.world, self.rank, M, T, Y, R, chunks, C.byref(h)),
                       "gk_p2p_create")
            self.handle = h
            _lib.check(self.lib.gk_p2p_ipc_handle(h, mine), "gk_p2p_ipc_handle")
        except _lib.GkError as e:
            err = str(e)
        every = [None] * self.world
        dist.all_gather_object(every, (err, bytes(mine)), group=group)
        self._agree([e for e, _ in every])
        allh = (C.c_char * (64 * self.world)).from_buffer_copy(b"".join(b for _, b in every))
        err = None
        try:
            _lib.check(self.lib.gk_p2p_connect(h, allh), "gk_p2p_connect")
        except _lib.GkError as e:
            err = str(e)
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)
        self._agree(errs)
        # every path the transport uses must deliver before a step waits on it
        err = None
        try:
            _lib.check(self.lib.gk_p2p_selftest_send(h), "gk_p2p_selftest_send")
        except _lib.GkError as e:
            err = str(e)
        dist.barrier(group=group)
        if err is None:
            try:
                _lib.check(self.lib.gk_p2p_selftest_check(h, SELFTEST_TIMEOUT_MS), "gk_p2p_selftest_check")
            except _lib.GkError as e:
                err = str(e)
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)
        self._agree(errs)

    def _agree(self, errors):
        bad = [(r, e) for r, e in enumerate(errors) if e]
        if bad:
            self.close()
            raise P2PUnavailable("; ".join(f"rank {r}: {e}" for r, e in bad))

    @property
    def window_bytes(self) -> int:
        return self.lib.gk_p2p_window_bytes(self.handle)

    def close(self):
        if self.handle:
            self.lib.gk_p2p_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CudaOps:
    """libgk kernels on device tensors (contiguous complex128), used by the torch
    backend; the NCCL backend calls gk_dist_step, which runs the same kernels."""

    def __init__(self, shape: GridShape, inputs: dict, dt: float, device, y_block: slice, nonlinear=True):
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

    def collision(self, h, out):
        _lib.check(self.lib.gk_collision(self.A.data_ptr(), h.data_ptr(), out.data_ptr(), h.shape[0], h.shape[1],
                                         h.shape[2] * h.shape[3], self._s()), "gk_collision")

    def nonlinear_blocked(self, recv, phi_g, send, m_k, n_blocks, ws):
        """recv/send [G][Mk][T][Y/G][R], phi_g [G][T][Y/G][R] (gk_nonlinear_blocked)."""
        _lib.check(self.lib.gk_nonlinear_blocked(self.plan.handle, recv.data_ptr(), phi_g.data_ptr(),
                                                 send.data_ptr(), m_k, self.shape.n_theta, n_blocks, ws.data_ptr(),
                                                 ws.numel(), self._s()), "gk_nonlinear_blocked")

    def nonlinear_workspace(self, m_local: int) -> torch.Tensor:
        n = self.lib.gk_bracket_workspace_bytes(self.plan.handle, m_local * self.shape.n_theta, self.shape.n_theta)
        return torch.empty(max(n, 16), dtype=torch.uint8, device=self.device)

    def finish(self, h, nl, c, out):
        """out = shear(h + dt * ((stream(h) + nl) + c)) in one pass (gk_step_finish)."""
        _lib.check(self.lib.gk_step_finish(h.data_ptr(), nl.data_ptr() if nl is not None else None, c.data_ptr(),
                                           self._st, len(self.stencil), self.shifts.data_ptr(), self.dt,
                                           out.data_ptr(), h.shape[0], h.shape[1], h.shape[2], h.shape[3],
                                           self._s()), "gk_step_finish")


class DistStepper:
    """One rank's share of the distributed step (toroidal-home layout).

    backend "p2p" (default, GK_TRANSPORT): gk_dist_step_p2p on a P2PComm -- CUDA
    IPC windows, copy-engine pushes and the return transpose fused into the
    bracket's x forward transform (P2P stores), no collective library; checked by
    a connectivity self-test at set-up, falling back to NCCL (all ranks together)
    when it fails.
    backend "nccl": gk_dist_step through the C-ABI on an NcclComm -- the rank step
    as one call, NCCL on its own stream pipelined with the compute.
    backend "torch": the same schedule over torch.distributed with ``ops``'
    kernels (CudaOps, or a CPU oracle in the gloo tests).
    """

    def __init__(self, shape: GridShape, inputs: dict | None = None, dt: float = 0.0, device=None, group=None,
                 nonlinear: bool = True, chunks: int | None = None, backend: str | None = None, ops=None):
        self.shape, self.device, self.group = shape, device, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nonlinear = nonlinear
        backend = backend or (default_backend() if ops is None else "torch")
        if backend == "p2p" and not nonlinear:
            backend = "nccl"  # nothing travels without the bracket: only the local kernels run
        self.backend = backend
        M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
        self.y0, self.y1 = shard_bounds(Y, self.world, self.rank)
        self.Yl = self.y1 - self.y0
        if chunks is None:
            chunks = auto_chunks(shape, self.world, nonlinear, backend or default_backend())
        self.chunks = choose_chunks(M, self.world, chunks, nonlinear)
        self.Mk = M // (self.world * self.chunks) if nonlinear else M
        self.comm_bytes_per_step = 0
        if nonlinear and self.world > 1:
            self.comm_bytes_per_step = 2 * (shape.state_bytes // self.world) * (self.world - 1) // self.world
        if backend in ("nccl", "p2p"):
            with on_device(device):  # windows / communicators / workspaces on the rank's device
                self._init_nccl(inputs, dt)
        elif backend == "torch":
            self._init_torch(ops)
        else:
            raise ValueError(f"unknown backend {backend!r}")

    # ---------------------------------------------------------------- NCCL / C-ABI
    def _init_nccl(self, inputs, dt):
        from .kernels import DEFAULT_STENCIL
        from .spectral import _plan_size, get_plan

        shape, dev = self.shape, self.device
        self.lib = _lib.load()
        self.dt = float(dt)
        if self.backend == "p2p":
            try:
                self.comm = P2PComm(shape, self.chunks, self.group)
            except P2PUnavailable as e:  # every rank lands here together
                import warnings
                warnings.warn(f"P2P transport unavailable ({e}); using NCCL")
                self.backend = "nccl"
        if self.backend != "p2p":
            self.comm = NcclComm(self.group)
        self.weights = torch.from_numpy(np.asarray(inputs["weights"], dtype=float).reshape(-1).copy()).to(dev)
        self.matrices = torch.from_numpy(np.ascontiguousarray(inputs["matrices"], dtype=float)).to(dev)
        self.stencil = np.asarray(inputs.get("stencil", DEFAULT_STENCIL), dtype=float)
        self._st = _lib.doubles(self.stencil)
        sh = np.asarray(inputs["shifts"], dtype=np.int32)[self.y0:self.y1]
        self.shifts = torch.from_numpy(np.ascontiguousarray(sh)).to(dev)
        self.plan = None
        nx = ny = 0
        if self.nonlinear:
            px, py = inputs["plans"]
            nx, ny = _plan_size(px), _plan_size(py)
            self.plan = get_plan(shape.n_radial, shape.n_toroidal, nx, ny, dev)
        M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
        ws_fn = self.lib.gk_dist_p2p_workspace_bytes if self.backend == "p2p" else self.lib.gk_dist_workspace_bytes
        nbytes = ws_fn(nx, ny, M, T, Y, R, self.world, self.chunks)
        if nbytes < 0:
            raise ValueError("gk_dist_workspace_bytes: bad geometry")
        self.workspace = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
        self.phi_l = torch.empty((T, self.Yl, R), dtype=torch.complex128, device=dev)
        self._matrices_sliced = False

    def _args(self, h, out):
        s = self.shape
        return (self.plan.handle if self.plan else None, h.data_ptr(), self.weights.data_ptr(), self._st,
                len(self.stencil), self.matrices.data_ptr(), self.shifts.data_ptr(), self.dt, out.data_ptr())

    def _check(self, t, name):
        want = (self.shape.velocity_size, self.shape.n_theta, self.Yl, self.shape.n_radial)
        if not isinstance(t, torch.Tensor) or t.dtype != torch.complex128 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous complex128 tensor")
        if t.numel() != int(np.prod(want)):
            raise ValueError(f"{name} must hold the home shard {want}")
        if self.backend != "torch" and (not t.is_cuda or t.device != torch.device(self.device)):
            raise ValueError(f"{name} must be on {self.device}")

    def home_slice(self, h_full: torch.Tensor) -> torch.Tensor:
        """This rank's home shard of a full state (..., T, Y, R) -> [M][T][Y/G][R]."""
        M, T = self.shape.velocity_size, self.shape.n_theta
        return h_full.reshape(M, T, self.shape.n_toroidal, self.shape.n_radial)[:, :, self.y0:self.y1].contiguous()

    def step(self, h: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """h, out: home shards [M][T][Y/G][R] (contiguous complex128)."""
        self._check(h, "h")
        self._check(out, "out")
        if self.backend == "torch":
            return self._torch_step(h, out)
        s = self.shape
        flags = 1 if self._matrices_sliced else 0  # GK_STEP_REUSE_MATRICES: this object owns its matrices copy
        with on_device(h.device):
            self._launch_step(h, out, flags)
        self._matrices_sliced = True
        return out

    def _launch_step(self, h, out, flags):
        s = self.shape
        if self.backend == "p2p":
            _lib.check(self.lib.gk_dist_step_p2p(
                self.comm.handle, *self._args(h, out), self.phi_l.data_ptr(), s.velocity_size, s.n_theta,
                s.n_toroidal, s.n_radial, self.workspace.data_ptr(), self.workspace.numel(), flags,
                _lib.stream_of(h.device)), "gk_dist_step_p2p")
        else:
            _lib.check(self.lib.gk_dist_step(
                self.comm.handle, *self._args(h, out), self.phi_l.data_ptr(), s.velocity_size, s.n_theta,
                s.n_toroidal, s.n_radial, self.chunks, self.workspace.data_ptr(), self.workspace.numel(), flags,
                _lib.stream_of(h.device)), "gk_dist_step")

    STAGES = ("field", "nl", "coll", "str", "comm")  # gk_dist_step_stage indices 0..4

    def stage(self, index: int, h: torch.Tensor, out: torch.Tensor) -> None:
        """One stage of the rank step (per-stage timing; NCCL serial on the compute
        stream): field, nl (phi gather + transposes + bracket), coll, str (finish),
        comm (the transposes alone)."""
        with on_device(h.device):
            self._launch_stage(index, h, out)

    def _launch_stage(self, index, h, out):
        s = self.shape
        if self.backend == "p2p":
            if index not in (0, 2, 3):
                raise ValueError("p2p: stages 0 (field), 2 (coll) and 3 (finish) run alone; the nonlinear "
                                 "stage's transfers are fused into it")
            _lib.check(self.lib.gk_dist_step_p2p_stage(
                index, self.comm.handle, *self._args(h, out), self.workspace.data_ptr(), self.workspace.numel(),
                _lib.stream_of(h.device)), "gk_dist_step_p2p_stage")
            return
        _lib.check(self.lib.gk_dist_step_stage(
            index, self.comm.handle, *self._args(h, out), s.velocity_size, s.n_theta, s.n_toroidal, s.n_radial,
            self.chunks, self.workspace.data_ptr(), self.workspace.numel(), _lib.stream_of(h.device)),
            "gk_dist_step_stage")

    # ---------------------------------------------------------------- torch.distributed
    def _init_torch(self, ops):
        if ops is None:
            raise ValueError("backend='torch' needs an ops object")
        self.ops = ops
        M, T, R = self.shape.velocity_size, self.shape.n_theta, self.shape.n_radial
        G, Yl, dev = self.world, self.Yl, self.device
        c128 = dict(dtype=torch.complex128, device=dev)
        self.coll = torch.empty((M, T, Yl, R), **c128)
        self.phi_l = torch.empty((T, Yl, R), **c128)
        if self.nonlinear:
            self.phi_g = torch.empty((G, T, Yl, R), **c128)
            ring = (2, G, self.Mk, T, Yl, R)
            self.recv, self.send = torch.empty(ring, **c128), torch.empty(ring, **c128)
            self.nl = torch.empty((2, G * self.Mk, T, Yl, R), **c128)
            self.ws = ops.nonlinear_workspace(self.Mk)

    def _chunk(self, a: torch.Tensor, k: int) -> torch.Tensor:
        """Home rows of chunk k: G*Mk contiguous velocity rows; rank q brackets the
        q-th Mk of them."""
        n = self.world * self.Mk
        return a[k * n:(k + 1) * n]

    def _torch_step(self, h, out):
        """gk_dist_step's schedule (dist.cu) over torch.distributed: fwd(k+1) in
        flight while chunk k is bracketed, back(k) while chunk k+1 computes, the
        same 2-deep rings."""
        ops, G, K, grp = self.ops, self.world, self.chunks, self.group
        ops.field(h, self.phi_l)
        if not self.nonlinear:
            ops.collision(h, self.coll)
            ops.finish(h, None, self.coll, out)
            return out
        fwd = lambda k: dist.all_to_all_single(_real(self.recv[k % 2]), _real(self._chunk(h, k)),  # noqa: E731
                                               group=grp, async_op=True)
        pend = {0: fwd(0)}
        dist.all_gather_into_tensor(_real(self.phi_g), _real(self.phi_l), group=grp)
        if K > 1:
            pend[1] = fwd(1)
        ops.collision(h, self.coll)
        backs = {}
        for k in range(K):
            pend.pop(k).wait()
            ops.nonlinear_blocked(self.recv[k % 2], self.phi_g, self.send[k % 2], self.Mk, G, self.ws)
            backs[k] = dist.all_to_all_single(_real(self.nl[k % 2]), _real(self.send[k % 2]), group=grp,
                                              async_op=True)
            if k + 2 < K:
                pend[k + 2] = fwd(k + 2)
            if k >= 1:
                backs.pop(k - 1).wait()
                ops.finish(self._chunk(h, k - 1), self.nl[(k - 1) % 2], self._chunk(self.coll, k - 1),
                           self._chunk(out, k - 1))
        backs.pop(K - 1).wait()
        ops.finish(self._chunk(h, K - 1), self.nl[(K - 1) % 2], self._chunk(self.coll, K - 1),
                   self._chunk(out, K - 1))
        return out
