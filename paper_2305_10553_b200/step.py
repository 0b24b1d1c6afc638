"""Builder-defined time step over the reference's kernels.

The reference exposes no step/RHS function (its compute API is the five kernels,
kernels.py:45-150), so the step is the composition of exactly those kernels:

    phi = field(h, w)
    rhs = (stream(h, c) + nonlinear(h, phi, plans)) + collision(h, A)
    h'  = shear(h + dt * rhs, shifts)

``Stepper`` keeps every auxiliary input, the spectral plan and the workspace
resident on the device and runs the whole step as one C-ABI call (gk_step);
its CPU counterpart (used only by tests and the bench's CPU baseline) is
``oracle.port.step``.  ``nonlinear=False`` is the linear-only path (config C2,
single toroidal mode, no bracket).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._device import device_method, require_cuda, to_device
from .grid import GridShape
from .kernels import DEFAULT_STENCIL
from .spectral import _plan_size, get_plan

GK_STEP_REUSE_MATRICES = 1  # include/gk.h


class Stepper:
    """``inplace=True``: the in-place step (gk_step_inplace) -- ``step_inplace(h)``
    overwrites h and the workspace holds one state-sized buffer instead of two plus
    the output, for states that do not fit gk_step's ~4 state buffers (em04b on one
    GPU).  Its rhs is associated as stream + (coll + nl) instead of
    (stream + nl) + coll, so it agrees with ``step`` to a few ulps of the rhs."""

    #: states up to this size replay the step as a CUDA graph (launch-bound sizes)
    GRAPH_MAX_STATE_BYTES = 256 << 20

    def __init__(self, shape: GridShape, inputs: dict, dt: float, nonlinear: bool = True, device=None,
                 inplace: bool = False, graph: bool | None = None):
        self.device = device or require_cuda()
        self._setup(shape, inputs, dt, nonlinear, inplace, graph)

    @device_method  # plans, workspaces and kernel attributes on the Stepper's device
    def _setup(self, shape, inputs, dt, nonlinear, inplace, graph):
        self.shape = shape
        self.dt = float(dt)
        self.nonlinear = bool(nonlinear)
        dev = self.device
        self.weights = to_device(inputs["weights"], torch.float64, dev)[0]
        m = inputs["matrices"]
        self.matrices = to_device(m, torch.float64, dev)[0]
        if isinstance(m, torch.Tensor) and self.matrices.data_ptr() == m.data_ptr():
            self.matrices = self.matrices.clone()  # owned: the steps reuse its int8 slices
        # the collision's int8 slices of `matrices` are made by the first step and
        # kept in the workspace (gk_step_ex GK_STEP_REUSE_MATRICES) -- the Stepper
        # owns its copy of the matrices, so they cannot change between steps
        self._matrices_sliced = False
        self.stencil = np.asarray(inputs.get("stencil", DEFAULT_STENCIL), dtype=float)
        shifts = np.asarray(inputs["shifts"], dtype=int)
        if shifts.shape != (shape.n_toroidal,) or np.any(np.abs(shifts) > shape.n_radial):
            raise ValueError("bad shear shifts")
        if self.stencil.shape[0] % 2 == 0 or self.stencil.shape[0] > shape.n_theta:
            raise ValueError("bad stream stencil")
        self.shifts = torch.from_numpy(shifts.astype(np.int32)).to(dev)
        self._stencil_c = _lib.doubles(self.stencil)
        self.lib = _lib.load()
        self.plan = None
        if self.nonlinear:
            plan_x, plan_y = inputs["plans"]
            self.n_x, self.n_y = _plan_size(plan_x), _plan_size(plan_y)
            self.plan = get_plan(shape.n_radial, shape.n_toroidal, self.n_x, self.n_y, dev)
        handle = self.plan.handle if self.plan else None
        self.n_vel = shape.velocity_size
        self.inplace = bool(inplace)
        if self.inplace:
            if len(self.stencil) > 9:
                raise ValueError("the in-place step supports stencil widths up to 9")
            nbytes = self.lib.gk_step_inplace_workspace_bytes(handle, self.n_vel, shape.n_theta, shape.n_toroidal,
                                                              shape.n_radial)
        else:
            nbytes = self.lib.gk_step_workspace_bytes_w(handle, len(self.stencil), self.n_vel, shape.n_theta,
                                                        shape.n_toroidal, shape.n_radial)
        self.workspace = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
        self.phi = torch.empty(shape.field_dims, dtype=torch.complex128, device=dev)
        # small states are launch-bound (~47 kernels per step): step() captures the
        # step for a (h, out) pair once and replays it (C1: 0.073 -> 0.060 ms/step)
        self.graph = (shape.state_bytes <= self.GRAPH_MAX_STATE_BYTES) if graph is None else bool(graph)
        self.graph = self.graph and not self.inplace
        self._graph = None
        self._graph_key = None
        self._graph_kernels = 0    # kernels one replay launches (counted during the capture)
        self.replayed_kernels = 0  # kernels launched by graph replays so far (gk_launch_counter misses them)

    def _check(self, t, name: str, host: bool = False) -> None:
        """The C-ABI gets raw pointers: reject anything that is not a contiguous
        complex128 state of this shape on this Stepper's device (or, host=True, in
        host memory) before launching."""
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch tensor")
        if t.dtype != torch.complex128:
            raise ValueError(f"{name} must be complex128, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if t.numel() != self.shape.state_bytes // 16:
            raise ValueError(f"{name} has {t.numel()} elements, the state has {self.shape.state_bytes // 16}")
        if host:
            if t.is_cuda:
                raise ValueError(f"{name} must be in host memory")
        else:
            want = torch.device(self.device)
            idx = want.index if want.index is not None else torch.cuda.current_device()
            if not t.is_cuda or t.device.index != idx:
                raise ValueError(f"{name} must be on cuda:{idx}, got {t.device}")

    @device_method
    def step_inplace(self, h: torch.Tensor, stage: int = -1) -> torch.Tensor:
        """One in-place step (needs ``inplace=True``): h is overwritten by the new state.
        ``stage`` 0..3 runs one stage (field, collision, nonlinear, finish) for timing."""
        if not self.inplace:
            raise ValueError("Stepper(inplace=True) required")
        self._check(h, "h")
        s = self.shape
        _lib.check(self.lib.gk_step_inplace(
            int(stage), self.plan.handle if self.plan else None, h.data_ptr(), self.weights.data_ptr(),
            self._stencil_c, len(self.stencil), self.matrices.data_ptr(), self.shifts.data_ptr(), self.dt,
            self.phi.data_ptr() if stage < 0 else None, self.n_vel, s.n_theta, s.n_toroidal, s.n_radial,
            self.workspace.data_ptr(), self.workspace.numel(), _lib.stream_of(h.device)), "gk_step_inplace")
        return h

    @device_method
    def step(self, h: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """One step on a device-resident state; returns the new state (h untouched)."""
        if self.inplace:
            if out is None:
                out = h.clone()
            elif out.data_ptr() != h.data_ptr():
                out.copy_(h)
            return self.step_inplace(out)
        if out is None:
            out = torch.empty_like(h)
        self._check(h, "h")
        self._check(out, "out")
        if out.data_ptr() == h.data_ptr():
            raise ValueError("out must not alias h (use Stepper(inplace=True))")
        if self.graph:
            # a replay repeats the captured kernels: recapture when the collision
            # arithmetic (gk_collision_mode) changed since the capture
            key = (h.data_ptr(), out.data_ptr(), self.lib.gk_collision_mode(-1))
            if key != self._graph_key:
                self._capture(h, out)
                self._graph_key = key
            self._graph.replay()
            self.replayed_kernels += self._graph_kernels
            return out
        self._launch(h, out)
        return out

    def _launch(self, h: torch.Tensor, out: torch.Tensor) -> None:
        s = self.shape
        _lib.check(self.lib.gk_step_ex(
            self.plan.handle if self.plan else None, h.data_ptr(), self.weights.data_ptr(), self._stencil_c,
            len(self.stencil), self.matrices.data_ptr(), self.shifts.data_ptr(), self.dt, out.data_ptr(),
            self.phi.data_ptr(), self.n_vel, s.n_theta, s.n_toroidal, s.n_radial, self.workspace.data_ptr(),
            self.workspace.numel(), GK_STEP_REUSE_MATRICES if self._matrices_sliced else 0,
            _lib.stream_of(h.device)), "gk_step_ex")
        self._matrices_sliced = True

    def _capture(self, h: torch.Tensor, out: torch.Tensor) -> None:
        """Record gk_step for this (h, out) pair as a CUDA graph (same kernels,
        same arguments; replays are bit-identical to eager launches)."""
        side = torch.cuda.Stream(device=h.device)
        side.wait_stream(torch.cuda.current_stream(h.device))
        with torch.cuda.stream(side):
            self._launch(h, out)  # warm-up outside the capture (plans, kernel attributes, pools)
            g = torch.cuda.CUDAGraph()
            n0 = self.lib.gk_launch_counter()
            with torch.cuda.graph(g, stream=side):
                self._launch(h, out)
            self._graph_kernels = self.lib.gk_launch_counter() - n0
        torch.cuda.current_stream(h.device).wait_stream(side)
        self._graph = g

    GK_STEP_HOST_OVERLAP = 2  # include/gk.h

    @device_method
    def step_host(self, h_host: torch.Tensor, out_host: torch.Tensor, h_dev: torch.Tensor | None = None,
                  out_dev: torch.Tensor | None = None, chunks: int = 16, overlap: bool = False) -> torch.Tensor:
        """One step with the state in (pinned) host memory, PCIe overlapped with compute.

        Copies h_host -> device, steps, copies the result -> out_host, pipelined
        over ``chunks`` theta chunks, each moved and finished as velocity blocks
        (GK_E2E_VBLOCKS, default 4; gk_step_host).  Bit-identical to step().
        Asynchronous on the current stream; synchronise before reading out_host.

        ``overlap=True`` (gk_step_host_ex, GK_STEP_HOST_OVERLAP): consecutive calls
        on alternating (h_dev, out_dev) pairs also overlap each other -- a call's
        copy-in runs during the previous call's compute and copy-out tail.  Call
        ``step_host_join()`` before reading out_host.
        """
        s = self.shape
        if h_dev is None:
            h_dev = torch.empty(h_host.shape, dtype=torch.complex128, device=self.device)
        if out_dev is None:
            out_dev = torch.empty_like(h_dev)
        self._check(h_host, "h_host", host=True)
        self._check(out_host, "out_host", host=True)
        self._check(h_dev, "h_dev")
        self._check(out_dev, "out_dev")
        flags = self.GK_STEP_HOST_OVERLAP if overlap else 0
        _lib.check(self.lib.gk_step_host_ex(
            self.plan.handle if self.plan else None, h_host.data_ptr(), h_dev.data_ptr(), out_dev.data_ptr(),
            out_host.data_ptr(), self.weights.data_ptr(), self._stencil_c, len(self.stencil),
            self.matrices.data_ptr(), self.shifts.data_ptr(), self.dt, self.n_vel, s.n_theta, s.n_toroidal,
            s.n_radial, int(chunks), self.workspace.data_ptr(), self.workspace.numel(), flags,
            _lib.stream_of(self.device)), "gk_step_host_ex")
        return out_host

    @device_method
    def step_host_join(self) -> None:
        """The current stream waits for the last copy-out of overlapped step_host calls."""
        _lib.check(self.lib.gk_step_host_join(_lib.stream_of(self.device)), "gk_step_host_join")

    STAGES = ("field", "nl", "coll", "str")  # gk_step_stage indices 0..3 ("str" = fused finish pass)

    @device_method
    def stage(self, index: int, h: torch.Tensor, out: torch.Tensor | None) -> None:
        """Run one stage of the step on the step's own workspace (per-stage timing).
        In-place steppers run the same stage of gk_step_inplace (out unused; the
        finish stage overwrites h)."""
        if self.inplace:
            self.step_inplace(h, (0, 2, 1, 3)[index])
            return
        self._check(h, "h")
        self._check(out, "out")
        s = self.shape
        _lib.check(self.lib.gk_step_stage(
            index, self.plan.handle if self.plan else None, h.data_ptr(), self.weights.data_ptr(), self._stencil_c,
            len(self.stencil), self.matrices.data_ptr(), self.shifts.data_ptr(), self.dt, out.data_ptr(), self.n_vel,
            s.n_theta, s.n_toroidal, s.n_radial, self.workspace.data_ptr(), self.workspace.numel(),
            _lib.stream_of(h.device)), "gk_step_stage")

    @device_method
    def run(self, h, n_steps: int):
        """n steps from h (numpy or tensor); returns the final state the way h came in."""
        x, carrier = to_device(h, torch.complex128, self.device)
        a, b = x.clone(), torch.empty_like(x)
        for _ in range(n_steps):
            self.step(a, b)
            a, b = b, a
        return carrier.back(a)


def step(h, inputs: dict, dt: float, nonlinear: bool = True):
    """Functional one-step API (numpy in -> numpy out)."""
    shape = GridShape(*(lambda d: (d[5], d[4], d[3], d[2], d[1], d[0]))(tuple(np.shape(h))))
    return Stepper(shape, inputs, dt, nonlinear).run(h, 1)
