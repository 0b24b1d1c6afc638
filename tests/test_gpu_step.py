"""GPU parity of the builder-defined step and the
north_star acceptance bar: distribution function and fields within 1e-10
relative L2 of the reference after N steps, on identical inputs."""
import numpy as np
import pytest
import torch

from conftest import ROOT, rel_err, rel_l2
from oracle import port
from paper_2305_10553_b200.grid import GridShape, make_case, random_state
from paper_2305_10553_b200.kernels import (collision_kernel, field_kernel, make_kernel_inputs,
                                           nonlinear_kernel, shear_kernel, stream_kernel)
from paper_2305_10553_b200.step import Stepper

pytestmark = pytest.mark.gpu

C1 = GridShape(16, 8, 8, 8, 4, 2)


def test_c1_ten_steps_match_reference(golden, tables):
    """Reference composition run by the reference package itself (golden)."""
    cfg = tables["step"]
    h = random_state(C1, cfg["seed"])
    inp = make_kernel_inputs(C1, cfg["seed"])
    got = Stepper(C1, inp, cfg["dt"]).run(h, cfg["n"])
    assert rel_l2(got, golden["c1_step10"]) < 1e-10


def test_c1_steps_and_fields_vs_oracle():
    h = random_state(C1, 7)
    inp = make_kernel_inputs(C1, 7)
    nx, ny = (p.n_padded for p in inp["plans"])
    st = Stepper(C1, inp, 1e-3)
    x_gpu = torch.from_numpy(h).cuda()
    x_cpu = h
    for _ in range(10):
        x_gpu = st.step(x_gpu)
        x_cpu, phi_cpu = port.step(x_cpu, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"],
                                   1e-3, nx, ny)
        assert rel_l2(st.phi.cpu().numpy(), phi_cpu) < 1e-10
    assert rel_l2(x_gpu.cpu().numpy(), x_cpu) < 1e-10


def test_benchmark_plan_steps_vs_oracle():
    """North-star bar at a benchmark-like shape: sh03b's grid (720 x 144 plan: the
    warp x kernels and ycol_sq) with 64 velocity rows (int8 tensor-core collision),
    3 steps against the oracle's composition -- h and phi within 1e-10 rel L2."""
    shape = GridShape(480, 48, 8, 8, 8, 1)
    h = random_state(shape, 21)
    inp = make_kernel_inputs(shape, 21)
    nx, ny = (p.n_padded for p in inp["plans"])
    assert (nx, ny) == (720, 144)
    st = Stepper(shape, inp, 1e-4)
    x_gpu, x_cpu = torch.from_numpy(h).cuda(), h
    for _ in range(3):
        x_gpu = st.step(x_gpu)
        x_cpu, phi_cpu = port.step(x_cpu, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"],
                                   1e-4, nx, ny)
        assert rel_l2(st.phi.cpu().numpy(), phi_cpu) < 1e-10
    assert rel_l2(x_gpu.cpu().numpy(), x_cpu) < 1e-10


@pytest.mark.parametrize("dims, plan, inplace", [((1344, 160, 8, 2, 1, 1), (2016, 480), False),   # C5a plan
                                                 ((1344, 288, 8, 1, 1, 1), (2016, 864), True)])   # em04b plan
def test_large_plan_steps_vs_oracle(dims, plan, inplace):
    """2 steps on the multiscale / em04b grids (team x kernels, ycol_rect; em04b
    through the in-place step) against the oracle within 1e-10."""
    shape = GridShape(*dims)
    h = random_state(shape, 22)
    inp = make_kernel_inputs(shape, 22)
    nx, ny = (p.n_padded for p in inp["plans"])
    assert (nx, ny) == plan
    st = Stepper(shape, inp, 1e-4, inplace=inplace)
    x_gpu, x_cpu = torch.from_numpy(h).cuda(), h
    for _ in range(2):
        x_gpu = st.step(x_gpu)
        x_cpu, phi_cpu = port.step(x_cpu, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"],
                                   1e-4, nx, ny)
        assert rel_l2(st.phi.cpu().numpy(), phi_cpu) < 1e-10
    assert rel_l2(x_gpu.cpu().numpy(), x_cpu) < 1e-10


def test_step_equals_composition_of_kernels():
    """gk_step is exactly the composition of the public kernels (same rounding)."""
    shape = make_case("sh03b-desk")
    h = random_state(shape, 3)
    inp = make_kernel_inputs(shape, 3)
    dt = 1e-4
    phi = field_kernel(h, inp["weights"])
    rhs = stream_kernel(h, inp["stencil"]) + nonlinear_kernel(h, phi, inp["plans"])
    rhs = rhs + collision_kernel(h, inp["matrices"])
    want = shear_kernel(h + dt * rhs, inp["shifts"])
    got = Stepper(shape, inp, dt).run(h, 1)
    assert np.array_equal(got, want)


def test_linear_only_path():
    """C2-style single toroidal mode, no bracket (configs[1])."""
    shape = GridShape(24, 1, 8, 6, 4, 3)
    h = random_state(shape, 11)
    inp = make_kernel_inputs(shape, 11)
    got = Stepper(shape, inp, 1e-2, nonlinear=False).run(h, 5)
    x = h
    for _ in range(5):
        x, _ = port.step(x, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"], 1e-2, 0, 0,
                         nonlinear_on=False)
    assert rel_l2(got, x) < 1e-12


def test_step_deterministic_bitwise():
    shape = make_case("em04b-desk")
    h = torch.from_numpy(random_state(shape, 5)).cuda()
    st = Stepper(shape, make_kernel_inputs(shape, 5), 1e-4)
    a = st.step(h).cpu().numpy()
    b = st.step(h).cpu().numpy()
    assert np.array_equal(a, b)
    assert rel_err(a, a) == 0.0


def test_step_stages_compose_to_the_step():
    """gk_step_stage 0..3 on the step's workspace reproduce gk_step bitwise."""
    shape = make_case("sh03b-desk")
    h = torch.from_numpy(random_state(shape, 8)).cuda()
    st = Stepper(shape, make_kernel_inputs(shape, 8), 1e-4)
    want = st.step(h)
    out = torch.empty_like(h)
    for i in range(4):
        st.stage(i, h, out)
    assert torch.equal(out, want)


@pytest.mark.parametrize("case, chunks", [("sh03b-desk", 1), ("sh03b-desk", 2), ("sh03b-desk", 4),
                                          ("sh03b-desk", 9), ("c1-tiny", 3), ("em04b-desk", 2),
                                          # chunks thinner than the stencil reach (2 planes):
                                          ("c1-tiny", 8), ("c1-tiny", 5), ("c1-tiny", 7), ("sh03b-desk", 64),
                                          # the last chunk inside the wrap planes (computed first)
                                          ("em04b-desk", 3), ("em04b-desk", 6), ("sh03b-desk", 16)])
def test_pipelined_host_step_is_bit_identical(case, chunks):
    """gk_step_host (theta-chunked H2D / compute / D2H overlap) == gk_step, bitwise."""
    shape = make_case(case)
    inp = make_kernel_inputs(shape, 4)
    h = torch.from_numpy(random_state(shape, 4))
    st = Stepper(shape, inp, 1e-4)
    want = st.step(h.cuda()).cpu()
    h_host = h.pin_memory()
    # NaN-filled outputs: a (plane, velocity block) the pipeline never finishes or
    # copies back cannot pass on stale memory
    out_host = torch.full_like(h_host, float("nan")).pin_memory()
    out_dev = torch.full_like(h, float("nan")).cuda()
    st.step_host(h_host, out_host, None, out_dev, chunks=chunks)
    torch.cuda.synchronize()
    assert torch.equal(out_host, want)


def test_range_kernels_cover_full_calls():
    from paper_2305_10553_b200 import _lib
    from paper_2305_10553_b200.spectral import get_plan
    shape = make_case("em04b-desk")
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    inp = make_kernel_inputs(shape, 6)
    h = torch.from_numpy(random_state(shape, 6)).cuda()
    w = torch.from_numpy(inp["weights"]).cuda()
    A = torch.from_numpy(inp["matrices"]).cuda()
    phi = torch.from_numpy(inp["phi"]).cuda()
    lib, s = _lib.load(), torch.cuda.current_stream().cuda_stream
    full_f, part_f = torch.empty((T, Y, R), dtype=torch.complex128, device="cuda"), torch.zeros(
        (T, Y, R), dtype=torch.complex128, device="cuda")
    full_c, part_c = torch.empty_like(h), torch.zeros_like(h)
    full_n, part_n = torch.empty_like(h), torch.zeros_like(h)
    nx, ny = (p.n_padded for p in inp["plans"])
    plan = get_plan(R, Y, nx, ny, h.device)
    ws = torch.empty(lib.gk_bracket_workspace_bytes(plan.handle, M * T, T), dtype=torch.uint8, device="cuda")
    _lib.check(lib.gk_field(h.data_ptr(), w.data_ptr(), full_f.data_ptr(), M, T, Y * R, s), "f")
    _lib.check(lib.gk_collision(A.data_ptr(), h.data_ptr(), full_c.data_ptr(), M, T, Y * R, s), "c")
    _lib.check(lib.gk_nonlinear(plan.handle, h.data_ptr(), phi.data_ptr(), full_n.data_ptr(), M, T, ws.data_ptr(),
                                ws.numel(), s), "n")
    for t0, t1 in ((0, 2), (2, 3), (3, T)):
        _lib.check(lib.gk_field_range(h.data_ptr(), w.data_ptr(), part_f.data_ptr(), M, T, Y * R, t0, t1, s), "fr")
        _lib.check(lib.gk_collision_range(A.data_ptr(), h.data_ptr(), part_c.data_ptr(), M, T, Y * R, t0, t1, s),
                   "cr")
        _lib.check(lib.gk_nonlinear_range(plan.handle, h.data_ptr(), phi.data_ptr(), part_n.data_ptr(), M, T, t0,
                                          t1, ws.data_ptr(), ws.numel(), s), "nr")
    assert torch.equal(part_f, full_f) and torch.equal(part_c, full_c) and torch.equal(part_n, full_n)


# ---------------------------------------------------------------- in-place step
# gk_step_inplace: one state-sized workspace buffer; rhs associated as
# stream + (coll + nl) instead of (stream + nl) + coll.

def test_inplace_step_equals_its_composition_of_kernels():
    """The in-place step is exactly shear(h + dt * (stream + (coll + nl))) of the
    public kernels (numpy adds, same rounding sequence)."""
    shape = make_case("sh03b-desk")
    h = random_state(shape, 3)
    inp = make_kernel_inputs(shape, 3)
    dt = 1e-4
    phi = field_kernel(h, inp["weights"])
    rhs = collision_kernel(h, inp["matrices"]) + nonlinear_kernel(h, phi, inp["plans"])
    rhs = stream_kernel(h, inp["stencil"]) + rhs
    want = shear_kernel(h + dt * rhs, inp["shifts"])
    st = Stepper(shape, inp, dt, inplace=True)
    x = torch.from_numpy(h).cuda()
    st.step_inplace(x)
    assert np.array_equal(x.cpu().numpy(), want)
    assert np.array_equal(st.phi.cpu().numpy(), phi)


@pytest.mark.parametrize("dims, nonlinear", [((16, 8, 8, 8, 4, 2), True), ((480, 48, 8, 2, 2, 2), True),
                                             ((24, 1, 8, 6, 4, 3), False)])
def test_inplace_step_matches_step(dims, nonlinear):
    shape = GridShape(*dims)
    h = random_state(shape, 5)
    inp = make_kernel_inputs(shape, 5)
    # one step: the random operators amplify by ~10^3 per step at dt = 1e-3, so
    # over several steps the two associations drift apart by the amplification
    a = Stepper(shape, inp, 1e-4, nonlinear=nonlinear).run(h, 1)
    b = Stepper(shape, inp, 1e-4, nonlinear=nonlinear, inplace=True).run(h, 1)
    assert rel_l2(b, a) < 1e-13
    assert rel_err(b, a) < 1e-12


def test_inplace_c1_ten_steps_match_reference(golden, tables):
    cfg = tables["step"]
    h = random_state(C1, cfg["seed"])
    inp = make_kernel_inputs(C1, cfg["seed"])
    got = Stepper(C1, inp, cfg["dt"], inplace=True).run(h, cfg["n"])
    assert rel_l2(got, golden["c1_step10"]) < 1e-10


def test_nonlinear_acc_adds_onto_out():
    from paper_2305_10553_b200 import _lib
    shape = GridShape(16, 8, 8, 3, 2, 1)
    h, inp = random_state(shape, 8), make_kernel_inputs(shape, 8)
    phi = field_kernel(h, inp["weights"])
    base = random_state(shape, 9)
    want = base + nonlinear_kernel(h, phi, inp["plans"])
    st = Stepper(shape, inp, 1e-3)
    lib = _lib.load()
    ht, pt, ot = (torch.from_numpy(x).cuda() for x in (h, phi, base))
    M, T = shape.velocity_size, shape.n_theta
    wsb = lib.gk_nonlinear_acc_workspace_bytes(st.plan.handle, M, T)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.gk_nonlinear_acc(st.plan.handle, ht.data_ptr(), pt.data_ptr(), ot.data_ptr(), M, T,
                                    ws.data_ptr(), wsb, _lib.stream_of(ht.device)), "gk_nonlinear_acc")
    assert np.array_equal(ot.cpu().numpy(), want)


def test_inplace_rejects_wide_stencils():
    shape = GridShape(16, 8, 12, 2, 2, 1)
    inp = make_kernel_inputs(shape, 1)
    inp["stencil"] = np.ones(11) / 11
    with pytest.raises(ValueError):
        Stepper(shape, inp, 1e-3, inplace=True)


def test_graph_replay_is_bit_identical():
    """Small states replay the step as a CUDA graph: same bits as eager launches,
    re-captured when the buffers change."""
    inp = make_kernel_inputs(C1, 5)
    h = torch.from_numpy(random_state(C1, 5)).cuda()
    eager = Stepper(C1, inp, 1e-3, graph=False)
    graphed = Stepper(C1, inp, 1e-3)
    assert graphed.graph
    a, b = torch.empty_like(h), torch.empty_like(h)
    want = eager.step(h, a).clone()
    for _ in range(3):
        assert torch.equal(graphed.step(h, b), want)
    c = torch.empty_like(h)
    assert torch.equal(graphed.step(h, c), want)  # new buffers: re-captured
    assert torch.equal(graphed.phi, eager.phi)


@pytest.mark.parametrize("graph", [False, True])
def test_reused_matrix_slices_are_bit_identical(graph):
    """The Stepper makes the collision's int8 slices of its matrices on the first
    step and reuses them (gk_step_ex GK_STEP_REUSE_MATRICES): every step equals a
    plain gk_step that slices them again; a caller's device tensor is copied, so
    changing it afterwards does not reach the Stepper."""
    from paper_2305_10553_b200 import _lib
    shape = GridShape(480, 1, 32, 24, 8, 3)  # C2 linear: int8 collision
    inp = make_kernel_inputs(shape, 11)
    dev_inp = dict(inp, matrices=torch.from_numpy(inp["matrices"]).cuda())
    st = Stepper(shape, dev_inp, 1e-4, nonlinear=False, graph=graph)
    assert st.lib.gk_step_workspace_bytes_w(None, len(st.stencil), st.n_vel, 32, 1, 480) > 0
    ref = Stepper(shape, inp, 1e-4, nonlinear=False, graph=False)
    x = torch.from_numpy(random_state(shape, 11)).cuda()
    want = x.clone()
    for _ in range(3):
        x = st.step(x)
        out = torch.empty_like(want)
        s = shape
        _lib.check(ref.lib.gk_step(None, want.data_ptr(), ref.weights.data_ptr(), ref._stencil_c, len(ref.stencil),
                                   ref.matrices.data_ptr(), ref.shifts.data_ptr(), ref.dt, out.data_ptr(),
                                   ref.phi.data_ptr(), ref.n_vel, s.n_theta, s.n_toroidal, s.n_radial,
                                   ref.workspace.data_ptr(), ref.workspace.numel(), _lib.stream_of(x.device)),
                   "gk_step")
        want = out
        assert torch.equal(x, want)
        assert torch.equal(st.phi, ref.phi)
        dev_inp["matrices"].mul_(2.0)  # the caller's tensor, not the Stepper's copy
    with pytest.raises(Exception):
        _lib.check(st.lib.gk_step_ex(None, x.data_ptr(), st.weights.data_ptr(), st._stencil_c, len(st.stencil),
                                     st.matrices.data_ptr(), st.shifts.data_ptr(), st.dt, want.data_ptr(), None,
                                     st.n_vel, 32, 1, 480, st.workspace.data_ptr(), st.workspace.numel(), 4,
                                     _lib.stream_of(x.device)), "gk_step_ex")


def test_stepper_rejects_bad_tensors():
    """Raw pointers cross the C-ABI: wrong dtype / shape / layout / device fail before launching."""
    shape = C1
    st = Stepper(shape, make_kernel_inputs(shape, 3), 1e-3)
    h = torch.from_numpy(random_state(shape, 3)).cuda()
    with pytest.raises(ValueError):
        st.step(h.to(torch.complex64))
    with pytest.raises(ValueError):
        st.step(h.reshape(-1)[:-1].clone())
    with pytest.raises(ValueError):
        st.step(h.transpose(4, 5))
    with pytest.raises(ValueError):
        st.step(h.cpu())
    with pytest.raises(ValueError):
        st.step(h, h)


def test_matrix_slice_reuse_after_dmma_steps_is_safe():
    """A Stepper whose first steps ran on the DMMA collision never sliced A; a later
    int8 step passing the reuse flag must slice A anyway (host-side tag in libgk),
    giving the same bits as a fresh int8 Stepper."""
    from paper_2305_10553_b200 import _lib
    shape = GridShape(480, 48, 8, 8, 8, 1)  # int8-eligible at M = 64
    inp = make_kernel_inputs(shape, 31)
    h = torch.from_numpy(random_state(shape, 31)).cuda()
    lib = _lib.load()
    prev = lib.gk_collision_mode(0)
    try:
        for graph in (False, True):
            st = Stepper(shape, inp, 1e-4, graph=graph)  # auto mode: the workspace has the slice areas
            lib.gk_collision_mode(1)
            out = torch.empty_like(h)
            st.step(h, out)  # DMMA: the A-slice region of the workspace stays unfilled
            lib.gk_collision_mode(0)
            got = st.step(h, out).clone()  # int8, passes GK_STEP_REUSE_MATRICES
            want = Stepper(shape, inp, 1e-4, graph=False).step(h)
            assert torch.equal(got, want), graph
    finally:
        lib.gk_collision_mode(prev)


def test_fused_field_collision_path_is_bit_identical(tmp_path):
    """GK_STEP_SLICES_MAX_GB=0 forces the step's grouped collision with the field
    moment folded into its B slicing (the C5a / in-place path); it must give the
    default path's bits for h' and phi."""
    import subprocess
    import sys
    shape = GridShape(480, 48, 8, 8, 8, 1)
    inp = make_kernel_inputs(shape, 41)
    h = random_state(shape, 41)
    st = Stepper(shape, inp, 1e-4)
    want = st.run(h, 1)
    phi = st.phi.cpu().numpy()
    script = f"""
import sys, numpy as np
sys.path.insert(0, {str(ROOT)!r})
from paper_2305_10553_b200.grid import GridShape, random_state
from paper_2305_10553_b200.kernels import make_kernel_inputs
from paper_2305_10553_b200.step import Stepper
shape = GridShape(480, 48, 8, 8, 8, 1)
st = Stepper(shape, make_kernel_inputs(shape, 41), 1e-4)
out = st.run(random_state(shape, 41), 1)
np.save({str(tmp_path / 'h.npy')!r}, out)
np.save({str(tmp_path / 'phi.npy')!r}, st.phi.cpu().numpy())
"""
    import os
    env = dict(os.environ, GK_STEP_SLICES_MAX_GB="0")
    res = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    assert np.array_equal(np.load(tmp_path / "h.npy"), want)
    assert np.array_equal(np.load(tmp_path / "phi.npy"), phi)


def test_overlapped_host_steps_are_bit_identical():
    """GK_STEP_HOST_OVERLAP: consecutive host-buffer steps on alternating device
    buffer pairs overlap each other's copies; every output equals Stepper.step on
    its own input (different inputs per call, so a stale buffer cannot pass)."""
    shape = make_case("sh03b-desk")
    inp = make_kernel_inputs(shape, 5)
    st = Stepper(shape, inp, 1e-4, graph=False)
    states = [random_state(shape, 50 + i) for i in range(5)]
    hosts = [torch.from_numpy(x).pin_memory() for x in states]
    outs = [torch.full(x.shape, float("nan"), dtype=torch.complex128).pin_memory() for x in states]
    pairs = [(torch.empty(shape.dims, dtype=torch.complex128, device="cuda"),
              torch.empty(shape.dims, dtype=torch.complex128, device="cuda")) for _ in range(2)]
    for i, (hh, oh) in enumerate(zip(hosts, outs)):
        hd, od = pairs[i % 2]
        st.step_host(hh, oh, hd, od, chunks=4, overlap=True)
    st.step_host_join()
    torch.cuda.synchronize()
    for x, oh in zip(states, outs):
        want = st.step(torch.from_numpy(x).cuda()).cpu()
        assert torch.equal(oh, want)
