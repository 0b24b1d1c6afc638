"""GPU pieces of the multi-GPU path that one GPU can exercise.

* gk_nonlinear_blocked (the bracket reading / writing a transpose's blocked
  layout) against gk_nonlinear on the contiguous arrays -- bitwise;
* gk_dist_step_sim: G ranks of the C++ rank step (gk_dist_step's phases, chunk
  rings and blocked layouts) in lock-step on one device, the exchanges as device
  copies -- bitwise equal to the single-GPU step for G = 1..8;
* the NCCL path through the C-ABI at world size 1 (gk_comm_init, gk_dist_step,
  the transposes) -- bitwise equal to Stepper.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2305_10553_b200 import _lib
from paper_2305_10553_b200.dist import CudaOps, DistStepper, NcclComm, choose_chunks
from paper_2305_10553_b200.grid import GridShape, make_case, random_state
from paper_2305_10553_b200.kernels import make_kernel_inputs
from paper_2305_10553_b200.spectral import _plan_size, get_plan
from paper_2305_10553_b200.step import Stepper

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_a, n_b, inner", [(2, 3, 5), (8, 576 * 4, 6 * 480 // 40), (1, 7, 1), (5, 1, 9)])
def test_permute_blocks_bitwise(n_a, n_b, inner):
    src = torch.randn((n_a, n_b, inner), dtype=torch.complex128, device="cuda")
    dst = torch.empty((n_b, n_a, inner), dtype=torch.complex128, device="cuda")
    lib = _lib.load()
    _lib.check(lib.gk_permute_blocks(src.data_ptr(), dst.data_ptr(), n_a, n_b, inner,
                                     torch.cuda.current_stream().cuda_stream), "permute")
    assert torch.equal(dst, src.transpose(0, 1).contiguous())


def _blocked(a, G):
    """[M][T][Y][R] -> [G][M][T][Y/G][R] (a transpose's receive layout)."""
    M, T, Y, R = a.shape
    return a.reshape(M, T, G, Y // G, R).permute(2, 0, 1, 3, 4).contiguous()


@pytest.mark.parametrize("dims, G", [((480, 48, 4, 4, 2, 1), 4),    # 720 x 144: warp x kernels, ycol_sq
                                     ((16, 8, 8, 8, 4, 2), 2),       # C1: generic engine
                                     ((1344, 160, 2, 2, 1, 1), 8),   # 2016 x 480: team x kernels, ycol_rect
                                     ((480, 48, 2, 1, 1, 1), 1)])
def test_nonlinear_blocked_equals_contiguous(dims, G):
    shape = GridShape(*dims)
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    inp = make_kernel_inputs(shape, 5)
    px, py = inp["plans"]
    plan = get_plan(R, Y, _plan_size(px), _plan_size(py), torch.device("cuda", 0))
    h = torch.from_numpy(random_state(shape, 5)).cuda().reshape(M, T, Y, R)
    phi = torch.from_numpy(random_state(GridShape(R, Y, T, 1, 1, 1), 6)).cuda().reshape(T, Y, R)
    lib = _lib.load()
    ws = torch.empty(lib.gk_bracket_workspace_bytes(plan.handle, M * T, T), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    want = torch.empty_like(h)
    _lib.check(lib.gk_nonlinear(plan.handle, h.data_ptr(), phi.data_ptr(), want.data_ptr(), M, T, ws.data_ptr(),
                                ws.numel(), st), "gk_nonlinear")
    hb, phib = _blocked(h, G), _blocked(phi[None], G)[:, 0].contiguous()
    got = torch.full_like(hb, float("nan"))
    _lib.check(lib.gk_nonlinear_blocked(plan.handle, hb.data_ptr(), phib.data_ptr(), got.data_ptr(), M, T, G,
                                        ws.data_ptr(), ws.numel(), st), "gk_nonlinear_blocked")
    assert torch.equal(got, _blocked(want, G))


def _sim_step(shape, inp, dt, G, chunks, nonlinear=True):
    """G ranks of gk_dist_step on this device (gk_dist_step_sim); returns the full
    new state and phi assembled from the ranks' home shards."""
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    K = choose_chunks(M, G, chunks, nonlinear)
    h = torch.from_numpy(random_state(shape, 9)).to(dev).reshape(M, T, Y, R)
    Yl = Y // G
    homes = [h[:, :, g * Yl:(g + 1) * Yl].contiguous() for g in range(G)]
    outs = [torch.full_like(x, float("nan")) for x in homes]
    phis = [torch.empty((T, Yl, R), dtype=torch.complex128, device=dev) for _ in range(G)]
    sh = np.asarray(inp["shifts"], dtype=np.int32)
    shifts = [torch.from_numpy(np.ascontiguousarray(sh[g * Yl:(g + 1) * Yl])).to(dev) for g in range(G)]
    plan, nx, ny = None, 0, 0
    if nonlinear:
        px, py = inp["plans"]
        nx, ny = _plan_size(px), _plan_size(py)
        plan = get_plan(R, Y, nx, ny, dev)
    nbytes = lib.gk_dist_workspace_bytes(nx, ny, M, T, Y, R, G, K)
    wss = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(G)]
    w = torch.from_numpy(np.asarray(inp["weights"], dtype=float).reshape(-1).copy()).to(dev)
    A = torch.from_numpy(np.ascontiguousarray(inp["matrices"], dtype=float)).to(dev)
    arr = lambda ts: (C.c_void_p * G)(*[t.data_ptr() for t in ts])  # noqa: E731
    stencil = _lib.doubles(inp["stencil"])
    _lib.check(lib.gk_dist_step_sim(G, plan.handle if plan else None, arr(homes), w.data_ptr(), stencil,
                                    len(inp["stencil"]), A.data_ptr(), arr(shifts), dt, arr(outs), arr(phis), M, T, Y,
                                    R, K, arr(wss), nbytes, torch.cuda.current_stream().cuda_stream),
               "gk_dist_step_sim")
    return h, torch.cat(outs, dim=2), torch.cat(phis, dim=1)


@pytest.mark.parametrize("dims, G, chunks", [((16, 8, 8, 8, 4, 2), 2, 4),        # C1, DMMA collision
                                             ((16, 8, 8, 8, 4, 2), 4, 3),
                                             ((16, 8, 8, 8, 4, 2), 8, 1),
                                             ((480, 48, 8, 8, 8, 1), 2, 4),      # sh03b plan, int8 collision
                                             ((480, 48, 8, 8, 8, 1), 8, 2),
                                             ((480, 48, 8, 8, 8, 1), 1, 3),
                                             ((1344, 160, 8, 2, 1, 1), 2, 1),    # C5a plan: team x, ycol_rect
                                             ((1344, 288, 8, 4, 1, 1), 4, 1)])   # em04b plan
def test_dist_step_sim_equals_single_gpu_step(dims, G, chunks):
    """The rank step at G ranks (layouts, rings, chunk order, field blocks, shears)
    is bit-identical to gk_step on the whole state."""
    shape = GridShape(*dims)
    inp = make_kernel_inputs(shape, 9)
    h, got, phi = _sim_step(shape, inp, 1e-4, G, chunks)
    st = Stepper(shape, inp, 1e-4, graph=False)
    want = st.step(h.reshape(shape.dims).contiguous())
    assert torch.equal(got.reshape(want.shape), want)
    assert torch.equal(phi, st.phi)


def test_dist_step_sim_linear_only():
    shape = GridShape(480, 4, 8, 8, 8, 1)  # M = 64: int8 collision, no bracket
    inp = make_kernel_inputs(shape, 12)
    h, got, phi = _sim_step(shape, inp, 1e-3, 2, 1, nonlinear=False)
    st = Stepper(shape, inp, 1e-3, nonlinear=False, graph=False)
    want = st.step(h.reshape(shape.dims).contiguous())
    assert torch.equal(got.reshape(want.shape), want)


def test_dist_step_sim_grouped_collision(tmp_path):
    """With the B slices over the cap (GK_STEP_SLICES_MAX_GB=0: the C5b / em04b
    path), the rank's grouped collision computes the field moment too -- same bits."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = f"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {os.path.join(root, 'tests')!r})
from test_gpu_dist_kernels import _sim_step
from paper_2305_10553_b200.grid import GridShape
from paper_2305_10553_b200.kernels import make_kernel_inputs
shape = GridShape(480, 48, 8, 8, 8, 1)
h, got, phi = _sim_step(shape, make_kernel_inputs(shape, 9), 1e-4, 4, 2)
torch.save((got.cpu(), phi.cpu()), {str(tmp_path / 'g.pt')!r})
"""
    res = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, GK_STEP_SLICES_MAX_GB="0"),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    got, phi = torch.load(tmp_path / "g.pt")
    shape = GridShape(480, 48, 8, 8, 8, 1)
    inp = make_kernel_inputs(shape, 9)
    st = Stepper(shape, inp, 1e-4, graph=False)
    h = torch.from_numpy(random_state(shape, 9)).cuda()
    want = st.step(h)
    assert torch.equal(got.reshape(want.shape), want.cpu())
    assert torch.equal(phi, st.phi.cpu())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture
def nccl_world1():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        yield dev
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case, chunks", [("sh03b-desk", 4), ("c1", 2)])
def test_single_rank_nccl_dist_stepper_equals_stepper(nccl_world1, case, chunks):
    """world_size 1: gk_comm_init + gk_dist_step (NCCL transposes to self) == Stepper
    (bitwise), twice (the second step reuses the collision matrices' slices)."""
    dev = nccl_world1
    shape = GridShape(16, 8, 8, 8, 4, 2) if case == "c1" else make_case(case)
    inp = make_kernel_inputs(shape, 3)
    h = torch.from_numpy(random_state(shape, 3)).to(dev)
    ds = DistStepper(shape, inp, 1e-4, dev, chunks=chunks, backend="nccl")
    info = ds.comm.info()
    assert info["nranks"] == 1 and info["rank"] == 0 and info["nccl_version"] > 20000
    st = Stepper(shape, inp, 1e-4, device=dev, graph=False)
    hh = ds.home_slice(h)
    out = torch.empty_like(hh)
    x = h
    for _ in range(2):
        ds.step(hh, out)
        x = st.step(x)
        assert torch.equal(out.reshape(x.shape), x)
        assert torch.equal(ds.phi_l, st.phi)
        hh, out = out, hh


def test_nccl_transposes_and_gather_through_c_abi(nccl_world1):
    """gk_transpose_to_nl / to_lin / gk_comm_allgather at world size 1 move the
    blocks exactly (self-exchange), on the caller's stream."""
    dev = nccl_world1
    comm = NcclComm()
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    src = torch.randn((6, 3, 5), dtype=torch.complex128, device=dev)
    dst = torch.empty_like(src)
    _lib.check(lib.gk_transpose_to_nl(comm.handle, src.data_ptr(), dst.data_ptr(), 6, 15, st), "to_nl")
    back = torch.empty_like(src)
    _lib.check(lib.gk_transpose_to_lin(comm.handle, dst.data_ptr(), back.data_ptr(), 6, 15, st), "to_lin")
    g = torch.empty_like(src)
    _lib.check(lib.gk_comm_allgather(comm.handle, src.data_ptr(), g.data_ptr(), src.numel(), st), "allgather")
    torch.cuda.synchronize()
    assert torch.equal(dst, src) and torch.equal(back, src) and torch.equal(g, src)
    comm.close()


def test_torch_backend_with_cuda_ops_equals_stepper(nccl_world1):
    """The Python schedule (backend='torch', the one the gloo tests check) with the
    libgk kernels (gk_nonlinear_blocked, gk_step_finish on chunks) == Stepper."""
    dev = nccl_world1
    shape = make_case("sh03b-desk")
    inp = make_kernel_inputs(shape, 4)
    h = torch.from_numpy(random_state(shape, 4)).to(dev)
    ops = CudaOps(shape, inp, 1e-4, dev, slice(0, shape.n_toroidal))
    ds = DistStepper(shape, device=dev, chunks=3, backend="torch", ops=ops)
    hh = ds.home_slice(h)
    out = torch.empty_like(hh)
    ds.step(hh, out)
    want = Stepper(shape, inp, 1e-4, device=dev, graph=False).step(h)
    assert torch.equal(out.reshape(want.shape), want)


@pytest.mark.parametrize("chunks", [1, 3])
def test_single_rank_p2p_dist_stepper_equals_stepper(nccl_world1, chunks):
    """world_size 1 over the P2P transport (window, flags, no peers) == Stepper."""
    dev = nccl_world1
    shape = make_case("sh03b-desk")
    inp = make_kernel_inputs(shape, 3)
    h = torch.from_numpy(random_state(shape, 3)).to(dev)
    ds = DistStepper(shape, inp, 1e-4, dev, chunks=chunks, backend="p2p")
    st = Stepper(shape, inp, 1e-4, device=dev, graph=False)
    hh = ds.home_slice(h)
    out = torch.empty_like(hh)
    x = h
    for _ in range(2):
        ds.step(hh, out)
        x = st.step(x)
        assert torch.equal(out.reshape(x.shape), x)
        hh, out = out, hh
