"""Multi-rank step on CPU: world_size 2 (and 4) over gloo.

Checks the exchange logic of paper_2305_10553_b200.dist -- home-layout
sharding, the all-to-all transposes, the phi all-gather and the block
permutations -- with the kernels supplied by the CPU oracle (oracle.port), so
no GPU is needed.  The distributed step must equal the single-process oracle
step of the full state.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_2305_10553_b200.dist import DistStepper, shard_bounds
from paper_2305_10553_b200.grid import GridShape, random_state
from paper_2305_10553_b200.kernels import make_kernel_inputs

SHAPE = GridShape(16, 8, 8, 8, 4, 2)  # C1: M = 64, Y = 8
DT = 1e-3


class OracleOps:
    """Same interface as dist.CudaOps, computed by the CPU oracle (test only)."""

    def __init__(self, inputs, y_block, nx, ny):
        self.inp = inputs
        self.shifts = np.asarray(inputs["shifts"])[y_block]
        self.nx, self.ny = nx, ny

    @staticmethod
    def _6d(t):
        m, tt, y, r = t.shape
        return t.numpy().reshape(m, 1, 1, tt, y, r)

    def field(self, h, out):
        w = np.asarray(self.inp["weights"]).reshape(-1, 1, 1)
        out.copy_(torch.from_numpy(port.field(self._6d(h), w)))

    def stream(self, h, out):
        out.copy_(torch.from_numpy(port.stream(self._6d(h), self.inp["stencil"]).reshape(out.shape)))

    def collision(self, h, out):
        out.copy_(torch.from_numpy(port.collision(self._6d(h), self.inp["matrices"]).reshape(out.shape)))

    def nonlinear(self, hv, phi, out, ws):
        res = port.nonlinear(self._6d(hv), phi.numpy(), self.nx, self.ny)
        out.copy_(torch.from_numpy(res.reshape(out.shape)))

    def nonlinear_workspace(self, m_local):
        return torch.empty(1)

    def finish(self, h, nl, c, out):
        s = torch.from_numpy(port.stream(self._6d(h), self.inp["stencil"]).reshape(h.shape))
        rhs = s + nl if nl is not None else s
        out.copy_(torch.from_numpy(port.shear((h + DT * (rhs + c)).numpy(), self.shifts)))

    def permute(self, src, dst, n_a, n_b, inner):
        dst.view(n_b, n_a, inner).copy_(src.reshape(n_a, n_b, inner).transpose(0, 1))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, outdir, nonlinear, chunks=4):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inp = make_kernel_inputs(SHAPE, 7)
        nx, ny = (p.n_padded for p in inp["plans"])
        y0, y1 = shard_bounds(SHAPE.n_toroidal, world, rank)
        ops = OracleOps(inp, slice(y0, y1), nx, ny)
        st = DistStepper(SHAPE, ops, torch.device("cpu"), nonlinear=nonlinear, chunks=chunks)
        h_full = torch.from_numpy(random_state(SHAPE, 7))
        h = st.home_slice(h_full)
        out = torch.empty_like(h)
        st.step(h, out)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), out.numpy())
        if nonlinear:
            # the standalone transposes (bench split) round-trip the home shard
            st.to_nonlinear_layout(h)
            st.nlv.copy_(st.hv)
            st.to_home_layout(st.nlv, st.nl)
            assert torch.equal(st.nl, h)
        if rank == 0:
            np.save(os.path.join(outdir, "comm.npy"), np.array([st.comm_bytes_per_step]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world, nonlinear, chunks", [(2, True, 4), (4, True, 3), (2, False, 1), (2, True, 1)])
def test_distributed_step_matches_single_process(tmp_path, world, nonlinear, chunks):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), nonlinear, chunks), nprocs=world,
                       start_method="spawn")
    inp = make_kernel_inputs(SHAPE, 7)
    nx, ny = (p.n_padded for p in inp["plans"])
    want, _ = port.step(random_state(SHAPE, 7), inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"],
                        DT, nx, ny, nonlinear_on=nonlinear)
    want = want.reshape(SHAPE.velocity_size, SHAPE.n_theta, SHAPE.n_toroidal, SHAPE.n_radial)
    parts = [np.load(tmp_path / f"rank{r}.npy") for r in range(world)]
    got = np.concatenate(parts, axis=2)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-13
    comm = int(np.load(tmp_path / "comm.npy")[0])
    expect = 2 * SHAPE.state_bytes // world * (world - 1) // world if nonlinear else 0
    assert comm == expect  # commsim.alltoall_volume with n1 = world, two transposes


def test_shard_bounds():
    assert shard_bounds(48, 8, 3) == (18, 24)
    with pytest.raises(ValueError):
        shard_bounds(10, 4, 0)
