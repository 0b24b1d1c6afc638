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
from paper_2305_10553_b200.dist import DistStepper, choose_chunks, shard_bounds
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

    def collision(self, h, out):
        out.copy_(torch.from_numpy(port.collision(self._6d(h), self.inp["matrices"]).reshape(out.shape)))

    def nonlinear_blocked(self, recv, phi_g, send, m_k, n_blocks, ws):
        """recv/send [G][Mk][T][Y/G][R], phi_g [G][T][Y/G][R] -- the layouts
        gk_nonlinear_blocked reads and writes on the GPU."""
        G, Mk, T, Yl, R = recv.shape
        hv = recv.permute(1, 2, 0, 3, 4).reshape(Mk, T, G * Yl, R)
        phi = phi_g.permute(1, 0, 2, 3).reshape(T, G * Yl, R)
        res = torch.from_numpy(port.nonlinear(self._6d(hv), phi.numpy(), self.nx, self.ny).reshape(Mk, T, G, Yl, R))
        send.copy_(res.permute(2, 0, 1, 3, 4))

    def nonlinear_workspace(self, m_local):
        return torch.empty(1)

    def finish(self, h, nl, c, out):
        s = torch.from_numpy(port.stream(self._6d(h), self.inp["stencil"]).reshape(h.shape))
        rhs = s + nl if nl is not None else s
        out.copy_(torch.from_numpy(port.shear((h + DT * (rhs + c)).numpy(), self.shifts)))


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
        st = DistStepper(SHAPE, device=torch.device("cpu"), nonlinear=nonlinear, chunks=chunks, backend="torch",
                         ops=ops)
        assert (st.y0, st.y1) == (y0, y1)
        h_full = torch.from_numpy(random_state(SHAPE, 7))
        h = st.home_slice(h_full)
        out = torch.empty_like(h)
        st.step(h, out)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), out.numpy())
        if rank == 0:
            np.save(os.path.join(outdir, "comm.npy"), np.array([st.comm_bytes_per_step]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world, nonlinear, chunks", [(2, True, 4), (4, True, 3), (2, False, 1), (2, True, 1),
                                                     (2, True, 2)])
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


def test_choose_chunks():
    assert choose_chunks(576, 8, 4) == 4       # sh03b at 8 ranks: 72 rows, 4 chunks of 18
    assert choose_chunks(432, 8, 4) == 3       # em04b: 54 rows -> 3 chunks of 18
    assert choose_chunks(64, 4, 3) == 2
    assert choose_chunks(64, 2, 4, nonlinear=False) == 1


def _unique_id_worker(rank, world, port_no, outdir):
    """The communicator's 128-byte id travels over the torch.distributed group as
    NcclComm sends it (broadcast_object_list from rank 0); gloo here."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        np.save(os.path.join(outdir, f"id{rank}.npy"), np.frombuffer(obj[0], dtype=np.uint8))
    finally:
        dist.destroy_process_group()


def test_unique_id_broadcast(tmp_path):
    mp.start_processes(_unique_id_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"id{r}.npy"), np.arange(128, dtype=np.uint8))


@pytest.mark.parametrize("case, world", [("sh03b", 2), ("sh03b", 8), ("em04b", 2), ("em04b", 4), ("em04b", 8),
                                         ("c5b-multiscale", 8), ("c5a-multiscale", 2)])
def test_rank_memory_fits_b200(case, world):
    """Per-rank memory of the distributed step (h + h' + gk_dist_step's workspace)
    inside 180 GB for every multi-GPU config, and <= 4 state shards for the two that
    need it (configs[3] em04b at 2 GPUs, configs[4] C5b at 8: 64 / 257 GB states)."""
    from paper_2305_10553_b200.dist import rank_memory_bytes
    from paper_2305_10553_b200.grid import make_case
    for backend in ("p2p", "nccl"):
        m = rank_memory_bytes(make_case(case), world, backend=backend)
        print(case, world, {k: (round(v / 1e9, 2) if isinstance(v, int) and v > 1e6 else v) for k, v in m.items()})
        assert m["fits_180GB"], m
        if (case, world) in (("em04b", 2), ("c5b-multiscale", 8)):
            assert m["states_per_rank"] <= 4.0, m
