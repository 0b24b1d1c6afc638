"""The P2P transport of the multi-GPU step (CUDA IPC windows, copy-engine pushes,
the return transpose fused into the bracket's x forward transform, stream memory
operations for ordering) with real separate processes: 2, 4 and 8 ranks share the
one GPU of this pool -- IPC works between processes on the same device and no
kernel waits on another process (the waits are stream front-end operations), so
this runs the full cross-process protocol.  Two steps (the second reuses the
windows, flags and matrix slices) must equal the single-GPU step bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_10553_b200.grid import GridShape, random_state_device, random_state_shard_device
from paper_2305_10553_b200.kernels import make_kernel_inputs
from paper_2305_10553_b200.step import Stepper

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, outdir, dims, chunks, steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_10553_b200.dist import DistStepper
        shape = GridShape(*dims)
        inp = make_kernel_inputs(shape, 9)
        dev = torch.device("cuda", 0)
        ds = DistStepper(shape, inp, 1e-4, dev, chunks=chunks, backend="p2p")
        h = random_state_shard_device(shape, 9, ds.y0, ds.y1, dev)
        out = torch.empty_like(h)
        for _ in range(steps):
            ds.step(h, out)
            h, out = out, h
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"h{rank}.npy"), h.cpu().numpy())
        np.save(os.path.join(outdir, f"phi{rank}.npy"), ds.phi_l.cpu().numpy())
        dist.barrier()  # nobody unmaps its window while a peer may still use it
        del ds
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("dims, world, chunks", [((480, 48, 8, 8, 8, 1), 2, 4),   # sh03b plan, int8 collision
                                                 ((16, 8, 8, 8, 4, 2), 2, 3),     # C1, DMMA collision
                                                 ((480, 48, 8, 4, 8, 1), 4, 2),
                                                 ((480, 48, 8, 8, 8, 1), 8, 2),   # 8 ranks, as on a full node
                                                 ((1344, 288, 8, 2, 1, 1), 2, 1)])  # em04b plan
def test_p2p_rank_step_equals_single_gpu_step(tmp_path, dims, world, chunks):
    steps = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), dims, chunks, steps), nprocs=world,
                       start_method="spawn")
    shape = GridShape(*dims)
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    st = Stepper(shape, make_kernel_inputs(shape, 9), 1e-4, graph=False)
    x = random_state_device(shape, 9)
    for _ in range(steps):
        phi_in = x
        x = st.step(x)
    got = np.concatenate([np.load(tmp_path / f"h{r}.npy") for r in range(world)], axis=2)
    assert np.array_equal(got, x.reshape(M, T, Y, R).cpu().numpy())
    phi = np.concatenate([np.load(tmp_path / f"phi{r}.npy") for r in range(world)], axis=1)
    assert np.array_equal(phi, st.phi.cpu().numpy())
    del phi_in
