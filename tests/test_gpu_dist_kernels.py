"""GPU pieces of the multi-GPU path that one GPU can exercise: the block
permutation behind the all-to-all transposes, and the single-rank
DistStepper (CudaOps) against the fused single-GPU step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2305_10553_b200 import _lib
from paper_2305_10553_b200.dist import CudaOps, DistStepper
from paper_2305_10553_b200.grid import GridShape, make_case, random_state
from paper_2305_10553_b200.kernels import make_kernel_inputs
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


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_single_rank_dist_stepper_equals_stepper():
    """world_size 1 over NCCL: DistStepper + CudaOps == Stepper (bitwise)."""
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        shape = make_case("sh03b-desk")
        inp = make_kernel_inputs(shape, 3)
        h = torch.from_numpy(random_state(shape, 3)).to(dev)
        ops = CudaOps(shape, inp, 1e-4, dev, slice(0, shape.n_toroidal))
        ds = DistStepper(shape, ops, dev)
        hh = ds.home_slice(h)
        out = torch.empty_like(hh)
        ds.step(hh, out)
        want = Stepper(shape, inp, 1e-4, device=dev).step(h)
        assert torch.equal(out.reshape(want.shape), want)
    finally:
        dist.destroy_process_group()
