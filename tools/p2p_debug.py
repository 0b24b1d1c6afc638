"""Two ranks of the P2P step on one GPU, with progress prints and a watchdog
(diagnostic).  python tools/p2p_debug.py [world] [chunks]"""
import faulthandler
import os
import socket
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def worker(rank, world, port, chunks, dims, steps):
    faulthandler.dump_traceback_later(90, exit=True)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_10553_b200.dist import DistStepper
    from paper_2305_10553_b200.grid import GridShape, random_state_shard_device
    from paper_2305_10553_b200.kernels import make_kernel_inputs
    shape = GridShape(*dims)
    inp = make_kernel_inputs(shape, 9)
    dev = torch.device("cuda", 0)
    print(rank, "init", flush=True)
    ds = DistStepper(shape, inp, 1e-4, dev, chunks=chunks, backend="p2p")
    print(rank, "connected window", ds.comm.window_bytes, flush=True)
    h = random_state_shard_device(shape, 9, ds.y0, ds.y1, dev)
    out = torch.empty_like(h)
    t0 = time.time()
    for i in range(steps):
        ds.step(h, out)
        h, out = out, h
        print(rank, "issued step", i, ds.chunks, time.time() - t0, flush=True)
        torch.cuda.synchronize()
        print(rank, "done step", i, time.time() - t0, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    dims = tuple(int(x) for x in sys.argv[4:10]) if len(sys.argv) > 9 else (16, 8, 8, 8, 4, 2)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(worker, args=(world, port, chunks, dims, steps), nprocs=world, start_method="spawn")
