"""Per-rank work of the multi-GPU step, measured on one GPU: gk_dist_step_sim runs
the G ranks' phases (home-layout field / collision / finish, velocity-chunked
bracket over blocked layouts, the exchanges as device copies) in lock-step on
this device, so its time / G is one rank's compute plus a local stand-in for the
NVLink transfers.   python tools/sim_scaling.py [case] [reps]"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402
from paper_2305_10553_b200.dist import auto_chunks  # noqa: E402
from paper_2305_10553_b200.grid import make_case, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.spectral import _plan_size, get_plan  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "sh03b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
shape = make_case(case)
lib = _lib.load()
dev = torch.device("cuda", 0)
M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
inp = make_kernel_inputs(shape, 1234)
px, py = inp["plans"]
nx, ny = _plan_size(px), _plan_size(py)
plan = get_plan(R, Y, nx, ny, dev)
h = random_state_device(shape, 1234, dev).reshape(M, T, Y, R)
w = torch.from_numpy(np.asarray(inp["weights"], dtype=float).reshape(-1).copy()).to(dev)
A = torch.from_numpy(np.ascontiguousarray(inp["matrices"], dtype=float)).to(dev)
stencil = _lib.doubles(inp["stencil"])
sh = np.asarray(inp["shifts"], dtype=np.int32)
dt = 1.5e-9
for G in (1, 2, 4, 8):
    if Y % G:
        continue
    K = auto_chunks(shape, G, True, "nccl")
    Yl = Y // G
    homes = [h[:, :, g * Yl:(g + 1) * Yl].contiguous() for g in range(G)]
    outs = [torch.empty_like(x) for x in homes]
    phis = [torch.empty((T, Yl, R), dtype=torch.complex128, device=dev) for _ in range(G)]
    shifts = [torch.from_numpy(np.ascontiguousarray(sh[g * Yl:(g + 1) * Yl])).to(dev) for g in range(G)]
    nbytes = lib.gk_dist_workspace_bytes(nx, ny, M, T, Y, R, G, K)
    wss = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(G)]
    arr = lambda ts: (C.c_void_p * G)(*[t.data_ptr() for t in ts])  # noqa: E731

    def run():
        _lib.check(lib.gk_dist_step_sim(G, plan.handle, arr(homes), w.data_ptr(), stencil, len(inp["stencil"]),
                                        A.data_ptr(), arr(shifts), dt, arr(outs), arr(phis), M, T, Y, R, K, arr(wss),
                                        nbytes, torch.cuda.current_stream().cuda_stream), "gk_dist_step_sim")

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{case} G={G} K={K}: all ranks {ms:.1f} ms -> per rank {ms / G:.2f} ms", flush=True)
    del homes, outs, phis, wss
    torch.cuda.empty_cache()
