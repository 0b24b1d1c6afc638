"""Per-kernel device timing at a named case (CUDA events, inputs resident).

    python tools/quick_timing.py sh03b [reps]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402
from paper_2305_10553_b200.grid import make_case  # noqa: E402
from paper_2305_10553_b200.kernels import DEFAULT_STENCIL, make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.spectral import get_plan  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "sh03b"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    shape = make_case(case)
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    g = torch.Generator(device=dev).manual_seed(0)
    h = torch.complex(torch.rand(shape.dims, dtype=torch.float64, device=dev, generator=g) * 2 - 1,
                      torch.rand(shape.dims, dtype=torch.float64, device=dev, generator=g) * 2 - 1)
    inp = make_kernel_inputs(shape, 7)
    w = torch.from_numpy(inp["weights"]).to(dev)
    A = torch.from_numpy(inp["matrices"]).to(dev)
    sh = torch.from_numpy(inp["shifts"].astype(np.int32)).to(dev)
    phi = torch.from_numpy(inp["phi"]).to(dev)
    out = torch.empty_like(h)
    M, T, Nc = shape.velocity_size, shape.n_theta, shape.n_toroidal * shape.n_radial
    nx, ny = (p.n_padded for p in inp["plans"])
    plan = get_plan(shape.n_radial, shape.n_toroidal, nx, ny, dev)
    wsb = lib.gk_bracket_workspace_bytes(plan.handle, M * T, T)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    fo = torch.empty(shape.field_dims, dtype=torch.complex128, device=dev)
    st = _lib.stream_of(dev)
    sc = _lib.doubles(DEFAULT_STENCIL)
    calls = {
        "field": lambda: lib.gk_field(h.data_ptr(), w.data_ptr(), fo.data_ptr(), M, T, Nc, st),
        "stream": lambda: lib.gk_stream(h.data_ptr(), sc, 5, 1, out.data_ptr(), M, T, Nc, st),
        "shear": lambda: lib.gk_shear(h.data_ptr(), sh.data_ptr(), out.data_ptr(), M * T, shape.n_toroidal,
                                      shape.n_radial, st),
        "collision": lambda: lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, st),
        "nonlinear": lambda: lib.gk_nonlinear(plan.handle, h.data_ptr(), phi.data_ptr(), out.data_ptr(), M, T,
                                              ws.data_ptr(), wsb, st),
    }
    S = shape.state_bytes
    res = {"case": case}
    for name, fn in calls.items():
        _lib.check(fn(), name)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        entry = {"ms": round(ms, 4)}
        if name in ("stream", "shear"):
            entry["GB/s"] = round(2 * S / ms / 1e6, 1)
        if name == "field":
            entry["GB/s"] = round(S * (1 + 1 / M) / ms / 1e6, 1)
        if name == "collision":
            entry["TFLOP/s"] = round(4.0 * M * M * Nc * T / ms / 1e9, 2)
        if name == "nonlinear":
            n = nx * ny
            fl = M * T * 3 * 2.5 * n * np.log2(n) + T * 2 * 2.5 * n * np.log2(n)
            entry["TFLOP/s(alg)"] = round(fl / ms / 1e9, 2)
            entry["GB/s"] = round(2 * S / ms / 1e6, 1)
        res[name] = entry
    print(json.dumps(res))


if __name__ == "__main__":
    main()
