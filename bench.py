"""Benchmark: wall-clock seconds per time step of the CGYRO-proxy hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--case sh03b]

Metric (BASELINE.json): "wallclock sec/step (nl, coll, str, comm split) at
1/2/4/8 B200 vs host CPU ref".  One step is the builder-defined composition of
the reference's five kernels:

    phi = field(h, w); rhs = (stream(h) + nonlinear(h, phi)) + collision(h)
    h'  = shear(h + dt * rhs, shifts)

on the sh03b shape (BASELINE configs[2]: (480, 48, 32, 24, 8, 3), 6.8 GB state,
bracket plan 720 x 144).  ``value`` is device time per step with the state
resident in HBM (each step reads h and writes h'; the 6.8 GB state is far larger
than the 126 MB L2, so no flush is needed between steps).  ``e2e`` is the same
step through the public API with the state copied from pinned host memory
and the new state copied back, every step.  N > 1 (torchrun, NCCL): the same
total problem (strong scaling) sharded toroidal-home with all-to-all transposes
(paper_2305_10553_b200/dist.py); time = max over ranks.

``--impl reference`` times the reference's CPU algorithm (the oracle port, the
same numpy calls as the reference; /root/reference is absent on the GPU box) on
the host cores, on a bounded sample of the same workload, extrapolated to one
step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "wallclock sec/step (nl, coll, str, comm split) at 1/2/4/8 B200 vs host CPU ref"
UNIT = "s/step"
DT = 1e-6
# Time step per case: dt = 0.01 / (|rhs| / |h|) with |rhs| / |h| estimated from one
# slice of the reference bracket (|nonlinear| / |h|: sh03b 6.9e6, em04b 4.2e8, C5a
# 1.75e8) or the collision (C2, ~14), so the explicit step moves the state ~1%
# and it stays bounded over the run.  The arithmetic does not depend on dt, but the
# int8 collision's accuracy certificate does look at the data: a state blown up by
# a too-large dt (dt = 1e-6 grows sh03b 7x and em04b 400x per step) develops a
# dynamic range whose tiles get recomputed in fp64.
DT_BY_CASE = {"c1-tiny": 1.3e-5, "c2-linear": 7e-4, "sh03b": 1.5e-9, "sh03b-desk": 2e-6, "em04b": 2.5e-11,
              "em04b-desk": 2.5e-7, "c5a-multiscale": 6e-11, "c5b-multiscale": 3e-12}
NOMINAL_FP64_TFLOPS = 37.0  # NVIDIA B200 datasheet FP64 / FP64 tensor core (MEASURED_PEAKS.json has no fp64)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--case", default="sh03b")
    ap.add_argument("--inplace", action="store_true",
                    help="in-place step (gk_step_inplace; automatic when gk_step's buffers do not fit)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-1core", action="store_true", help="skip the 1-core CPU reference sample")
    ap.add_argument("--dist-stepper", action="store_true",
                    help="N=1: run the multi-GPU rank step (gk_dist_step over a 1-rank NCCL communicator) "
                         "instead of gk_step, to compare the two on one GPU")
    ap.add_argument("--no-fp64-variant", action="store_true",
                    help="skip the strict-fp64 (DMMA collision) step timing beside the headline")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="(tests) spawn --gpus ranks on CPU/gloo, rendezvous, max-reduce a timing, print the line")
    return ap.parse_args()


# Tests only: GK_BENCH_SHARED_GPU=1 runs every rank on cuda:0 with a gloo
# rendezvous (the P2P transport works between processes sharing a device), so the
# multi-rank path of this script runs end to end on a one-GPU box.  Never a
# performance configuration.
SHARED_GPU = os.environ.get("GK_BENCH_SHARED_GPU") == "1"


def _barrier(local):
    import torch.distributed as dist
    if SHARED_GPU:
        dist.barrier()
    else:
        dist.barrier(device_ids=[local])


def _max_over_ranks(x: float, dev) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARED_GPU else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def nccl_init_log(env) -> None:
    """NCCL's INIT log on (it names every rank and the communicator size): an
    inherited NCCL_DEBUG below INFO (e.g. VERSION) is raised to INFO."""
    if env.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        env["NCCL_DEBUG"] = "INFO"
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")


def spawn_ranks(args) -> int:
    """``python bench.py --gpus N`` (N > 1) without torchrun: relaunch this script
    as N ranks under torch.distributed.run on this node (127.0.0.1 rendezvous);
    rank 0 prints the JSON line.  NCCL's INIT log (NCCL_DEBUG=INFO,
    NCCL_DEBUG_SUBSYS=INIT) stays on so the run shows the communicator's rank count."""
    env = dict(os.environ)
    nccl_init_log(env)
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def launcher_selftest(args):
    """The multi-rank plumbing of run_ours without GPUs: gloo rendezvous, barrier,
    max over ranks of a per-rank time, one JSON line from rank 0."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dist.init_process_group("gloo")
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.barrier()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": float(t.item()), "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "launcher_selftest": True,
                          "nccl_debug": os.environ.get("NCCL_DEBUG")}), flush=True)
    dist.destroy_process_group()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- CPU reference (oracle port)

def cpu_sample(shape, rows: int, threads: int, seed: int = 5):
    """Time the reference algorithm on a bounded sample and extrapolate to one step.

    nonlinear, stream, field, shear and the axpy run on `rows` of the M velocity
    rows (all theta; the work is linear in rows); collision on 1 of T theta
    planes with all velocity rows.  `threads` caps both the bracket's thread pool
    (kernels.py:143-149) and the BLAS pool.  Returns (seconds per full step, split).
    """
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import port

    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    rng = np.random.default_rng(seed)
    sub = (rows, 1, 1, T, Y, R)
    h = rng.uniform(-1, 1, sub) + 1j * rng.uniform(-1, 1, sub)
    phi = rng.uniform(-1, 1, (T, Y, R)) + 1j * rng.uniform(-1, 1, (T, Y, R))
    shifts = rng.integers(-3, 4, Y)
    nx, ny = port.plan_sizes(R, Y)
    scale = M / rows
    t = {}
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        s = port.stream(h, port.DEFAULT_STENCIL)
        t["str"] = (time.perf_counter() - t0) * scale
        t0 = time.perf_counter()
        nl = port.nonlinear(h, phi, nx, ny, threads=threads) if Y > 1 else np.zeros_like(h)
        t["nl"] = (time.perf_counter() - t0) * scale
        hp = rng.uniform(-1, 1, (M, 1, 1, 1, Y, R)) + 1j * rng.uniform(-1, 1, (M, 1, 1, 1, Y, R))
        A = rng.uniform(-1, 1, (1, M, M))
        t0 = time.perf_counter()
        c = port.collision(hp, A)
        t["coll"] = (time.perf_counter() - t0) * T
        # field is a full-velocity contraction per (theta, cell): time it on the same theta plane
        t0 = time.perf_counter()
        port.field(hp.reshape(shape.n_species, shape.n_energy, shape.n_xi, 1, Y, R),
                   rng.uniform(-1, 1, (shape.n_species, shape.n_energy, shape.n_xi)))
        t["field"] = (time.perf_counter() - t0) * T
        c = np.resize(c, h.shape)
        t0 = time.perf_counter()
        port.shear(h + DT * ((s + nl) + c), shifts)
        t["axpy_shear"] = (time.perf_counter() - t0) * scale
    return sum(t.values()), t


def cpu_rows_for(shape, cores):
    return max(1, min(shape.velocity_size, max(16, 2 * cores) if shape.n_toroidal > 1 else shape.velocity_size))


def cpu_sample_note(shape, rows):
    M, T = shape.velocity_size, shape.n_theta
    return (f"oracle port (the reference's numpy algorithm) on {rows} of {M} velocity rows x all {T} theta "
            f"(nl, str, axpy+shear: sample fraction {rows / M:.4f}) and 1 of {T} theta planes x all velocity "
            f"rows (coll, field: fraction {1 / T:.4f}), each part extrapolated linearly to one full step")


def cpu_one_core(shape, reps: int = 1):
    """The same sample on one core (BASELINE.md 4.1 asks for 1-core beside all-core)."""
    rows = cpu_rows_for(shape, 1)
    cpu_sample(shape, rows, 1)  # warm
    vals = [cpu_sample(shape, rows, 1)[0] for _ in range(reps)]
    return {"value": statistics.median(vals), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": cpu_sample_note(shape, rows), "sample_fraction_rows": rows / shape.velocity_size}


def run_reference(args, shape):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # under torchrun only rank 0 times the CPU reference
    cores = host_cores()
    rows = cpu_rows_for(shape, cores)
    for _ in range(args.warmup):
        cpu_sample(shape, rows, cores)
    vals, splits = [], []
    for _ in range(args.steps):
        v, sp = cpu_sample(shape, rows, cores)
        vals.append(v)
        splits.append(sp)
    value = statistics.median(vals)
    split = {k: statistics.median(s[k] for s in splits) for k in splits[0]}
    sample = cpu_sample_note(shape, rows)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (numpy RNG, U[-1,1] components)",
        "config": {"workload": workload_name(shape, args.case), "case": args.case, "dims": list(shape.dims)},
        "split_s": split,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "sample_fraction_rows": rows / shape.velocity_size,
                         "sample_fraction_theta": 1 / shape.n_theta},
        "cpu_baseline_1core": None if args.no_cpu_1core else cpu_one_core(shape),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_CONFIG_OF_CASE = {  # BASELINE.json configs index of the named cases
    "c1-tiny": "configs[0]: tiny nonlinear ITG case",
    "c2-linear": "configs[1]: linear-only single toroidal mode (no bracket)",
    "sh03b": "configs[2]: sh03b electrostatic nonlinear step",
    "em04b": "configs[3]: em04b-shaped nonlinear step",
    "c5a-multiscale": "configs[4]: multiscale grid (C5a, one-GPU size)",
    "c5b-multiscale": "configs[4]: multiscale grid (C5b, 8-GPU size)",
}


def workload_name(shape, case):
    what = _CONFIG_OF_CASE.get(case, "nonlinear step")
    return (f"{case} ({what}): (R,Y,T,X,E,Sp)="
            f"({shape.n_radial},{shape.n_toroidal},{shape.n_theta},{shape.n_xi},{shape.n_energy},{shape.n_species}),"
            f" complex128 state {shape.state_bytes / 1e9:.2f} GB")


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------- GPU arm

def fp64_peak(lib):
    import ctypes as C
    a, b = C.c_double(), C.c_double()
    if lib.gk_probe_fp64_peak(C.byref(a), C.byref(b)) != 0:
        return None, None
    return a.value, b.value


def i8_peak(lib):
    import ctypes as C
    v = C.c_double()
    return v.value if lib.gk_probe_i8_peak(C.byref(v)) == 0 else None


def collision_is_i8(lib, shape, world=1):
    """Mirror of the C-side choice (collision_i8.cu collision_use_i8); ranks of the
    multi-GPU step decide from the global column count (dist.cu), like one GPU."""
    mode = lib.gk_collision_mode(-1)
    M, N, T = shape.velocity_size, 2 * shape.n_toroidal * shape.n_radial, shape.n_theta
    if mode == 1 or M > 8192:
        return False
    return mode == 2 or (M >= 64 and M * M * N * T >= 2**30)


def grouped_field_in_collision(lib, shape, inplace):
    """Mirror of step.cu: the int8 collision slices B theta group by theta group (and
    computes the field moment there) when the step's B-slice buffer would exceed
    GK_STEP_SLICES_MAX_GB, and always in the in-place step."""
    if not collision_is_i8(lib, shape):
        return False
    if inplace:
        return True
    M, N, T = shape.velocity_size, 2 * shape.n_toroidal * shape.n_radial, shape.n_theta
    slices = T * (-(-N // 128)) * (-(-M // 32)) * 7 * 4096 + T * (-(-N // 128)) * 128 * 16
    return slices > float(os.environ.get("GK_STEP_SLICES_MAX_GB", "8")) * 1e9


def collision_fixups(lib) -> int:
    import ctypes as C
    v = C.c_int64()
    return v.value if lib.gk_collision_fixups(C.byref(v)) == 0 else -1


def measured_hbm():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def case_dt(case: str) -> float:
    return DT_BY_CASE.get(case, DT)


def run_ours(args, shape):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2305_10553_b200 import _lib
    from paper_2305_10553_b200.dist import DistStepper, rank_memory_bytes, shard_bounds
    from paper_2305_10553_b200.kernels import make_kernel_inputs
    from paper_2305_10553_b200.spectral import bracket_plans

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:  # the INIT log shows every rank joining the N-rank communicator
        nccl_init_log(os.environ)
        if torch.cuda.device_count() < world and not SHARED_GPU:
            raise SystemExit(f"--gpus {world} but only {torch.cuda.device_count()} CUDA devices are visible")
    if SHARED_GPU:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.dist_stepper
    if world > 1:
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    elif use_dist:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=dev)
    lib = _lib.load()
    inputs = make_kernel_inputs(shape, 1234)
    nonlinear = shape.n_toroidal > 1
    y0, y1 = shard_bounds(shape.n_toroidal, world, rank) if world > 1 else (0, shape.n_toroidal)
    plan_sizes = [p.n_padded for p in bracket_plans(shape.n_radial, shape.n_toroidal)] if nonlinear else None
    memory = None
    if use_dist:
        stepper = DistStepper(shape, inputs, case_dt(args.case), dev, nonlinear=nonlinear)
        memory = rank_memory_bytes(shape, world, nonlinear=nonlinear, backend=stepper.backend)
    else:
        from paper_2305_10553_b200.step import Stepper
        # gk_step needs h, h' and ~2 more state buffers; a state too large for that
        # (em04b: 64 GB) steps in place (gk_step_inplace: h + one rhs buffer)
        handle_need = 2 * shape.state_bytes + lib.gk_step_workspace_bytes_w(
            None, len(inputs["stencil"]), shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial)
        inplace = args.inplace or (handle_need + 3 * shape.state_bytes // shape.n_theta
                                   > torch.cuda.mem_get_info(dev)[1] * 0.9)
        stepper = Stepper(shape, inputs, case_dt(args.case), nonlinear=nonlinear, device=dev, inplace=inplace)
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    # the reference's own generator (Philox4x64-10, seed 1234), bit-exact, on the
    # device -- each rank generates only its home shard
    from paper_2305_10553_b200.grid import random_state_device, random_state_shard_device
    if world > 1:
        h = random_state_shard_device(shape, 1234, y0, y1, dev)
    else:
        h = random_state_device(shape, 1234, dev).reshape(M, T, Y, R)
    inplace = getattr(stepper, "inplace", False)
    out = None if inplace else torch.empty_like(h)
    stream = torch.cuda.current_stream(dev)

    def step():
        if inplace:
            stepper.step_inplace(h)
        else:
            stepper.step(h, out)

    def barrier():
        if world > 1:
            _barrier(local)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    f0 = collision_fixups(lib)
    n0 = lib.gk_launch_counter()
    r0 = getattr(stepper, "replayed_kernels", 0)  # CUDA-graph replays (small states) bypass the counter
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    launches = lib.gk_launch_counter() - n0 + getattr(stepper, "replayed_kernels", 0) - r0
    fixups = collision_fixups(lib) - f0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        ms = _max_over_ranks(ms, dev)

    # ---- per-component split (separate untimed-for-headline pass, CUDA events per stage)
    split = component_split(lib, shape, inputs, None, stepper, h, out, dev, world, nonlinear, step_s=ms / 1e3)

    # ---- roofline per component and the dominant one
    hbm, hbm_src = measured_hbm()
    dfma, dmma = fp64_peak(lib)
    i8 = i8_peak(lib) if collision_is_i8(lib, shape, world) else None
    roof = rooflines(shape, split, hbm, hbm_src, dmma, dfma, world, args.case, i8, inplace)
    dom = max(roof, key=lambda r: r["time_s"])

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = (end_to_end_inplace(stepper, h, dev, args.e2e_steps) if inplace else
               end_to_end(stepper, h, out, dev, args.e2e_steps, world, local))

    strict = None
    if (not use_dist and not inplace and not args.no_fp64_variant and collision_is_i8(lib, shape)
            and torch.cuda.mem_get_info(dev)[0] > 5 * shape.state_bytes):
        strict = strict_fp64_variant(lib, shape, inputs, h, out, dev, max(3, args.steps // 2), nonlinear,
                                     case_dt(args.case))

    comm_model = None
    if world > 1:  # the reference's analytic model (commsim.py) on a B200 NVSwitch node, beside the measured split
        from paper_2305_10553_b200.commtopo import step_comm_seconds
        m = step_comm_seconds(shape, world)
        comm_model = {"step_s": m["step_s"], "alltoall_s": m["alltoall_s"],
                      "alltoall_bytes_per_rank": m["alltoall_bytes"],
                      "note": "commsim model on topologies/b200_nvswitch.txt (900 GB/s per GPU): "
                              "2 transposes + phi all-gather per step"}
    result = None
    if rank == 0:
        result = {
            "metric": METRIC, "value": ms / 1e3, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": f"synthetic: reference generator random_state({args.case}, 1234) (Philox4x64-10) run on the device",
            "config": {"workload": workload_name(shape, args.case), "case": args.case, "dims": list(shape.dims),
                       "bracket_plan": plan_sizes, "dt": case_dt(args.case),
                       "parallelism": f"toroidal-home x{world}" + (
                           (f" + P2P transposes of {stepper.chunks} velocity chunks: CUDA IPC windows, copy-engine "
                            "pushes, return transpose fused into the bracket (gk_dist_step_p2p)"
                            if getattr(stepper, "backend", "") == "p2p" else
                            f" + NCCL all-to-all transposes of {stepper.chunks} velocity chunks (gk_dist_step)")
                           if use_dist else ""),
                       "step": (f"{'gk_dist_step_p2p' if getattr(stepper, 'backend', '') == 'p2p' else 'gk_dist_step'}"
                                " (one C-ABI call per rank step)" if use_dist else
                                "in-place (gk_step_inplace: h + one rhs buffer; gk_step's buffers do not fit)"
                                if inplace else "gk_step"),
                       "l2": (f"state {shape.state_bytes / 1e9:.1f} GB >> 126 MB L2 per step: no flush needed"
                              if shape.state_bytes > 1 << 30 else "state smaller than L2")},
            "split_s": {k: v for k, v in split.items()},
            "split_note": ("stage times of one step with CUDA events on the launch stream; str = fused stream + "
                           "axpy + shear pass" + ("; nl includes the chunked all-to-all transposes pipelined with "
                                                  "the bracket, comm = the transposes alone (hidden inside nl)"
                                                  if world > 1 else "; comm = 0 on one GPU")
                           + ("; field and coll are timed as separate passes here, but in the step the field "
                              "moment is computed inside the collision's grouped B slicing (one read of h)"
                              if world == 1 and grouped_field_in_collision(lib, shape, inplace) else "")),
            "roofline": {k: dom[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")} |
                        {"kernel": dom["kernel"], "peak_source": dom["peak_source"],
                         "traffic_source": dom["traffic_source"]} |
                        ({"frac_of_nominal_fp64": dom["frac_of_nominal_fp64"], "nominal_fp64_tflops":
                          NOMINAL_FP64_TFLOPS} if "frac_of_nominal_fp64" in dom else {}),
            "roofline_all": roof,
            "comm_model": comm_model,
            "rank_memory": memory,
            "gpu_launches": launches,
            "collision_certificate": {
                "uncertified_tiles_recomputed_fp64": fixups,
                "note": "int8-slice collision tiles whose error bound exceeded 2^-37 sum_k |A_ik||B_kj| for some "
                        "element, recomputed in fp64, over the timed steps (collision_i8.cu)"},
            "clocks": clocks.summary(),
            "e2e": e2e,
            "strict_fp64": strict,
        }
    if use_dist:
        _barrier(local) if world > 1 else dist.barrier(device_ids=[local])
        del stepper  # its gk_comm before the process group
        dist.destroy_process_group()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        rows = cpu_rows_for(shape, cores)
        cpu_sample(shape, rows, cores)  # warm
        vals = [cpu_sample(shape, rows, cores)[0] for _ in range(2)]
        result["cpu_baseline"] = {
            "value": statistics.median(vals), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": cpu_sample_note(shape, rows), "sample_fraction_rows": rows / M,
            "sample_fraction_theta": 1 / T}
        if not args.no_cpu_1core:
            result["cpu_baseline_1core"] = cpu_one_core(shape)
    if rank == 0:
        print(json.dumps(result), flush=True)


def strict_fp64_variant(lib, shape, inputs, h, out, dev, steps, nonlinear, dt):
    """The same step with the collision as a plain fp64 DMMA GEMM (gk_collision_mode(1),
    the reference's arithmetic: kernels.py:119-123 is an fp64 matmul), timed and split
    like the headline, plus the headline int8-slice collision's error against it on
    this very state (max-abs relative as the reference's tests measure it, and rel L2)."""
    import torch

    from paper_2305_10553_b200 import _lib
    from paper_2305_10553_b200.step import Stepper

    stream = torch.cuda.current_stream(dev)
    prev = lib.gk_collision_mode(1)
    try:
        st = Stepper(shape, inputs, dt, nonlinear=nonlinear, device=dev)
        for _ in range(2):
            st.step(h, out)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            st.step(h, out)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / steps
        split = component_split(lib, shape, inputs, None, st, h, out, dev, 1, nonlinear)
        del st
        torch.cuda.empty_cache()
        # int8 slices vs DMMA on the benchmark state: the full collision of every theta
        A = torch.from_numpy(inputs["matrices"]).to(dev)
        M, T = shape.velocity_size, shape.n_theta
        cells = shape.n_toroidal * shape.n_radial
        c_dmma = torch.empty_like(h)
        _lib.check(lib.gk_collision(A.data_ptr(), h.data_ptr(), c_dmma.data_ptr(), M, T, cells,
                                    _lib.stream_of(dev)), "gk_collision (dmma)")
        lib.gk_collision_mode(2)
        c_i8 = torch.empty_like(h)
        _lib.check(lib.gk_collision(A.data_ptr(), h.data_ptr(), c_i8.data_ptr(), M, T, cells,
                                    _lib.stream_of(dev)), "gk_collision (int8)")
        a, b = torch.view_as_real(c_i8), torch.view_as_real(c_dmma)
        a.sub_(b)
        err = {"max_abs_rel": float(a.abs().max() / b.abs().max()),
               "rel_l2": float(torch.linalg.vector_norm(a) / torch.linalg.vector_norm(b))}
        del a, b, c_i8, c_dmma
    finally:
        lib.gk_collision_mode(prev)
    torch.cuda.synchronize(dev)
    return {"value": ms / 1e3, "unit": UNIT, "ms_per_step": ms, "split_s": split,
            "collision": "fp64 DMMA GEMM (mma.sync m8n8k4 f64, csrc/collision.cu; gk_collision_mode(1))",
            "headline_collision": "int8 slice products on tcgen05 (Ozaki, 6 slices ~ 46 mantissa bits; "
                                  "csrc/collision_i8.cu)",
            "int8_vs_dmma_collision_error": err}


def component_split(lib, shape, inputs, ops, stepper, h, out, dev, world, nonlinear, reps=3, step_s=None):
    """Seconds per step of each stage, timed with events on the launch stream.
    Multi-GPU over NCCL: gk_dist_step_stage (NCCL serial on the compute stream): nl
    includes the phi gather and the transposes, comm is the transposes alone.
    Multi-GPU over P2P: field, coll, str timed alone; the transfers are fused into
    the nonlinear stage, so nl = step - (field + coll + str) and comm is not split."""
    import torch

    from paper_2305_10553_b200.dist import DistStepper

    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    acc = {}

    def timed(name, fn):
        a, b = ev(), ev()
        a.record(stream)
        fn()
        b.record(stream)
        return name, a, b

    p2p = isinstance(stepper, DistStepper) and stepper.backend == "p2p"
    if p2p:
        idx = {"field": 0, "coll": 2, "str": 3}
        stages_fn = [(n, (lambda i=i: stepper.stage(i, h, out))) for n, i in idx.items()]
    elif isinstance(stepper, DistStepper):
        names = ["field"] + (["nl", "comm"] if nonlinear else []) + ["coll", "str"]
        idx = {"field": 0, "nl": 1, "coll": 2, "str": 3, "comm": 4}
        stages_fn = [(n, (lambda i=idx[n]: stepper.stage(i, h, out))) for n in names]
    else:
        stages_fn = [("field", lambda: stepper.stage(0, h, out))]
        if nonlinear:
            stages_fn.append(("nl", lambda: stepper.stage(1, h, out)))
        stages_fn += [("coll", lambda: stepper.stage(2, h, out)), ("str", lambda: stepper.stage(3, h, out))]
    for _ in range(reps):
        recs = [timed(n, f) for n, f in stages_fn]
        torch.cuda.synchronize(dev)
        for n, a, b in recs:
            acc.setdefault(n, []).append(a.elapsed_time(b) / 1e3)
    split = {k: statistics.median(v) for k, v in acc.items()}
    if p2p:
        split["nl"] = max(0.0, (step_s or 0.0) - sum(split.values()))
        split["comm"] = None  # fused into nl (copy-engine pushes + P2P stores from the x forward transform)
    if world == 1 and not p2p:
        split["comm"] = 0.0
    return split


def measured_traffic(case):
    """DRAM bytes per call from the committed ncu captures (profiles/*_traffic.json), or {}."""
    out = {}
    for path in sorted((ROOT / "profiles").glob("*_traffic.json")):
        try:
            doc = json.loads(path.read_text())
        except (OSError, ValueError):
            continue
        if doc.get("case") != case:
            continue
        for k, v in doc.items():
            if isinstance(v, dict):
                t = v.get("traffic_bytes_per_launch") or v.get("traffic_bytes_per_call")
                if t:
                    out[k] = {"bytes": t, "source": f"profiles/{path.name}"}
    return out


def rooflines(shape, split, hbm, hbm_src, dmma, dfma, world, case="sh03b", i8=None, inplace=False):
    """Algorithmic work per stage (SURVEY.md §8 d) / measured stage time."""
    traffic = measured_traffic(case) if world == 1 and not inplace else {}
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    S = shape.state_bytes / world
    Nc = Y * R / world
    out = []
    fp64_peak = dmma or 37.0
    src = "measured fp64 DMMA probe (gk_probe_fp64_peak, this run)" if dmma else "nominal fp64 (no probe)"

    def add(kernel, bound, work, unit, peak, psrc):
        t = split.get(kernel)
        if not t:
            return
        ach = work / t / (1e12 if unit in ("TFLOP/s", "TOPS") else 1e9)
        tr = traffic.get(kernel)
        out.append({"kernel": kernel, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                    "frac": ach / peak, "traffic": tr["bytes"] if tr else None,
                    "traffic_source": tr["source"] if tr else None, "time_s": t, "peak_source": psrc})

    if i8:
        # int8 slice products on tcgen05: 21 exact int8 GEMMs (slice pairs s + t <= 5)
        # of the fp64 one; achieved = int8 ops executed / stage time (slicing included)
        # 21 digit-slice products + the certificate's magnitude product (collision_i8.cu)
        add("coll", "tensor", 22 * 4.0 * M * M * Nc * T, "TOPS", i8,
            "measured int8 tcgen05 probe (gk_probe_i8_peak, this run)")
        if out and out[-1]["kernel"] == "coll":
            out[-1]["fp64_equiv_tflops"] = 4.0 * M * M * Nc * T / split["coll"] / 1e12
            out[-1]["frac_of_nominal_fp64"] = out[-1]["fp64_equiv_tflops"] / NOMINAL_FP64_TFLOPS
            out[-1]["note"] = ("fp64 GEMM as int8 slice products (Ozaki scheme, 6 slices) + a per-tile accuracy "
                               "certificate (one more int8 product), collision_i8.cu")
    else:
        add("coll", "tensor", 4.0 * M * M * Nc * T, "TFLOP/s", fp64_peak, src)
    if Y > 1:
        from paper_2305_10553_b200.spectral import bracket_plans
        nx, ny = (p.n_padded for p in bracket_plans(R, Y))
        n = nx * ny
        flops = (M / world) * T * 3 * 2.5 * n * math.log2(n) + T * 2 * 2.5 * n * math.log2(n)
        add("nl", "tensor", flops, "TFLOP/s", dfma or fp64_peak,
            "measured fp64 DFMA probe (gk_probe_fp64_peak, this run)" if dfma else src)
        if out and out[-1]["kernel"] == "nl":
            out[-1]["frac_of_nominal_fp64"] = out[-1]["achieved"] / NOMINAL_FP64_TFLOPS
    if inplace:
        # in-place finish: rhs = h + dt * (stream(h) + rhs) (reads h, rhs; writes rhs), then h = shear(rhs)
        add("str", "hbm", 5 * S, "GB/s", hbm, hbm_src)
        add("field", "hbm", S * (1 + 1 / M), "GB/s", hbm, hbm_src)
        for r in out:
            if r["kernel"] == "coll":
                r["note"] = r.get("note", "") + "; in-place step: the stage includes the B slicing"
        return out
    # "str" = the fused finish pass: stream(h) + axpy + shear; reads h, (nl,) coll, writes h'
    add("str", "hbm", (4 if Y > 1 else 3) * S, "GB/s", hbm, hbm_src)
    nks, ncb = -(-M // 32), -(-(2 * Y * R // world) // 128)
    slices = T * ncb * nks * 7 * 4096 + T * ncb * 128 * 16  # 6 digit slices + the magnitude slice; column stats
    cap = float(os.environ.get("GK_STEP_SLICES_MAX_GB", "8")) * 1e9  # step.cu step_i8, dist.cu Geom
    if i8 and slices <= cap:
        # the step's field stage is one pass (slice_b with phi): reads S, writes phi (S/M)
        # and the collision's int8 B slices (6 bytes per padded (v, theta, column))
        add("field", "hbm", S + slices + S / M, "GB/s", hbm, hbm_src)
        if out and out[-1]["kernel"] == "field":
            out[-1]["note"] = "field moment + the collision's int8 B slices in one pass (slice_b)"
        for r in out:
            if r["kernel"] == "coll":
                r["note"] += "; B slicing is done in the field stage (stage time excludes it)"
    else:
        add("field", "hbm", S * (1 + 1 / M), "GB/s", hbm, hbm_src)
    return out


def end_to_end_inplace(stepper, h, dev, steps):
    """The in-place step (em04b's 64 GB state on one GPU) with the state in pinned
    host memory: copy in, step in place, copy back into the same host buffer, every
    step (no device room for a second buffer pair, so the copies do not overlap the
    compute)."""
    import torch

    h_host = torch.empty(h.shape, dtype=h.dtype, pin_memory=True)
    h_host.copy_(h)
    stream = torch.cuda.current_stream(dev)

    def one():
        h.copy_(h_host, non_blocking=True)
        stepper.step_inplace(h)
        h_host.copy_(h, non_blocking=True)

    one()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    nbytes = h.numel() * 16
    return {"value": e0.elapsed_time(e1) / 1e3 / steps, "unit": UNIT, "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes,
            "api": "copy in, Stepper.step_inplace (gk_step_inplace), copy back into the same pinned host buffer "
                   "(no device room for overlapping buffers)", "steps_timed": steps}


def end_to_end(stepper, h, out, dev, steps, world, local):
    """Public API with host buffers: pinned H2D of h, step, D2H of h' -- every step.

    One GPU: Stepper.step_host (gk_step_host), the state streamed in and out in
    theta chunks so PCIe overlaps the compute.  N GPUs: copy in, step, copy out."""
    import torch
    import torch.distributed as dist

    h_host = torch.empty(h.shape, dtype=h.dtype, pin_memory=True)
    h_host.copy_(h)
    o_host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    stream = torch.cuda.current_stream(dev)
    pipelined = world == 1 and hasattr(stepper, "step_host")
    # consecutive steps overlap too (copy-in of step n+1 under the compute and
    # copy-out tail of step n) on two alternating device buffer pairs, when they fit
    pairs = [(h, out)]
    if torch.cuda.mem_get_info(dev)[0] > 2 * h.numel() * 16 + (4 << 30):
        pairs.append((torch.empty_like(h), torch.empty_like(out)))
    overlap = len(pairs) == 2
    calls = [0]
    # ranks (DistStepper): the same cross-step overlap with torch streams -- step
    # n+1's copy-in (side stream) under step n's compute, step n's copy-out on a
    # second side stream; a buffer is refilled only after its last reader is done
    cin, cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    in_done = [torch.cuda.Event() for _ in pairs]
    step_done = [torch.cuda.Event() for _ in pairs]
    out_done = [torch.cuda.Event() for _ in pairs]
    for e in step_done + out_done:
        e.record(stream)

    def one():
        i = calls[0] % len(pairs)
        hd, od = pairs[i]
        calls[0] += 1
        if pipelined:
            stepper.step_host(h_host, o_host, hd, od, chunks=int(os.environ.get("GK_E2E_CHUNKS", "16")),
                              overlap=overlap)
            return
        cin.wait_event(step_done[i])  # hd was last read by the step two calls ago
        with torch.cuda.stream(cin):
            hd.copy_(h_host, non_blocking=True)
        in_done[i].record(cin)
        stream.wait_event(in_done[i])
        stream.wait_event(out_done[i])  # od's previous result has been copied out
        stepper.step(hd, od)
        step_done[i].record(stream)
        cout.wait_event(step_done[i])
        with torch.cuda.stream(cout):
            o_host.copy_(od, non_blocking=True)
        out_done[i].record(cout)

    def join():
        if pipelined:
            if overlap:
                stepper.step_host_join()
        else:
            for e in out_done:
                stream.wait_event(e)

    one()
    join()
    torch.cuda.synchronize(dev)
    if world > 1:
        _barrier(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one()
    join()  # the timed region ends with the last step's copy-out
    e1.record(stream)
    torch.cuda.synchronize(dev)
    s = e0.elapsed_time(e1) / 1e3 / steps
    if world > 1:
        s = _max_over_ranks(s, dev)
    nbytes = h.numel() * 16
    return {"value": s, "unit": UNIT, "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world,
            "api": ("Stepper.step_host (gk_step_host_ex C-ABI): pinned host state in / out each step, PCIe "
                    "copies pipelined with the compute over theta chunks (16 by default) x 4 velocity blocks"
                    + ("; consecutive steps overlap (step n+1's copy-in under step n's compute and copy-out, "
                       "two device buffer pairs, GK_STEP_HOST_OVERLAP); the timed region ends after the last "
                       "step's copy-out" if overlap else "")) if pipelined else
                   ("copy in, Stepper.step / DistStepper.step, copy out (pinned host buffers)"
                    + ("; consecutive steps overlap (step n+1's copy-in on a side stream under step n's "
                       "compute, copy-out on a second side stream, two device buffer pairs); the timed region "
                       "ends after the last step's copy-out" if overlap else "")),
            "steps_timed": steps}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    if args.launcher_selftest:
        launcher_selftest(args)
        return
    from paper_2305_10553_b200.grid import make_case
    shape = make_case(args.case)
    if args.impl == "reference":
        run_reference(args, shape)
    else:
        run_ours(args, shape)


if __name__ == "__main__":
    main()
