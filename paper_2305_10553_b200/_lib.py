"""ctypes binding of libgk.so, the C-ABI declared in include/gk.h.

There is no fallback: if the library is missing or fails to load, every entry
point raises.  Tensor arguments cross the boundary as raw device pointers; the
stream is torch's current stream on the tensor's device.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

# GK_LIB_PATH: load a variant build (tools/build_variant.sh) for A/B timing
LIB_PATH = Path(os.environ.get("GK_LIB_PATH") or Path(__file__).resolve().parent / "libgk.so")
ABI_VERSION = 1

_p = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double

# name -> (restype, argtypes); mirrors include/gk.h one to one
SIGNATURES = {
    "gk_version": (_int, []),
    "gk_last_error": (C.c_char_p, []),
    "gk_device_info": (_int, [_int, C.POINTER(_int), C.POINTER(_int), C.POINTER(_int), C.POINTER(_i64)]),
    "gk_launch_counter": (_i64, []),
    "gk_probe_fp64_peak": (_int, [C.POINTER(_dbl), C.POINTER(_dbl)]),
    "gk_field": (_int, [_p, _p, _p, _i64, _i64, _i64, _p]),
    "gk_stream": (_int, [_p, C.POINTER(_dbl), _int, _int, _p, _i64, _i64, _i64, _p]),
    "gk_stream_wide": (_int, [_p, _p, _int, _int, _p, _i64, _i64, _i64, _p]),
    "gk_shear": (_int, [_p, _p, _p, _i64, _i64, _i64, _p]),
    "gk_collision": (_int, [_p, _p, _p, _i64, _i64, _i64, _p]),
    "gk_spectral_plan_create": (_int, [_i64, _i64, _i64, _i64, C.POINTER(_p)]),
    "gk_spectral_plan_destroy": (_int, [_p]),
    "gk_bracket_workspace_bytes": (_i64, [_p, _i64, _i64]),
    "gk_bracket": (_int, [_p, _p, _p, _p, _i64, _p, _p, _i64, _i64, _p, _i64, _p]),
    "gk_nonlinear": (_int, [_p, _p, _p, _p, _i64, _i64, _p, _i64, _p]),
    "gk_transform_workspace_bytes": (_i64, [_p, _i64]),
    "gk_to_real": (_int, [_p, _p, _p, _i64, _p, _i64, _p]),
    "gk_to_spectrum": (_int, [_p, _p, _p, _i64, _p, _i64, _p]),
    "gk_axpy3": (_int, [_p, _p, _p, _p, _dbl, _p, _i64, _p]),
    "gk_step_finish": (_int, [_p, _p, _p, C.POINTER(_dbl), _int, _p, _dbl, _p, _i64, _i64, _i64, _i64, _p]),
    "gk_step_workspace_bytes": (_i64, [_p, _i64, _i64, _i64, _i64]),
    "gk_step_workspace_bytes_w": (_i64, [_p, _int, _i64, _i64, _i64, _i64]),
    "gk_step_stage": (_int, [_int, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _i64, _i64, _i64, _i64,
                             _p, _i64, _p]),
    "gk_step": (_int, [_p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _p, _i64, _i64, _i64, _i64,
                       _p, _i64, _p]),
    "gk_step_ex": (_int, [_p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _p, _i64, _i64, _i64, _i64,
                          _p, _i64, _int, _p]),
    "gk_field_range": (_int, [_p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p]),
    "gk_collision_range": (_int, [_p, _p, _p, _i64, _i64, _i64, _i64, _i64, _p]),
    "gk_collision_mode": (_int, [C.c_int]),
    "gk_probe_i8_peak": (_int, [C.POINTER(_dbl)]),
    "gk_collision_fixups": (_int, [C.POINTER(_i64)]),
    "gk_nonlinear_range": (_int, [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _p, _i64, _p]),
    "gk_step_finish_range": (_int, [_p, _p, _p, C.POINTER(_dbl), _int, _p, _dbl, _p, _i64, _i64, _i64, _i64, _i64,
                                    _i64, _p]),
    "gk_step_host": (_int, [_p, _p, _p, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _i64, _i64, _i64, _i64,
                            _int, _p, _i64, _p]),
    "gk_step_host_ex": (_int, [_p, _p, _p, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _i64, _i64, _i64,
                               _i64, _int, _p, _i64, _int, _p]),
    "gk_step_host_join": (_int, [_p]),
    "gk_philox_uniform": (_int, [C.c_uint64, C.c_uint64, _i64, _i64, _dbl, _dbl, _p, _i64, _p]),
    "gk_philox_uniform_rows": (_int, [C.c_uint64, C.c_uint64, _i64, _i64, _i64, _i64, _dbl, _dbl, _p, _i64, _p]),
    "gk_permute_blocks": (_int, [_p, _p, _i64, _i64, _i64, _p]),
    "gk_step_inplace_workspace_bytes": (_i64, [_p, _i64, _i64, _i64, _i64]),
    "gk_step_inplace": (_int, [_int, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _i64, _i64, _i64, _i64,
                               _p, _i64, _p]),
    "gk_nonlinear_acc": (_int, [_p, _p, _p, _p, _i64, _i64, _p, _i64, _p]),
    "gk_nonlinear_acc_workspace_bytes": (_i64, [_p, _i64, _i64]),
    "gk_stream_axpy_inplace": (_int, [_p, _p, C.POINTER(_dbl), _int, _dbl, _i64, _i64, _i64, _p]),
    "gk_comm_unique_id": (_int, [_p]),
    "gk_comm_init": (_int, [_int, _int, _p, C.POINTER(_p)]),
    "gk_comm_destroy": (_int, [_p]),
    "gk_comm_info": (_int, [_p, C.POINTER(_int), C.POINTER(_int), C.POINTER(_int)]),
    "gk_transpose_to_nl": (_int, [_p, _p, _p, _i64, _i64, _p]),
    "gk_transpose_to_lin": (_int, [_p, _p, _p, _i64, _i64, _p]),
    "gk_comm_allgather": (_int, [_p, _p, _p, _i64, _p]),
    "gk_nonlinear_blocked": (_int, [_p, _p, _p, _p, _i64, _i64, _i64, _p, _i64, _p]),
    "gk_dist_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64, _i64, _int, _i64]),
    "gk_dist_step": (_int, [_p, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _p, _i64, _i64, _i64, _i64,
                            _i64, _p, _i64, _int, _p]),
    "gk_dist_step_stage": (_int, [_int, _p, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _i64, _i64, _i64,
                                  _i64, _i64, _p, _i64, _p]),
    "gk_dist_step_sim": (_int, [_int, _p, C.POINTER(_p), _p, C.POINTER(_dbl), _int, _p, C.POINTER(_p), _dbl,
                                C.POINTER(_p), C.POINTER(_p), _i64, _i64, _i64, _i64, _i64, C.POINTER(_p), _i64,
                                _p]),
    "gk_p2p_create": (_int, [_int, _int, _i64, _i64, _i64, _i64, _i64, C.POINTER(_p)]),
    "gk_p2p_window_bytes": (_i64, [_p]),
    "gk_p2p_ipc_handle": (_int, [_p, _p]),
    "gk_p2p_connect": (_int, [_p, _p]),
    "gk_p2p_destroy": (_int, [_p]),
    "gk_p2p_selftest_send": (_int, [_p]),
    "gk_p2p_selftest_check": (_int, [_p, _int]),
    "gk_dist_p2p_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64, _i64, _int, _i64]),
    "gk_dist_step_p2p_stage": (_int, [_int, _p, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _p, _i64, _p]),
    "gk_dist_step_p2p": (_int, [_p, _p, _p, _p, C.POINTER(_dbl), _int, _p, _p, _dbl, _p, _p, _i64, _i64, _i64, _i64,
                                _p, _i64, _int, _p]),
}

_lock = threading.Lock()
_lib = None


class GkError(RuntimeError):
    """A libgk call returned a nonzero status."""


def load() -> C.CDLL:
    """Load (once) and type the library; raises if it is absent or stale."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2305_10553_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.gk_version() != ABI_VERSION:
            raise ImportError(f"libgk ABI {lib.gk_version()} != expected {ABI_VERSION}; rebuild")
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().gk_last_error().decode(errors="replace")
        raise GkError(f"{what} failed (status {rc}): {msg}")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_of(device) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def doubles(values) -> C.Array:
    vals = [float(v) for v in values]
    return (_dbl * max(1, len(vals)))(*vals)
