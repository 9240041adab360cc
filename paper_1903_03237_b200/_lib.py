"""ctypes binding of the C ABI in include/fastmnmf.h (libfastmnmf.so).

This is the only way the package reaches compute: every operator below calls
hand-written sm_100a kernels through the shared library. There is no CPU
fallback -- importing the package on a machine without the built library, or
calling an operator without a CUDA device, raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfastmnmf.so")

FM_F32 = 0
FM_F64 = 1
FM_STATUS_CLEAR = 0xFFFFFFFFFFFFFFFF

_c_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)


class FmDims(ctypes.Structure):
    _fields_ = [
        ("B", _c_i64), ("F", _c_i64), ("T", _c_i64), ("M", _c_i64), ("N", _c_i64),
        ("K", _c_i64), ("f_offset", _c_i64), ("dtype", ctypes.c_int32),
        ("normalize", ctypes.c_int32), ("ip_sweeps", ctypes.c_int32),
        ("dp", ctypes.c_int32),
    ]


class FmState(ctypes.Structure):
    _fields_ = [
        ("X", _vp), ("xt", _vp), ("Q", _vp), ("g", _vp), ("W", _vp), ("H", _vp),
        ("floor", _vp), ("trace", _vp), ("status", _vp), ("work", _vp),
    ]


class FmDp(ctypes.Structure):
    _fields_ = [
        ("D", _c_i64), ("Hd", _c_i64),
        ("W1", _vp), ("b1", _vp), ("W2", _vp), ("b2", _vp), ("W3", _vp), ("b3", _vp),
        ("u", _vp), ("v", _vp), ("z", _vp), ("r", _vp), ("adam_m", _vp), ("adam_v", _vp),
        ("adam_step", _vp), ("work", _vp),
        ("adam_steps", ctypes.c_int32), ("lr", ctypes.c_float), ("beta1", ctypes.c_float),
        ("beta2", ctypes.c_float), ("eps", ctypes.c_float),
        ("decoder_kind", ctypes.c_int32), ("mh_steps", ctypes.c_int32), ("mh_std", ctypes.c_double),
        ("mh_noise", _vp), ("mh_unif", _vp), ("mh_seed", ctypes.c_uint64),
    ]


# (name, restype, argtypes) -- the exported surface of fastmnmf.h
SIGNATURES = [
    ("fm_fullrank_workspace_bytes", ctypes.c_size_t, [ctypes.c_int, _c_i64, _c_i64, _c_i64]),
    ("fm_fullrank_stats", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int,
      ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("fm_update_scm", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _vp]),
    ("fm_wiener_fullrank", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, ctypes.c_double, _vp, _vp, _vp]),
    ("fm_nmf_mu", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, ctypes.c_int, _vp]),
    ("fm_nmf_absorb", ctypes.c_int, [ctypes.c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp]),
    ("fm_reconstruct_scm", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp]),
    ("fm_stft_frames", _c_i64, [_c_i64, _c_i64, _c_i64]),
    ("fm_stft", ctypes.c_int, [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp]),
    ("fm_istft_workspace_bytes", ctypes.c_size_t, [ctypes.c_int, _c_i64, _c_i64, _c_i64]),
    ("fm_istft", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp]),
    ("fm_fast_stats", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, ctypes.c_double,
      ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp, _dp, _vp]),
    ("fm_mix_power", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, ctypes.c_double, _vp, _vp]),
    ("fm_ip_weights", ctypes.c_int, [ctypes.c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp]),
    ("fm_project_power", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp]),
    ("fm_update_diagonalizer", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, ctypes.c_int, _vp, _vp]),
    ("fm_logdet", ctypes.c_int, [ctypes.c_int, _c_i64, _c_i64, _vp, _vp, _vp]),
    ("fm_wiener_fast", ctypes.c_int,
     [ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("fm_nmf_lambda", ctypes.c_int, [ctypes.POINTER(FmDims), _vp, _vp, _vp, _vp]),
    ("fm_data_term", ctypes.c_int, [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), _dp, _vp]),
    ("fm_dp_workspace_bytes", ctypes.c_size_t, [ctypes.POINTER(FmDims), ctypes.POINTER(FmDp)]),
    ("fm_prologue_dp", ctypes.c_int,
     [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), ctypes.POINTER(FmDp), _vp]),
    ("fm_iterate_dp", ctypes.c_int,
     [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), ctypes.POINTER(FmDp), _vp]),
    ("fm_run_dp", ctypes.c_int,
     [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), ctypes.POINTER(FmDp), ctypes.c_int,
      ctypes.c_int, _vp]),
    ("fm_workspace_bytes", ctypes.c_size_t, [ctypes.POINTER(FmDims)]),
    ("fm_prologue", ctypes.c_int, [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), _vp]),
    ("fm_refresh", ctypes.c_int, [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), _vp]),
    ("fm_schedule", ctypes.c_int, [ctypes.POINTER(FmDims)]),
    ("fm_iterate", ctypes.c_int, [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), _vp]),
    ("fm_iterate_phase", ctypes.c_int,
     [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), ctypes.c_int, _vp, _vp]),
    ("fm_iterate_profiled", ctypes.c_int,
     [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), ctypes.POINTER(ctypes.c_float),
      ctypes.POINTER(ctypes.c_int), _vp]),
    ("fm_run", ctypes.c_int,
     [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), ctypes.c_int, ctypes.c_int, _vp]),
    ("fm_iterate_dp_profiled", ctypes.c_int,
     [ctypes.POINTER(FmDims), ctypes.POINTER(FmState), ctypes.POINTER(FmDp),
      ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int), _vp]),
    ("fm_observation_stats", ctypes.c_int, [ctypes.POINTER(FmDims), _vp, _dp, _dp, _vp]),
    ("fm_scale_observation", ctypes.c_int, [ctypes.POINTER(FmDims), _vp, _dp, _vp]),
    ("fm_spatial_init", ctypes.c_int, [ctypes.POINTER(FmDims), _vp, _vp, _vp, _vp]),
    ("fm_last_error", ctypes.c_char_p, []),
    ("fm_version", ctypes.c_int, []),
]

_lib = None


# fm_schedule() values (fastmnmf.h FM_SCHED_*)
SCHEDULES = {0: "split", 1: "fused", 2: "bin"}


def load():
    """Load libfastmnmf.so (built by ``make`` / ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library with `make` (or "
            "__graft_entry__.build()); this package has no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc, what):
    if rc != 0:
        msg = load().fm_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (rc={rc}): {msg}")


def ptr(t):
    """Device address of a torch tensor (None -> NULL). The kernels read raw
    memory, so lazily conjugated/negated views and non-contiguous tensors are
    rejected rather than silently misread."""
    if t is None:
        return None
    if t.is_conj() or t.is_neg() or not t.is_contiguous():
        raise ValueError("tensor passed to libfastmnmf must be contiguous and materialised "
                         "(resolve_conj / resolve_neg)")
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(device=None):
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
