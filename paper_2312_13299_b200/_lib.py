"""ctypes binding of libplas_b200.so (include/plas_b200.h).

The extension is REQUIRED: there is no CPU or eager-PyTorch fallback.  Every
GPU entry point of the package goes through `lib()`, which raises if the
shared library has not been built or no CUDA device is visible.  PyTorch is
used only for device memory (workspaces, staging tensors) and the current
CUDA stream.
"""

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PLAS_LIB_PATH") or os.path.join(HERE, "libplas_b200.so")  # PLAS_LIB_PATH: A/B builds

PLAS_OK = 0
PLAS_ERR_INVALID = -1
PLAS_ERR_CUDA = -2
PLAS_ERR_NONFINITE = -3
PLAS_ERR_CAPACITY = -4
PLAS_ERR_WORKSPACE = -5

PLAS_F32, PLAS_F64 = 0, 1
PLAS_RNG_PARITY, PLAS_RNG_DEVICE = 0, 1
PLAS_BLUR_SEPARABLE, PLAS_BLUR_RENORMALIZED, PLAS_BLUR_BORDER_WEIGHT = 0, 1, 2

P = ctypes.c_void_p
i32, i64, u64, f64, sz = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t

# int (*exchange)(void* ctx, int op, int64_t a, int64_t b, const int64_t* sizes) of
# plas_sort_args (multi-GPU sharding)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                               ctypes.POINTER(ctypes.c_int64))
PLAS_XCHG_PASS, PLAS_XCHG_ALLGATHER, PLAS_XCHG_ALLTOALL = 0, 1, 2
XPART = 4  # doubles per rank in the pass exchange (int128 change as 2 words, moved count, pad)


class SortArgs(ctypes.Structure):
    _fields_ = [
        ("features", P), ("features_dtype", i32), ("dim", i32), ("n", i64),
        ("improvement_threshold", f64), ("radius_decay", f64), ("initial_radius", f64),
        ("min_block_size", i32), ("seed", u64), ("rng_mode", i32), ("num_levels", i32),
        ("radii", P), ("weights", P), ("weight_offsets", P), ("initial_perm", P),
        ("trace_capacity", i64), ("stream", P), ("profile", P),
        ("rank", i32), ("world", i32), ("exchange", EXCHANGE_FN), ("exchange_ctx", P),
        ("xchg_send", P), ("xchg_recv", P), ("xchg_part", P), ("xchg_part_all", P),
    ]


class SortProfile(ctypes.Structure):
    _fields_ = [(f"{k}_{name}", t) for name in ("pass", "blur0", "blur1", "border", "distance",
                                                 "control", "select")
                for k, t in (("ms", f64), ("n", i64))]


class SortResult(ctypes.Structure):
    _fields_ = [
        ("perm", P), ("initial_vad", f64), ("final_vad", f64), ("reorders", i64),
        ("levels_done", i32), ("level_counts", P), ("trace", P), ("trace_len", i64),
        ("gpu_ms", f64), ("cells_moved", i64), ("exact_warps", i64), ("banded_levels", i64),
    ]


# exported symbols and their ctypes signatures (restype, argtypes); the
# CPU test checks this list against include/plas_b200.h
class Attr(ctypes.Structure):
    """include/plas_b200.h: plas_attr (one attribute of normalize_for_sorting)."""
    _fields_ = [("values", ctypes.c_void_p), ("row_stride", ctypes.c_int64), ("channels", ctypes.c_int32),
                ("activation", ctypes.c_int32), ("weight", ctypes.c_double)]


SIGNATURES = {
    "plas_abi_version": (i32, []),
    "plas_sizeof_sort_args": (sz, []),
    "plas_sizeof_sort_result": (sz, []),
    "plas_last_error": (ctypes.c_char_p, []),
    "plas_num_levels": (i32, [i64, f64, f64]),
    "plas_sort_workspace_bytes": (sz, [i64, i32, i32, i64, i64, i32]),
    "plas_sort_workspace_bytes_sharded": (sz, [i64, i32, i32, i64, i64, i32, i32]),
    "plas_sort": (i32, [ctypes.POINTER(SortArgs), ctypes.POINTER(SortResult), P, sz]),
    "plas_assign_groups": (i32, [P, P, P, i32, i32, P, i64, i32, P]),
    "plas_assign_groups_f64t": (i32, [P, P, P, i32, i32, P, i64, i32, P]),
    "plas_aux_workspace_bytes": (sz, [i32, i32, i32]),
    "plas_blur": (i32, [P, P, i32, i32, i32, i32, P, i32, i32, P, sz, P]),
    "plas_blur_tiers_workspace_bytes": (sz, [i32, i32, i32, i32]),
    "plas_blur_target_tiers": (i32, [P, P, i32, i32, i32, P, i32, i32, P, P, sz, P]),
    "plas_grid_distance_workspace_bytes": (sz, [i64]),
    "plas_grid_distance": (i32, [P, P, P, i64, i32, P, P, sz, P]),
    "plas_vad_workspace_bytes": (sz, [i32, i32, i32]),
    "plas_vad": (i32, [P, i32, i32, i32, i32, P, P, sz, P]),
    "plas_smoothness_plane": (i32, [P, P, i32, i32, i32, f64, f64, i32, P, i32, P, P, sz, P]),
    "plas_prune_workspace_bytes": (sz, [i64]),
    "plas_prune_to_grid": (i32, [P, i64, i64, P, P, sz, P]),
    "plas_normalize_workspace_bytes": (sz, [i64, i32]),
    "plas_normalize_for_sorting": (i32, [P, i32, i64, P, i32, P, P, P, sz, P]),
    "plas_gather_rows": (i32, [P, i64, P, i64, P, P]),
    "plas_quantize_workspace_bytes": (sz, [i64, i32]),
    "plas_quantize_planes": (i32, [P, i64, i32, i64, i32, i32, f64, f64, i32, i32, i32, P, P, P, P, sz, P]),
    "plas_seed_key": (None, [u64, P]),
    "plas_host_permutation": (i32, [u64, i64, P]),
}

_lib = None
_lock = threading.Lock()


def load_library(path=LIB_PATH):
    """Load the .so and bind signatures (no CUDA call is made)."""
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the CUDA extension with __graft_entry__.build() "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def lib():
    """The bound library, after checking that a CUDA device is present."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch
                if not torch.cuda.is_available():
                    raise RuntimeError("paper_2312_13299_b200 needs a CUDA device (B200, sm_100a); "
                                       "there is no CPU fallback")
                torch.cuda.init()
                _lib = load_library()
    return _lib


def check(code, what):
    if code == PLAS_OK:
        return
    msg = lib().plas_last_error().decode(errors="replace")
    if code == PLAS_ERR_NONFINITE:
        raise ValueError("features must be finite")
    if code == PLAS_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({code}): {msg}")


def stream_handle():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device (torch) or host (numpy) data pointer as c_void_p; None -> NULL."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(t.data_ptr())


_ws = threading.local()


def workspace(nbytes, tag="main"):
    """A cached uint8 device buffer of at least nbytes (torch caching allocator).

    Buffers are private to (calling thread, device, current stream): the C ABI
    releases the GIL (ctypes), so two threads sorting at once, or one thread
    queueing asynchronous API calls on two streams, never share scratch memory.
    A thread's buffers are freed with the thread."""
    import torch
    dev = torch.cuda.current_device()
    cache = getattr(_ws, "bufs", None)
    if cache is None:
        cache = _ws.bufs = {}
    key = (tag, dev, torch.cuda.current_stream(dev).cuda_stream)
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=f"cuda:{dev}")
        cache[key] = buf
    return buf


def to_device(a, dtype):
    """numpy/torch array -> contiguous CUDA tensor of `dtype` (torch dtype)."""
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device="cuda", dtype=dtype, non_blocking=False).contiguous()
