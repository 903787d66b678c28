"""ctypes binding of libtpshift_b200.so (the C ABI in include/tpshift_b200.h).

The CUDA engine is the only execution path: if the library is missing or the
device is not sm_100, every runtime entry point raises. There is no CPU or
eager-PyTorch fallback for the hot path.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, PlanVerificationError

LIB_NAME = "libtpshift_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
# dev A/B only: TPS_LIB_PATH points at an alternative build of the same library
LIB_PATH = os.environ.get("TPS_LIB_PATH", LIB_PATH)

TPS_OK = 0
TPS_EINVAL = -22
TPS_EPLAN = -1001
TPS_ECUDA = -1002

# Every entry point declared in include/tpshift_b200.h, with its ctypes signature.
_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_f32 = ctypes.c_float
_pp = ctypes.c_void_p  # pointer to a host array of device pointers

SIGNATURES = {
    "tps_version": (ctypes.c_char_p, []),
    "tps_last_error": (ctypes.c_char_p, []),
    "tps_init": (_i32, [_i32, ctypes.POINTER(_i32)]),
    "tps_set_pdl": (None, [_i32]),
    "tps_linear_splits": (_i32, [_i64, _i64, _i64]),
    "tps_cluster_splits": (_i32, [_i64, _i64, _i64]),
    "tps_linear_argmax": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _i32, _vp]),
    "tps_linear_push_ll_cluster": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _pp, _i32, _vp,
                                          ctypes.c_uint32, ctypes.c_uint32, _vp]),
    "tps_gemv_max_rows": (_i32, []),
    "tps_gemv": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp]),
    "tps_gemv_silu": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp]),
    "tps_gemv_push_ll": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _pp, _i32, _vp, ctypes.c_uint32,
                                ctypes.c_uint32, _vp]),
    "tps_gemv_argmax": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _i32, _vp]),
    "tps_prefill_group_positions": (_i32, [_i32]),
    "tps_prefill_attention": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _i32, _i32, _i32, _i32, _vp,
                                     _vp]),
    "tps_linear": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _vp, _i32, _vp]),
    "tps_linear_push": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _pp, _i32, _i64, _i32, _pp, _i32,
                                _vp, _vp]),
    "tps_linear_push_ll": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _pp, _i32, _i64, _i32, _vp,
                                   ctypes.c_uint32, ctypes.c_uint32, _vp]),
    "tps_add_norm_ll": (_i32, [_vp, _vp, _i32, _i64, _vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _f32, _i32, _i32,
                               _vp, _i32, _vp, ctypes.c_uint64, _vp]),
    "tps_linear_silu": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _vp]),
    "tps_embed": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp, _i32, _i32, _vp, _vp]),
    "tps_add_norm": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp, _f32, _i32, _i32, _vp, _i32, _vp]),
    "tps_reduce_push_ll": (_i32, [_vp, _i32, _i64, _pp, _i32, _i64, _vp, ctypes.c_uint32, ctypes.c_uint32, _vp]),
    "tps_reduce_push": (_i32, [_vp, _i32, _i64, _pp, _i32, _i64, _pp, _i32, _vp, _vp]),
    "tps_qkv_rope_append": (_i32, [_vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _i32, _i32,
                                   _i32, _i32, _vp, _vp, _vp, _vp]),
    "tps_attn_splits": (_i32, [_i32, _i32, _i32]),
    "tps_attn_workspace": (_i64, [_i32, _i32, _i32, _i32]),
    "tps_paged_attention": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32,
                                   _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp]),
    "tps_silu_mul": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _i32, _vp]),
    "tps_argmax_stage1": (_i32, [_vp, _i32, _i64, _i32, _i32, _i32, _i32, _vp, _pp, _i32, _vp, _vp]),
    "tps_sample_stage1": (_i32, [_vp, _i32, _i64, _i32, _i32, _i32, _i32, _vp, _pp, _i32, _vp, _vp, _vp, _vp, _vp,
                                  _f32, _vp]),
    "tps_argmax_finalize": (_i32, [_pp, _i32, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "tps_epoch_advance": (_i32, [_vp, _vp]),
    "tps_sum_partials": (_i32, [_vp, _i32, _i64, _i64, _vp, _vp]),
    "tps_abort_status": (ctypes.c_uint32, []),
    "tps_abort_clear": (None, []),
    "tps_copy_items": (_i32, [_vp, _i32, _i32, _i32, _vp]),
    "tps_kv_move_items": (_i32, [_vp, _i32, _i64, _vp, _i32, _i32, _i64, _vp, _vp, _vp]),
    "tps_barrier": (_i32, [_pp, _i32, _vp, _i32, _i32, ctypes.c_uint64, _vp]),
    "tps_ipc_get_handle": (_i32, [_vp, _vp, ctypes.POINTER(_i64)]),
    "tps_ipc_open": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "tps_ipc_close": (_i32, [_vp]),
    "tps_trace_enable": (_i32, [_vp, _vp, ctypes.c_uint]),
    "tps_persist_struct_bytes": (_i64, [_i32]),
    "tps_persist_supported": (_i32, [_vp, _vp, _i32]),
    "tps_persist_work_bytes": (_i64, [_vp, _vp, _i32]),
    "tps_persist_ctx_bytes": (_i64, [_vp, _i32]),
    "tps_persist_prepare": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _vp]),
    "tps_persist_launch": (_i32, [_vp, _i32, _i32, _i32, _vp]),
}


class PersistGeom(ctypes.Structure):
    """tps_persist_geom (include/tpshift_b200.h)."""
    _fields_ = [("num_layers", _i32), ("hidden", _i32), ("head_dim", _i32), ("n_phases", _i32),
                ("rms_eps", _f32)]


class PersistRank(ctypes.Structure):
    """tps_persist_rank (include/tpshift_b200.h)."""
    _fields_ = [("w_qkv", _vp), ("b_qkv", _vp), ("w_o", _vp), ("w_gu", _vp), ("w_d", _vp), ("ln1", _vp),
                ("ln2", _vp), ("embed", _vp), ("ln_f", _vp), ("lm_head", _vp), ("k_cache", _vp), ("v_cache", _vp),
                ("nq", _i32), ("nkv", _i32), ("ffn", _i32), ("vocab", _i32), ("vocab_off", _i32),
                ("nq_of", _i32 * 8), ("row_slot", _vp), ("pos", _vp), ("page_table", _vp), ("max_pages", _i32), ("history", _vp),
                ("hist_ld", _i32), ("prompt_len", _vp), ("out_tok", _vp), ("logits", _vp), ("cos_t", _vp),
                ("sin_t", _vp), ("work", _vp), ("work_bytes", _i64), ("tp", _i32), ("rank", _i32),
                ("loopback", _i32), ("ll_par_stride", _i64), ("ll_src_stride", _i64), ("ll_peer", _vp * 8),
                ("ll_mine", _vp), ("am_peer", _vp * 8), ("am_mine", _vp), ("epoch", _vp), ("ctr", _vp), ("trace", _vp),
                ("trace_layer", _i32)]


class TpsWait(ctypes.Structure):
    _fields_ = [("ctr", ctypes.c_void_p), ("epoch", ctypes.c_void_p),
                ("mult", ctypes.c_uint64), ("add", ctypes.c_uint64)]


COPY_ITEM_BYTES = 32

_lock = threading.Lock()
_lib = None


class NativeUnavailable(RuntimeError):
    """The CUDA engine library could not be loaded."""


def load_library(path: str = LIB_PATH):
    """Load the library and bind every declared symbol (raises if any is absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `make` (or __graft_entry__.build()); "
                "the B200 engine has no fallback path")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError if the ABI is incomplete
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


def check_abort(what: str = "") -> None:
    """Raise if a device watchdog fired (the soft-abort word, include/tpshift_b200.h): the work
    queued since is garbage. The word is cleared so the process can continue after reporting."""
    code = lib().tps_abort_status()
    if code:
        lib().tps_abort_clear()
        raise RuntimeError(f"libtpshift_b200 device watchdog fired (code {code}){': ' + what if what else ''}; "
                           f"results since are invalid")


def check(rc: int, what: str = "") -> None:
    if rc == TPS_OK:
        if _lib is not None and _lib.tps_abort_status():
            check_abort(what)
        return
    msg = lib().tps_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == TPS_EINVAL:
        raise ConfigError(text)
    if rc == TPS_EPLAN:
        raise PlanVerificationError(text)
    raise RuntimeError(f"libtpshift_b200 error {rc}: {text}")


def ptr_array(ptrs) -> ctypes.Array:
    """Host array of device pointers (kept alive by the caller for the call)."""
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = int(p)
    return arr


def wait_spec(ctr: int | None, epoch: int | None = None, mult: int = 0, add: int = 0):
    if not ctr:
        return None
    return ctypes.byref(TpsWait(ctypes.c_void_p(int(ctr)),
                                ctypes.c_void_p(int(epoch)) if epoch else None,
                                int(mult), int(add)))


_initialized_devices: set[int] = set()


def init_device(device: int) -> int:
    """tps_init: bind + verify sm_100; returns the SM count."""
    sm = ctypes.c_int(0)
    check(lib().tps_init(int(device), ctypes.byref(sm)), "tps_init")
    _initialized_devices.add(int(device))
    return sm.value
