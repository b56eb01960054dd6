"""ctypes binding of the in-tree native library (include/warmserve.h).

The library is the product path: if it is missing this module raises at
import time — there is no Python or CPU fallback for anything it provides.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libwarmserve.so"

WS_OK = 0
WS_ERR_INVALID = 1
WS_ERR_INSUFFICIENT = 2
WS_ERR_DUPLICATE = 3
WS_ERR_NO_SLOT = 4
WS_ERR_STATE = 5
WS_ERR_CUDA = 6
WS_ERR_NO_DEVICE = 7
WS_ERR_KV_BUSY = 8
WS_ERR_FRAGMENTED = 9


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(no CPU fallback exists)"
    )

lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)

i32, i64, f64, f32 = C.c_int32, C.c_int64, C.c_double, C.c_float
vp = C.c_void_p
P = C.POINTER


class TransferPlanC(C.Structure):
    _fields_ = [
        ("total_bytes", i64),
        ("bandwidth", f64),
        ("chunk_pages", i64),
        ("page_size", i64),
        ("n_chunks", i64),
        ("first_chunk_map_ms", f64),
        ("finish_ms", f64),
        ("critical_path_stall_ms", f64),
    ]


class PoolCounts(C.Structure):
    _fields_ = [
        ("total_pages", i64),
        ("free_pages", i64),
        ("slot_pages", i64),
        ("kv_pages_mapped", i64),
        ("kv_pages_used", i64),
        ("kv_capacity_pages", i64),
        ("kv_pages_allocated", i64),
        ("n_slots", i64),
        ("pending_unmaps", i64),
    ]


# name -> argtypes; every function returns int status.
SIGNATURES: dict[str, list] = {
    "ws_version": [P(C.c_int), P(C.c_int)],
    "ws_kernel_launches": [P(i64)],
    "ws_fallback_counts": [P(i64), i32],
    "ws_required_prewarm_layers": [i64, i32, i32, f64, f64, f64, i32, P(i32)],
    "ws_catchup_stall_ms": [i64, i32, i32, f64, f64, i32, f64, i32, P(f64)],
    "ws_reservation_target": [f64, i32, i32, f64, P(f64)],
    "ws_partition_pages": [i64, i32, i64, P(i64), P(i64)],
    "ws_pipelined_load": [i64, f64, f64, i64, i64, P(TransferPlanC)],
    "ws_background_kv_mapping": [i64, f64, f64, P(f64)],
    "ws_pool_create": [i32, i64, i64, P(vp)],
    "ws_pool_create_ex": [i32, i64, i64, i64, P(vp)],
    "ws_pool_handle_pages": [vp, P(i64)],
    "ws_pool_destroy": [vp],
    "ws_pool_counts_get": [vp, P(PoolCounts)],
    "ws_pool_owner_map": [vp, P(i32), i64],
    "ws_pool_device_owner_map": [vp, P(i32), i64],
    "ws_pool_window": [vp, P(vp)],
    "ws_pool_timing": [vp, P(f64), P(f64), P(f64)],
    "ws_pool_sync_unmaps": [vp],
    "ws_slot_create": [vp, i64, i64, i32, P(vp)],
    "ws_slot_create_keyed": [vp, i64, i64, i32, C.c_uint64, P(vp)],
    "ws_pool_map_stats": [vp, P(i64), P(i64)],
    "ws_slot_map_chunk": [vp, i64, i64, i64],
    "ws_slot_evict": [vp, i64, vp],
    "ws_slot_info": [vp, i64, P(i64), P(i64), P(vp)],
    "ws_slot_pages": [vp, i64, P(i32), i64, P(i64)],
    "ws_slot_placement": [vp, i64, P(i32), P(i64)],
    "ws_pool_export_slot": [vp, i64, P(i32), P(i64), i64, P(i64), P(i64)],
    "ws_peer_map_import": [i32, P(i32), P(i64), i64, P(vp), P(vp)],
    "ws_peer_map_release": [vp],
    "ws_device_can_access_peer": [i32, i32, P(i32)],
    "ws_kv_map_all": [vp, vp, P(i64)],
    "ws_kv_reclaim": [vp, i32, i32, f64, vp, P(i64)],
    "ws_kv_resize": [vp, i64, vp],
    "ws_kv_release": [vp, vp],
    "ws_pool_seq_config": [vp, i32, i32],
    "ws_seq_open": [vp, P(i32)],
    "ws_seq_reserve": [vp, i32, i32, vp],
    "ws_seq_close": [vp, i32],
    "ws_seq_blocks": [vp, i32, P(i32), i32, P(i32)],
    "ws_pool_block_tables": [vp, P(vp), P(i32)],
    "ws_pool_last_switch": [vp, P(f64), P(i64)],
    "ws_streamer_create": [i32, P(vp)],
    "ws_streamer_destroy": [vp],
    "ws_streamer_start": [vp, vp, vp, P(i64), i32, vp],
    "ws_streamer_start_packed": [vp, vp, vp, P(i64), i32, vp, i64, vp, vp],
    "ws_streamer_wait": [vp, i32, vp],
    "ws_streamer_progress": [vp, P(i32)],
    "ws_streamer_sync": [vp, i32],
    "ws_streamer_times": [vp, P(f32), i32],
    "ws_peer_buffer_bytes": [i64, P(i64)],
    "ws_peer_buffer_alloc": [i64, P(vp), P(C.c_uint8), i32],
    "ws_peer_buffer_free": [vp],
    "ws_peer_buffer_open": [P(C.c_uint8), P(vp)],
    "ws_peer_buffer_close": [vp],
    "ws_peer_create": [i32, i32, P(vp), i64, P(vp)],
    "ws_peer_destroy": [vp],
    "ws_peer_allreduce_f32": [vp, vp, i64, vp],
    "ws_comm_set_peer": [vp, vp, i64],
    "ws_peer_next_slot": [vp, P(vp)],
    "ws_peer_reduce_add_f32": [vp, vp, i64, vp],
    "ws_peer_gemm_reduce_add": [vp, vp, vp, i32, i32, i32, vp, vp],
    "ws_peer_allgather_f32": [vp, vp, vp, i64, vp],
    "ws_comm_create_peer": [i32, i32, i32, vp, i64, P(vp)],
}

lib.ws_last_error.restype = C.c_char_p
lib.ws_last_error.argtypes = []


def _bind(name, argtypes):
    fn = getattr(lib, name)
    fn.argtypes = argtypes
    fn.restype = C.c_int
    return fn


fns = {}


def register(sigs: dict) -> None:
    for name, argtypes in sigs.items():
        fns[name] = _bind(name, argtypes)


register(SIGNATURES)


def call(name: str, *args) -> None:
    rc = fns[name](*args)
    if rc != WS_OK:
        raise NativeError(rc, lib.ws_last_error().decode(errors="replace"))


def kernel_launches() -> int:
    v = C.c_int64()
    call("ws_kernel_launches", C.byref(v))
    return v.value


def last_error() -> str:
    return lib.ws_last_error().decode(errors="replace")


def declared_symbols() -> list[str]:
    """Every function include/warmserve.h declares (for the export test)."""
    import re

    hdr = Path(__file__).resolve().parent.parent / "include"
    names = []
    for h in sorted(hdr.glob("*.h")):
        names += re.findall(r"^\s*(?:int|const char\*)\s+(ws_\w+)\s*\(", h.read_text(), re.M)
    return names


def fallback_counts() -> dict:
    """Legacy-kernel fallbacks since load (ws_fallback_counts)."""
    out = (C.c_int64 * 3)()
    call("ws_fallback_counts", out, 3)
    return {"gemm_mma_sync": out[0], "gemm_gemv": out[1], "attn_prefill_mma_sync": out[2]}
