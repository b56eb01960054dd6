"""Memory-switch model API of the reference, computed natively.

Drop-in for ``prewarmsim.memswitch`` (memswitch.py:21-122): the schedule of the
chunked map/copy weight loader, the background KV-mapping race and the async
unmap cost. The B200 worker uses ``pipelined_load`` to plan its own loader and
reports the *measured* per-page map cost next to the modeled one.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native as N


@dataclass(frozen=True)
class MappingOp:
    """memswitch.py:21-40."""

    gpu_id: int
    target: str
    pages: int
    kind: str
    issue_ms: float
    map_ms_per_page: float

    def __post_init__(self):
        if self.pages < 1:
            raise ValueError("mapping op needs at least one page")
        if self.map_ms_per_page <= 0:
            raise ValueError("map latency must be positive")
        if self.kind not in ("map", "unmap"):
            raise ValueError(f"unknown mapping kind {self.kind!r}")

    @property
    def duration_ms(self) -> float:
        return self.pages * self.map_ms_per_page


@dataclass(frozen=True)
class TransferPlan:
    """memswitch.py:43-56."""

    total_bytes: int
    bandwidth: float
    chunk_pages: int
    page_size: int
    n_chunks: int
    first_chunk_map_ms: float
    finish_ms: float
    critical_path_stall_ms: float

    @property
    def transfer_ms(self) -> float:
        return self.total_bytes / self.bandwidth


def pipelined_load(total_bytes: int, bandwidth: float, map_ms_per_page: float, chunk_pages: int,
                   page_size: int) -> TransferPlan:
    """memswitch.py:59-98 via ws_pipelined_load."""
    out = N.TransferPlanC()
    try:
        N.call("ws_pipelined_load", int(total_bytes), float(bandwidth), float(map_ms_per_page),
               int(chunk_pages), int(page_size), C.byref(out))
    except N.NativeError as e:
        raise ValueError(str(e)) from None
    return TransferPlan(out.total_bytes, out.bandwidth, out.chunk_pages, out.page_size, out.n_chunks,
                        out.first_chunk_map_ms, out.finish_ms, out.critical_path_stall_ms)


def background_kv_mapping(pages: int, map_ms_per_page: float, consumption_rate: float) -> float:
    """memswitch.py:101-117 via ws_background_kv_mapping."""
    out = C.c_double()
    try:
        N.call("ws_background_kv_mapping", int(pages), float(map_ms_per_page), float(consumption_rate),
               C.byref(out))
    except N.NativeError as e:
        raise ValueError(str(e)) from None
    return out.value


def unmap_cost_ms(pages: int, map_ms_per_page: float) -> float:
    """memswitch.py:120-122."""
    return pages * map_ms_per_page
