"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference memory-switch model.

Restates ``/root/reference/pkg/src/prewarmsim/memswitch.py`` and the
sequential (numba) pipeline schedule of ``kernels.py:68-77`` with explicit
per-chunk loops, so that finish/stall values are reproduced bit-for-bit in
float64. Pinned against the reference's own outputs (``tests/golden``).
"""

from __future__ import annotations

import math


def chunk_plan(total_bytes: int, chunk_pages: int, page_size: int):
    """Per-chunk (pages, bytes): memswitch.py:78-84. The last chunk holds the
    remainder of the page count and the last page may be partial."""
    pages = int(math.ceil(total_bytes / page_size))
    n_chunks = int(math.ceil(pages / chunk_pages))
    out = []
    done_pages = 0
    done_bytes = 0
    for c in range(n_chunks):
        cp = chunk_pages if c < n_chunks - 1 else pages - chunk_pages * (n_chunks - 1)
        done_pages += cp
        end = min(done_pages * page_size, total_bytes)
        out.append((cp, end - done_bytes))
        done_bytes = end
    return out


def pipeline_finish(map_ms, transfer_ms) -> float:
    """Two-stage schedule: maps back to back; copy c starts after map c and
    copy c-1 — kernels.py:68-77 (the sequential form the reference runs)."""
    mapped = 0.0
    done = 0.0
    for m, t in zip(map_ms, transfer_ms):
        mapped += m
        done = (mapped if mapped > done else done) + t
    return done


def pipelined_load(total_bytes, bandwidth, mu, chunk_pages, page_size):
    """memswitch.py:59-98 → dict(n_chunks, first_chunk_map_ms, finish_ms, stall_ms)."""
    if bandwidth <= 0:
        raise ValueError("bandwidth must be > 0")
    if total_bytes <= 0:
        raise ValueError("total_bytes must be > 0")
    if chunk_pages < 1:
        raise ValueError("chunk_pages must be >= 1")
    plan = chunk_plan(total_bytes, chunk_pages, page_size)
    map_ms = [float(p) * mu for p, _ in plan]
    tr_ms = [float(b) / bandwidth for _, b in plan]
    finish = pipeline_finish(map_ms, tr_ms)
    stall = finish - total_bytes / bandwidth - map_ms[0]
    return dict(
        n_chunks=len(plan),
        first_chunk_map_ms=map_ms[0],
        finish_ms=finish,
        stall_ms=stall if stall > 0.0 else 0.0,
    )


def background_kv_mapping(pages, mu, rate) -> float:
    """pages * (mu - 1/rate) when positive — memswitch.py:101-117."""
    if pages < 0:
        raise ValueError("pages must be >= 0")
    if mu <= 0 or rate <= 0:
        raise ValueError("rates must be positive")
    deficit = mu - 1.0 / rate
    return pages * deficit if deficit > 0 else 0.0


def unmap_cost_ms(pages, mu) -> float:
    """memswitch.py:120-122."""
    return pages * mu


def slot_layers_at(layers_loaded, load_start, load_finish, t, layers, partition_bytes, layer_bytes):
    """Linear layer residency during a transfer — engine.py:426-432."""
    if load_finish is None or t >= load_finish:
        return layers_loaded
    if load_start is None or t <= load_start:
        return 0
    frac = (t - load_start) / (load_finish - load_start)
    return min(layers, int(frac * partition_bytes // layer_bytes))
