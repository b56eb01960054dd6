"""Zero-copy torch views of native device memory (slot VAs, the page window).

torch is plumbing here: it provides tensors over addresses the native pool
owns, via the CUDA array interface, so kernels and tests can address slot
weights and KV pages without copies.
"""

from __future__ import annotations

import torch

_TYPESTR = {
    torch.uint8: "|u1",
    torch.int8: "|i1",
    torch.int32: "<i4",
    torch.int64: "<i8",
    torch.float32: "<f4",
    torch.bfloat16: "<V2",  # no bf16 typestr; viewed as int16 then reinterpreted
    torch.float16: "<f2",
    torch.int16: "<i2",
}


class _Raw:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape),
            "typestr": typestr,
            "data": (int(ptr), False),
            "version": 3,
            "strides": None,
        }


def view(ptr: int, shape, dtype: torch.dtype, device: int = 0) -> torch.Tensor:
    """Tensor aliasing ``ptr`` (no ownership; the pool keeps the memory)."""
    if not ptr:
        raise ValueError("null device pointer")
    if dtype == torch.bfloat16:
        t = torch.as_tensor(_Raw(ptr, shape, "<i2"), device=f"cuda:{device}")
        return t.view(torch.bfloat16)
    return torch.as_tensor(_Raw(ptr, shape, _TYPESTR[dtype]), device=f"cuda:{device}")


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
