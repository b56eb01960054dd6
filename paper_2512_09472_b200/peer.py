"""Allreduce over peer memory (csrc/peer.cu) for the TP row-parallel partials.

Each rank exports one CUDA IPC buffer; the 64-byte handles are exchanged over
a torch.distributed group (any backend — the data path does not use it), and
every rank maps every peer's buffer. ``allreduce_(t)`` sums an fp32 CUDA
tensor in place across the group; every rank must issue the same sequence of
calls. The replacement for ``ncclAllReduce`` on the O / down partials
(SURVEY §8e); on one node the peer loads travel over NVLink / NVSwitch.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N

HANDLE_BYTES = 64


class PeerAllreduce:
    def __init__(self, max_count: int, group=None):
        import torch.distributed as dist

        single = not dist.is_initialized()
        self._group = group
        self._single = single
        self.rank = 0 if single else dist.get_rank(group)
        self.world = 1 if single else dist.get_world_size(group)
        self.max_count = int(max_count)
        own = C.c_void_p()
        handle = (C.c_uint8 * HANDLE_BYTES)()
        N.call("ws_peer_buffer_alloc", self.max_count, C.byref(own), handle, HANDLE_BYTES)
        self._own = own
        handles: list = [bytes(handle)]
        if not single:
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(handle), group=group)
        self._opened = []
        ptrs = (C.c_void_p * self.world)()
        for r, h in enumerate(handles):
            if r == self.rank:
                ptrs[r] = own.value
                continue
            p = C.c_void_p()
            hb = (C.c_uint8 * HANDLE_BYTES).from_buffer_copy(h)
            N.call("ws_peer_buffer_open", hb, C.byref(p))
            self._opened.append(p)
            ptrs[r] = p.value
        self._h = C.c_void_p()
        N.call("ws_peer_create", self.rank, self.world, ptrs, self.max_count, C.byref(self._h))

    def allreduce_(self, t: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("allreduce_ takes a contiguous fp32 CUDA tensor")
        st = stream if stream is not None else torch.cuda.current_stream(t.device)
        N.call("ws_peer_allreduce_f32", self._h, C.c_void_p(t.data_ptr()), t.numel(), C.c_void_p(st.cuda_stream))
        return t

    def next_slot(self, count: int, device: int | None = None) -> torch.Tensor:
        """fp32 view of this rank's exported slot for the next call: write the
        partial here, then reduce_add_ (no staging copy)."""
        from .devmem import view

        p = C.c_void_p()
        N.call("ws_peer_next_slot", self._h, C.byref(p))
        return view(p.value, (count,), torch.float32, torch.cuda.current_device() if device is None else device)

    def reduce_add_(self, x: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """x += sum over ranks of the partials each rank wrote into next_slot()."""
        if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
            raise ValueError("reduce_add_ takes a contiguous fp32 CUDA tensor")
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        N.call("ws_peer_reduce_add_f32", self._h, C.c_void_p(x.data_ptr()), x.numel(), C.c_void_p(st.cuda_stream))
        return x

    def gemm_reduce_add_(self, x: torch.Tensor, A: torch.Tensor, W: torch.Tensor,
                         stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """x[M, N] += sum over ranks of A_r W_r^T (bf16 A [M, K], W [N, K]):
        the row-parallel GEMM fused with its allreduce (ws_peer_gemm_reduce_add)."""
        if x.dtype != torch.float32 or A.dtype != torch.bfloat16 or W.dtype != torch.bfloat16:
            raise ValueError("gemm_reduce_add_ takes fp32 x and bf16 A, W")
        M, K = A.shape
        Nn = W.shape[0]
        if tuple(x.shape) != (M, Nn) or W.shape[1] != K or not (x.is_contiguous() and A.is_contiguous()
                                                                and W.is_contiguous()):
            raise ValueError("gemm_reduce_add_: x [M, N], A [M, K], W [N, K], contiguous")
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        N.call("ws_peer_gemm_reduce_add", self._h, C.c_void_p(A.data_ptr()), C.c_void_p(W.data_ptr()), M, Nn, K,
               C.c_void_p(x.data_ptr()), C.c_void_p(st.cuda_stream))
        return x

    def close(self) -> None:
        if self._h:
            torch.cuda.synchronize()
            if not self._single:
                # A slower peer may still be inside its last peer kernel, reading
                # this rank's exported slot: free nothing until every rank is done.
                import torch.distributed as dist

                dist.barrier(group=self._group)
            N.call("ws_peer_destroy", self._h)
            self._h = C.c_void_p()
            for p in self._opened:
                N.call("ws_peer_buffer_close", p)
            self._opened = []
            N.call("ws_peer_buffer_free", self._own)
