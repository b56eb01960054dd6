"""Peer-memory allreduce (csrc/peer.cu): two or three processes sharing cuda:0
map each other's IPC buffers (the one-GPU stand-in for NVLink peers) and sum fp32
partials; the result must equal the rank-ordered sum bit for bit on both
ranks, across repeated calls (both data slots, epoch flags) and ragged
sizes."""

from __future__ import annotations

import os
import socket

import pytest
import torch

# two-shot from 1 MiB (262,144 floats): ragged sizes exercise the scalar tails of
# the chunk reduce / gather (n % 4 != 0, a short last chunk)
# (M, N, K) of the fused row-parallel GEMM + allreduce: 256-row tiles, a ragged
# last 128-row block (300, 1537), several waves of tiles (1024 x 1024), and the
# unfused fallback below 256 rows (40)
FUSED = [(512, 1024, 512), (300, 512, 256), (1024, 1024, 320), (40, 256, 128), (1537, 256, 256)]
SIZES = [1, 3, 1000, 4096 * 8 + 5, 1 << 20, 17, 1 << 20, (1 << 18) + 3, (1 << 20) + 7, (1 << 18) + 1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(rank, n, step):
    g = torch.Generator().manual_seed(1000 * step + 10 * rank + 7)
    return torch.randn(n, generator=g)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_09472_b200.peer import PeerAllreduce

        torch.cuda.set_device(0)
        pa = PeerAllreduce(max_count=(1 << 20) + 64)
        bad, fused_out = [], []
        for step, n in enumerate(SIZES):
            t = _inputs(rank, n, step).cuda()
            pa.allreduce_(t)
            want = _inputs(0, n, step)
            for r in range(1, world):
                want = want + _inputs(r, n, step)
            got = t.cpu()
            if not torch.equal(got, want):
                bad.append((step, n, (got - want).abs().max().item()))
        # fused form: partial written straight into the exported slot, x += sum
        for step, n in enumerate([4096 * 8 + 5, 1 << 20, 3, (1 << 18) + 3, (1 << 20) + 7]):
            x = _inputs(9, n, 50 + step).cuda()
            pa.next_slot(n).copy_(_inputs(rank, n, 100 + step).cuda())
            pa.reduce_add_(x)
            s = _inputs(0, n, 100 + step)
            for r in range(1, world):
                s = s + _inputs(r, n, 100 + step)
            want = _inputs(9, n, 50 + step) + s
            if not torch.equal(x.cpu(), want):
                bad.append(("fused", n, (x.cpu() - want).abs().max().item()))
        # row-parallel GEMM fused with its allreduce: block-pipelined two-shot
        # (M >= 256) and the unfused fallback (M < 256); x identical on all ranks
        for step, (M, Nn, K) in enumerate(FUSED):
            g = torch.Generator().manual_seed(7 * step + rank)
            A = torch.randn(M, K, generator=g).bfloat16()
            Wt = (torch.randn(Nn, K, generator=g) * 0.05).bfloat16()
            x0 = torch.randn(M, Nn, generator=torch.Generator().manual_seed(99 + step))
            x = x0.cuda()
            pa.gemm_reduce_add_(x, A.cuda(), Wt.cuda())
            torch.cuda.synchronize()
            want = x0.clone()
            for r in range(world):
                gr = torch.Generator().manual_seed(7 * step + r)
                Ar = torch.randn(M, K, generator=gr).bfloat16()
                Wr = (torch.randn(Nn, K, generator=gr) * 0.05).bfloat16()
                want += Ar.float() @ Wr.float().T
            got = x.cpu()
            rel = ((got - want).norm() / (want - x0).norm()).item()
            if not rel < 1e-2:
                bad.append(("gemm_reduce_add", M, Nn, K, rel))
            fused_out.append(got)
        with pytest.raises(Exception):
            pa.allreduce_(torch.zeros(8, device="cuda", dtype=torch.float64))
        pa.close()
        q.put((rank, (bad, [t.numpy().tobytes() for t in fused_out])))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_peer_allreduce_processes_share_one_gpu(cuda_device, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=240) for _ in range(world))  # read before joining
    finally:
        for p in procs:
            p.join(60)
            if p.exitcode is None:
                p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert {r: v[0] for r, v in res.items()} == {r: [] for r in range(world)}, res
    # the fused GEMM + allreduce leaves the same bits on every rank
    assert all(res[r][1] == res[0][1] for r in range(world))
