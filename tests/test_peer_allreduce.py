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
        bad = []
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
        with pytest.raises(Exception):
            pa.allreduce_(torch.zeros(8, device="cuda", dtype=torch.float64))
        pa.close()
        q.put((rank, bad))
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
    assert res == {r: [] for r in range(world)}, res
