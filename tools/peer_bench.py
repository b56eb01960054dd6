"""Peer-memory allreduce vs NCCL at the TP row-parallel shapes (config 4).

    torchrun --nproc-per-node N tools/peer_bench.py [--rows 2048] [--hidden 8192] [--iters 50]

One rank per GPU. For each message (rows x hidden fp32 — the O / down
partial of a Llama-3-70B prefill shard) times, with CUDA events and the max
over ranks: torch.distributed NCCL allreduce, and the peer kernel
(PeerAllreduce.allreduce_). Prints one JSON line per size on rank 0. With
N = 1 it only checks the plumbing (no link is crossed).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import torch.distributed as dist

    from paper_2512_09472_b200.peer import PeerAllreduce

    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="1,16,128,2048")
    ap.add_argument("--hidden", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    rows = [int(r) for r in a.rows.split(",")]
    pa = PeerAllreduce(max(rows) * a.hidden)

    def timed(fn, x):
        for _ in range(5):
            fn(x)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn(x)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for r in rows:
        x = torch.randn(r * a.hidden, device="cuda")
        ref = x.clone()
        dist.all_reduce(ref)
        y = x.clone()
        pa.allreduce_(y)
        ok = torch.allclose(y, ref, rtol=1e-5, atol=1e-5)
        nccl_ms = timed(lambda t: dist.all_reduce(t), x.clone())
        peer_ms = timed(lambda t: pa.allreduce_(t), x.clone())
        nbytes = r * a.hidden * 4
        if rank == 0:
            print(json.dumps({"world": world, "rows": r, "hidden": a.hidden, "bytes": nbytes, "match_nccl": ok,
                              "nccl_us": nccl_ms * 1e3, "peer_us": peer_ms * 1e3,
                              "peer_busbw_gbs": 2 * (world - 1) / world * nbytes / (peer_ms / 1e3) / 1e9
                              if world > 1 else None}), flush=True)
    pa.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
