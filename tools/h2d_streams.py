"""Pinned-host -> device copy bandwidth with 1 / 2 / 4 concurrent copy streams
(4 GiB total): the PCIe Gen5 ceiling the cold-start stream runs at
(~55 GB/s on this B200 whatever the stream count).

    python tools/h2d_streams.py
"""
import torch, time
n = 1 << 30  # 1 GiB
h = torch.empty(4 * n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(4 * n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chunk = 4 * n // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams={ns}: {4 * n / dt / 1e9:.1f} GB/s")
