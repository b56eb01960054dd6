"""Device page pool on a real B200: VMM aliasing, switch kernel, migrations,
async unmap, layer streamer. Parity: device owner map == host ledger ==
oracle-derived identities; block tables rewritten bit-exactly."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PAGE = 2 * 1024 * 1024


@pytest.fixture()
def torch_cuda(cuda_device):
    import torch

    torch.cuda.set_device(cuda_device)
    return torch


def _pool(n_pages):
    from paper_2512_09472_b200 import _native as N

    h = C.c_void_p()
    N.call("ws_pool_create", 0, n_pages, PAGE, C.byref(h))
    return h


def _owner(h, n, device=True):
    from paper_2512_09472_b200 import _native as N

    out = np.empty(n, np.int32)
    fn = "ws_pool_device_owner_map" if device else "ws_pool_owner_map"
    N.call(fn, h, out.ctypes.data_as(C.POINTER(C.c_int32)), n)
    return out


def test_slot_va_aliases_page_window(torch_cuda):
    torch = torch_cuda
    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200.devmem import view

    n = 64
    h = _pool(n)
    try:
        va1, va2 = C.c_void_p(), C.c_void_p()
        N.call("ws_slot_create", h, 0, 5, 1, C.byref(va1))
        N.call("ws_slot_create", h, 1, 7, 1, C.byref(va2))
        N.call("ws_slot_evict", h, 0, None)
        va3 = C.c_void_p()
        N.call("ws_slot_create", h, 2, 9, 1, C.byref(va3))  # takes pages 0-4 then 12-15
        ids = (C.c_int32 * 9)()
        cnt = C.c_int64()
        N.call("ws_slot_pages", h, 2, ids, 9, C.byref(cnt))
        assert list(ids) == [0, 1, 2, 3, 4, 12, 13, 14, 15]
        slot = view(va3.value, (9 * PAGE // 4,), torch.int32)
        slot.copy_(torch.arange(slot.numel(), device="cuda", dtype=torch.int32))
        base = C.c_void_p()
        N.call("ws_pool_window", h, C.byref(base))
        win = view(base.value, (n * PAGE // 4,), torch.int32)
        torch.cuda.synchronize()
        per = PAGE // 4
        for j, p in enumerate(ids):
            assert torch.equal(win[p * per:(p + 1) * per], slot[j * per:(j + 1) * per])
        host = _owner(h, n, device=False)
        dev = _owner(h, n, device=True)
        assert np.array_equal(host, dev)
        assert host[:5].tolist() == [2] * 5 and host[5:12].tolist() == [1] * 7
        N.call("ws_pool_sync_unmaps", h)
        init_ms, map_pp, unmap_pp = C.c_double(), C.c_double(), C.c_double()
        N.call("ws_pool_timing", h, C.byref(init_ms), C.byref(map_pp), C.byref(unmap_pp))
        print(f"\nVMM: init {init_ms.value:.1f} ms for {n} pages, map {map_pp.value*1e3:.1f} us/page, "
              f"unmap {unmap_pp.value*1e3:.1f} us/page")
        assert map_pp.value > 0 and unmap_pp.value > 0
    finally:
        N.call("ws_pool_destroy", h)


def test_switch_promote_reclaim_release_device_parity(torch_cuda):
    torch = torch_cuda
    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200.devmem import view

    n = 96
    h = _pool(n)
    try:
        for sid, pages in ((0, 20), (1, 30), (2, 10)):
            N.call("ws_slot_create", h, sid, pages, 1, C.byref(C.c_void_p()))
        N.call("ws_slot_evict", h, 0, None)
        N.call("ws_slot_evict", h, 2, None)
        kv = C.c_int64()
        N.call("ws_kv_map_all", h, None, C.byref(kv))
        assert kv.value == n - 30
        N.call("ws_pool_seq_config", h, 4, 32)
        s = C.c_int32()
        N.call("ws_seq_open", h, C.byref(s))
        N.call("ws_seq_reserve", h, s.value, 3, None)  # pages 0,1,2
        t = C.c_int32()
        N.call("ws_seq_open", h, C.byref(t))
        N.call("ws_seq_reserve", h, t.value, 2, None)  # pages 3,4
        N.call("ws_seq_close", h, s.value)  # frees 0,1,2 (still KV)
        # live block pages 3,4 carry a signature
        base = C.c_void_p()
        N.call("ws_pool_window", h, C.byref(base))
        win = view(base.value, (n, PAGE // 4), torch.int32)
        win[3].fill_(333)
        win[4].fill_(444)
        # shrink KV to 3 pages: 3,4 must migrate to 0,1
        N.call("ws_kv_resize", h, 3, None)
        torch.cuda.synchronize()
        blk = (C.c_int32 * 2)()
        nb = C.c_int32()
        N.call("ws_seq_blocks", h, t.value, blk, 2, C.byref(nb))
        assert list(blk) == [0, 1]
        assert int(win[0][0]) == 333 and int(win[1][-1]) == 444
        bt_dev, maxb = C.c_void_p(), C.c_int32()
        N.call("ws_pool_block_tables", h, C.byref(bt_dev), C.byref(maxb))
        bt = view(bt_dev.value, (4, maxb.value), torch.int32)
        assert bt[t.value, :2].tolist() == [0, 1]
        assert np.array_equal(_owner(h, n, False), _owner(h, n, True))
        ms, ent = C.c_double(), C.c_int64()
        N.call("ws_pool_last_switch", h, C.byref(ms), C.byref(ent))
        print(f"\nswitch kernel (2 migrations): {ms.value*1e3:.1f} us")
        N.call("ws_seq_close", h, t.value)
        N.call("ws_kv_release", h, None)
        own = _owner(h, n, True)
        assert np.array_equal(own, _owner(h, n, False))
        assert (own == -2).sum() == 0 and (own == 1).sum() == 30
    finally:
        N.call("ws_pool_destroy", h)


def test_streamer_host_to_slot(torch_cuda):
    torch = torch_cuda
    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200.devmem import view

    n = 40
    h = _pool(n)
    st = C.c_void_p()
    N.call("ws_streamer_create", 8, C.byref(st))
    try:
        va = C.c_void_p()
        N.call("ws_slot_create", h, 0, 32, 1, C.byref(va))
        src = torch.randint(0, 1 << 30, (32 * PAGE // 4,), dtype=torch.int32).pin_memory()
        ranges = (C.c_int64 * 24)()
        per = 4 * PAGE
        for i in range(8):
            ranges[3 * i], ranges[3 * i + 1], ranges[3 * i + 2] = i * per, i * per, per
        copy = torch.cuda.Stream()
        N.call("ws_streamer_start", st, va, C.c_void_p(src.data_ptr()), ranges, 8, C.c_void_p(copy.cuda_stream))
        comp = torch.cuda.current_stream()
        N.call("ws_streamer_wait", st, 7, C.c_void_p(comp.cuda_stream))
        dst = view(va.value, (32 * PAGE // 4,), torch.int32)
        got = dst.clone()
        torch.cuda.synchronize()
        assert torch.equal(got.cpu(), src)
        times = (C.c_float * 8)()
        N.call("ws_streamer_times", st, times, 8)
        gbs = 32 * PAGE / (times[7] * 1e-3) / 1e9
        print(f"\nH2D stream 64 MiB in 8 ranges: {times[7]:.2f} ms = {gbs:.1f} GB/s")
        assert list(times) == sorted(times)
    finally:
        N.call("ws_streamer_destroy", st)
        N.call("ws_pool_destroy", h)


def test_device_cluster_replays_config3_golden(torch_cuda, ledger_traces):
    """The config-3 trace (89,600-page ledger, 4 models) replayed on a
    device-backed Cluster at reduced page count is impossible (counts must
    match), so replay the KAT ledger trace with a device pool (page_size 1
    is ledger-only); here: a 2 MiB-page scenario built from the walker ops."""
    from ledger_replay import ClusterBackend, replay

    for t in ledger_traces:
        if t["name"] == "engine_grace":
            servers, per, pages, page, bw = t["init"]
            if pages * page > 8 << 30:
                continue
            replay(t, ClusterBackend(t["init"], devices={0: 0}))
