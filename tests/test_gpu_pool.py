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


def _pool(n_pages, handle_pages=16):
    from paper_2512_09472_b200 import _native as N

    h = C.c_void_p()
    N.call("ws_pool_create_ex", 0, n_pages, PAGE, handle_pages, C.byref(h))
    return h


def _owner(h, n, device=True):
    from paper_2512_09472_b200 import _native as N

    out = np.empty(n, np.int32)
    fn = "ws_pool_device_owner_map" if device else "ws_pool_owner_map"
    N.call(fn, h, out.ctypes.data_as(C.POINTER(C.c_int32)), n)
    return out


def _check_slot_data(torch, h, n, va, ids):
    """Write through the slot VA, read through the page window: slot page j
    must be physical page ids[j]."""
    from paper_2512_09472_b200 import _native as N
    from paper_2512_09472_b200.devmem import view

    slot = view(va, (len(ids) * PAGE // 4,), torch.int32)
    slot.copy_(torch.arange(slot.numel(), device="cuda", dtype=torch.int32))
    base = C.c_void_p()
    N.call("ws_pool_window", h, C.byref(base))
    win = view(base.value, (n * PAGE // 4,), torch.int32)
    torch.cuda.synchronize()
    per = PAGE // 4
    for j, p in enumerate(ids):
        assert torch.equal(win[p * per:(p + 1) * per], slot[j * per:(j + 1) * per]), (j, p)


def _placement(h, sid):
    from paper_2512_09472_b200 import _native as N

    kind, nh = C.c_int32(), C.c_int64()
    N.call("ws_slot_placement", h, sid, C.byref(kind), C.byref(nh))
    ids = (C.c_int32 * 4096)()
    cnt = C.c_int64()
    N.call("ws_slot_pages", h, sid, ids, 4096, C.byref(cnt))
    return kind.value, nh.value, list(ids)[: cnt.value]


def test_windowed_slots_alias_the_page_window(torch_cuda):
    """A slot on a contiguous free run IS a range of the page window: its VA
    is window + first*page, created and evicted with no driver call."""
    torch = torch_cuda
    from paper_2512_09472_b200 import _native as N

    n = 64
    h = _pool(n)
    try:
        va1, va2 = C.c_void_p(), C.c_void_p()
        N.call("ws_slot_create", h, 0, 5, 1, C.byref(va1))
        N.call("ws_slot_create", h, 1, 7, 1, C.byref(va2))
        N.call("ws_slot_evict", h, 0, None)
        va3 = C.c_void_p()
        N.call("ws_slot_create", h, 2, 9, 1, C.byref(va3))  # pages 0-4 are too short: run 12-20
        kind, nh, ids = _placement(h, 2)
        assert (kind, nh, ids) == (0, 0, list(range(12, 21)))
        base = C.c_void_p()
        N.call("ws_pool_window", h, C.byref(base))
        assert va3.value == base.value + 12 * PAGE and va2.value == base.value + 5 * PAGE
        _check_slot_data(torch, h, n, va3.value, ids)
        host = _owner(h, n, device=False)
        assert np.array_equal(host, _owner(h, n, device=True))
        assert host[5:12].tolist() == [1] * 7 and host[12:21].tolist() == [2] * 9
        init_ms, map_pp, unmap_pp = C.c_double(), C.c_double(), C.c_double()
        N.call("ws_pool_timing", h, C.byref(init_ms), C.byref(map_pp), C.byref(unmap_pp))
        assert map_pp.value == 0.0  # no driver call for windowed slots
        rm, ru = C.c_int64(), C.c_int64()
        N.call("ws_pool_map_stats", h, C.byref(rm), C.byref(ru))
        assert (rm.value, ru.value) == (0, 21)
    finally:
        N.call("ws_pool_destroy", h)


def test_composite_slot_maps_whole_handles(torch_cuda):
    """No contiguous run is long enough: the slot is [free suffix of handle 1]
    + whole free handle 2 + [free prefix of handle 0], each 16-page handle
    mapped whole into the slot's own VA; eviction unmaps asynchronously.
    A placement that needs sub-handle pieces beyond one head and one tail
    fails on a device pool (WS_ERR_FRAGMENTED) and changes nothing."""
    torch = torch_cuda
    from paper_2512_09472_b200 import _native as N

    n = 96
    h = _pool(n)
    try:
        for sid, pages in ((0, 12), (1, 8), (2, 28), (3, 8), (4, 40)):
            N.call("ws_slot_create", h, sid, pages, 1, C.byref(C.c_void_p()))
        N.call("ws_slot_evict", h, 0, None)  # frees 0-11
        N.call("ws_slot_evict", h, 2, None)  # frees 20-47 (longest run: 28)
        va = C.c_void_p()
        N.call("ws_slot_create", h, 5, 36, 0, C.byref(va))
        kind, nh, ids = _placement(h, 5)
        assert kind == 1 and nh == 3
        assert ids == list(range(20, 48)) + list(range(0, 8))
        for first in range(0, 36, 10):  # the pipelined loader's chunked map
            N.call("ws_slot_map_chunk", h, 5, first, min(10, 36 - first))
        _check_slot_data(torch, h, n, va.value, ids)
        assert np.array_equal(_owner(h, n, False), _owner(h, n, True))
        N.call("ws_slot_evict", h, 3, None)  # free: 8-11 (mid-handle) and 48-55 (prefix of handle 3)
        free_before = _owner(h, n, False)
        rc = N.fns["ws_slot_create"](h, 6, 9, 1, C.byref(C.c_void_p()))
        assert rc == N.WS_ERR_FRAGMENTED, rc
        assert np.array_equal(_owner(h, n, False), free_before)
        N.call("ws_slot_evict", h, 5, None)
        N.call("ws_pool_sync_unmaps", h)
        init_ms, map_pp, unmap_pp = C.c_double(), C.c_double(), C.c_double()
        N.call("ws_pool_timing", h, C.byref(init_ms), C.byref(map_pp), C.byref(unmap_pp))
        rm, ru = C.c_int64(), C.c_int64()
        N.call("ws_pool_map_stats", h, C.byref(rm), C.byref(ru))
        print(f"\nVMM: init {init_ms.value:.1f} ms for {n} pages, map {map_pp.value*1e3:.1f} us per slot page "
              f"({rm.value} driver-mapped, {ru.value} windowed), unmap {unmap_pp.value*1e3:.1f} us/page")
        assert rm.value == 48 and unmap_pp.value > 0
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
