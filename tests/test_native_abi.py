"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes as C

from paper_2512_09472_b200 import _native as N


def test_every_declared_symbol_is_exported_and_bound():
    from paper_2512_09472_b200 import models  # noqa: F401  (binds the model entry points)

    declared = N.declared_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(N.lib, name), f"{name} declared in include/ but not exported"
    # every declared function is also bound with argtypes (except ws_last_error)
    missing = [n for n in declared if n not in N.fns and n != "ws_last_error"]
    assert not missing, missing


def test_version_and_error_channel():
    a, b = C.c_int(), C.c_int()
    N.call("ws_version", C.byref(a), C.byref(b))
    assert (a.value, b.value) >= (0, 1)
    rc = N.fns["ws_pool_create"](0, -1, 1, C.byref(C.c_void_p()))
    assert rc == N.WS_ERR_INVALID
    assert "pool needs pages" in N.last_error()


def test_ledger_only_pool_page_identities():
    """Documented identity rules on a ledger-only pool: lowest free pages to a
    new slot, all free pages to KV, highest KV pages returned on shrink."""
    h = C.c_void_p()
    N.call("ws_pool_create", -1, 16, 1, C.byref(h))
    try:
        N.call("ws_slot_create", h, 7, 5, 1, C.byref(C.c_void_p()))
        N.call("ws_slot_create", h, 9, 3, 1, C.byref(C.c_void_p()))
        N.call("ws_slot_evict", h, 7, None)
        kv = C.c_int64()
        N.call("ws_kv_map_all", h, None, C.byref(kv))
        assert kv.value == 13
        N.call("ws_pool_seq_config", h, 2, 8)
        s = C.c_int32()
        N.call("ws_seq_open", h, C.byref(s))
        N.call("ws_seq_reserve", h, s.value, 3, None)
        N.call("ws_kv_resize", h, 4, None)  # keep 4 KV pages: 0,1,2,3 stay
        import numpy as np

        own = np.empty(16, np.int32)
        N.call("ws_pool_owner_map", h, own.ctypes.data_as(C.POINTER(C.c_int32)), 16)
        assert own.tolist() == [-2, -2, -2, -2, -1, 9, 9, 9] + [-1] * 8
        ids = (C.c_int32 * 8)()
        n = C.c_int32()
        N.call("ws_seq_blocks", h, s.value, ids, 8, C.byref(n))
        assert list(ids[: n.value]) == [0, 1, 2]
        # shrinking below the live blocks migrates them; below their count fails
        rc = N.fns["ws_kv_resize"](h, 2, None)
        assert rc == N.WS_ERR_KV_BUSY
    finally:
        N.call("ws_pool_destroy", h)


def test_kv_shrink_migrates_live_blocks():
    import numpy as np

    h = C.c_void_p()
    N.call("ws_pool_create", -1, 10, 1, C.byref(h))
    try:
        kv = C.c_int64()
        N.call("ws_kv_map_all", h, None, C.byref(kv))
        N.call("ws_pool_seq_config", h, 4, 10)
        a, b = C.c_int32(), C.c_int32()
        N.call("ws_seq_open", h, C.byref(a))
        N.call("ws_seq_reserve", h, a.value, 6, None)  # pages 0..5
        N.call("ws_seq_open", h, C.byref(b))
        N.call("ws_seq_reserve", h, b.value, 2, None)  # pages 6, 7
        N.call("ws_seq_close", h, a.value)  # frees 0..5
        N.call("ws_kv_resize", h, 5, None)  # drop pages 9..5: 6,7 live -> 0,1
        ids = (C.c_int32 * 4)()
        n = C.c_int32()
        N.call("ws_seq_blocks", h, b.value, ids, 4, C.byref(n))
        assert list(ids[:2]) == [0, 1]
        own = np.empty(10, np.int32)
        N.call("ws_pool_owner_map", h, own.ctypes.data_as(C.POINTER(C.c_int32)), 10)
        assert own.tolist() == [-2] * 5 + [-1] * 5
    finally:
        N.call("ws_pool_destroy", h)


def test_ledger_only_pool_placement_rules():
    """The slot placement rule (include/warmserve.h) on a ledger-only pool with
    16-page handles: lowest contiguous run; composite head suffix + whole
    handles + tail prefix; scattered lowest free pages where a device pool
    would report WS_ERR_FRAGMENTED; a keyed slot takes its last run back."""
    h = C.c_void_p()
    N.call("ws_pool_create_ex", -1, 96, 1, 16, C.byref(h))

    def place(sid):
        kind, nh = C.c_int32(), C.c_int64()
        N.call("ws_slot_placement", h, sid, C.byref(kind), C.byref(nh))
        ids = (C.c_int32 * 96)()
        cnt = C.c_int64()
        N.call("ws_slot_pages", h, sid, ids, 96, C.byref(cnt))
        return kind.value, nh.value, list(ids)[: cnt.value]

    try:
        for sid, pages in ((0, 12), (1, 8), (2, 28), (3, 8), (4, 40)):
            N.call("ws_slot_create", h, sid, pages, 1, C.byref(C.c_void_p()))
        assert place(2) == (0, 0, list(range(20, 48)))
        N.call("ws_slot_evict", h, 0, None)
        N.call("ws_slot_evict", h, 2, None)
        N.call("ws_slot_create", h, 5, 36, 1, C.byref(C.c_void_p()))
        assert place(5) == (1, 3, list(range(20, 48)) + list(range(8)))
        N.call("ws_slot_evict", h, 3, None)
        N.call("ws_slot_create", h, 6, 9, 1, C.byref(C.c_void_p()))
        assert place(6) == (2, 0, [8, 9, 10, 11, 48, 49, 50, 51, 52])
    finally:
        N.call("ws_pool_destroy", h)
    h = C.c_void_p()
    N.call("ws_pool_create", -1, 64, 1, C.byref(h))
    try:
        N.call("ws_slot_create_keyed", h, 0, 4, 1, 0, C.byref(C.c_void_p()))
        N.call("ws_slot_create_keyed", h, 1, 6, 1, 77, C.byref(C.c_void_p()))  # pages 4-9
        N.call("ws_slot_evict", h, 0, None)
        N.call("ws_slot_evict", h, 1, None)
        N.call("ws_slot_create_keyed", h, 2, 6, 1, 77, C.byref(C.c_void_p()))
        assert place(2)[2] == list(range(4, 10))  # not the lowest run 0-5: its own last run
    finally:
        N.call("ws_pool_destroy", h)
