"""BASELINE config 3 on a real B200: Llama-3-8B, Qwen2.5-7B, Mistral-7B and
Phi-3-mini co-prewarmed on one worker, a seeded burst of weight<->KV memory
switches (promote -> prefill -> grace -> reclaim -> proactive prewarm ->
release). Every ledger op is replayed on the reference-pinned oracle
(oracle/ledger.py, restating cluster.py:245-387) and the worker's ledger must
match it exactly after each op — role, free / KV-mapped / KV-capacity /
KV-used pages, resident slots, evicted (gpu, model) list, freed bytes — and
the device owner map must equal the host ledger at the end. Switch latency
must stay under the north_star's 1 ms."""

import os
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))


def test_config3_switch_burst_matches_oracle(cuda_device):
    from config3_switch_burst import run_burst

    from oracle import ledger as OL
    from paper_2512_09472_b200 import models as M

    pool_pages = 32768
    ol = OL.new_cluster(1, 1, pool_pages, M.PAGE)
    iid = {}
    checked = {"ops": 0}

    def check(tag, w):
        g = ol["gpus"][0]
        cnt = w.gpu.counts()
        got = (w.gpu.role.value, cnt.free_pages, cnt.kv_pages_mapped, cnt.kv_capacity_pages, cnt.kv_pages_used,
               [s for s in w.gpu.slots])
        want = (g["role"], OL.free_pages(g), g["kv_mapped"], g["kv_cap"], g["kv_used"],
                [s["model"] for s in g["slots"]])
        assert got == want, (tag, got, want)
        checked["ops"] += 1

    def on_op(kind, w, **a):
        if kind == "prewarm":
            OL.begin_prewarm(ol, 0, a["model"], a["pages"], a["required"])
        elif kind == "promote":
            i, evicted = OL.promote(ol, [0], a["model"], 1, a["weight_bytes"], a["max_batch"], a["required"])
            iid["cur"] = i
            assert [tuple(e) for e in a["evicted"]] == [tuple(e) for e in evicted], (a["evicted"], evicted)
        elif kind == "grace":
            OL.enter_grace(ol, iid["cur"])
        elif kind == "reclaim":
            assert a["freed"] == OL.reclaim(ol, 0, a["inflight"], a["max_batch"], a["used"])
        elif kind == "release":
            OL.release(ol, iid["cur"])
        check(kind, w)
        assert not OL.invariants(ol)

    n = int(os.environ.get("WS_CONFIG3_SWITCHES", "300"))
    out = run_burst(switches=n, pool_pages=pool_pages, device=cuda_device, on_op=on_op)
    assert out["device_owner_map_equals_ledger"]
    assert checked["ops"] >= 4 * n
    for kind in ("promote", "reclaim", "release"):
        assert out["switch_us"][kind]["n"] == n
        assert out["switch_us"][kind]["p99"] < 1000.0, (kind, out["switch_us"][kind])
    assert out["slots_evicted_per_promote_mean"] > 0.5  # the burst really evicts co-resident slots
