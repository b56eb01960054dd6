"""The config-5 decision log (tests/golden/config5_trace.json.gz, recorded by
oracle/gen_config5_trace.py from the reference engine on this framework's
Cluster) is self-consistent, and the live replay's summariser recomposes
TTFT as documented — both without a GPU. The GPU replay itself is
tests/test_gpu_config5.py."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))

from oracle import ledger as OL  # noqa: E402


def test_trace_replays_on_the_ledger_oracle():
    """Every op of every logical GPU, replayed on the reference-pinned ledger
    oracle, yields the ledger the engine recorded (counts, roles, slot order,
    evictions, freed bytes)."""
    from config5_live import load_trace

    t = load_trace()
    page = t["page_size"]
    sizes = {n: m["weight_bytes"] for n, m in t["models"].items()}
    for pol in t["policies"].values():
        cl = OL.new_cluster(1, t["gpus"], t["pages_per_gpu"], page)
        iid = {}
        seqs = [o["seq"] for o in pol["ops"]]
        assert seqs == sorted(seqs)
        for o in pol["ops"]:
            g = o["gpu"]
            if o["op"] == "prewarm":
                OL.begin_prewarm(cl, g, o["model"], o["pages"], o["required"])
            elif o["op"] == "evict":
                OL.evict_slot(cl, g, o["model"])
            elif o["op"] == "promote":
                i, ev = OL.promote(cl, [g], o["model"], 1, sizes[o["model"]], o["max_batch"], o["required"])
                iid[o["instance"]] = i
                assert [list(e) for e in ev] == o["evicted"]
            elif o["op"] == "grace":
                cl["instances"][iid[o["instance"]]]["state"] = OL.ACTIVE
                OL.enter_grace(cl, iid[o["instance"]])
            elif o["op"] == "reclaim":
                assert OL.reclaim(cl, g, o["inflight"], o["max_batch"], o["used"]) == o["freed"]
            elif o["op"] == "release":
                OL.release(cl, iid[o["instance"]])
            gg = cl["gpus"][g]
            got = [gg["role"], OL.free_pages(gg), gg["kv_mapped"], gg["kv_cap"], gg["kv_used"],
                   [s["model"] for s in gg["slots"]]]
            assert got == o["ledger"], (o, got)
        assert not OL.invariants(cl)


def test_live_ttft_recomposition():
    """TTFT = engine queueing + measured prefill (+ the instance's measured
    startup when the request waited for the activation)."""
    from config5_live import load_trace, summarize

    t = load_trace()
    pol = t["policies"]["warmserve"]
    adm = [a for a in pol["admissions"] if a["gpu"] == 0]
    res = [{"gpu": 0, "ledger_checks": 1, "mismatches": [], "activations": [],
            "prefill_ms": {a["request"]: 2.0 for a in adm},
            "startup_ms": {str(a["instance"]): 100.0 for a in adm}, "op_us": {}}]
    out = summarize(t, "warmserve", res)
    want = sorted(a["queue_ms"] + 2.0 + (100.0 if a["activation"] else 0.0) for a in adm)
    assert out["requests"] == len(adm)
    assert abs(out["ttft_ms"]["p50"] - want[(len(want) - 1) // 2]) < 1.0
