"""Parity of the page ledger and planning math with the reference.

The golden vectors were produced by running the unmodified reference
(oracle/gen_golden.py). Three checks, all CPU:
  * oracle (oracle/ledger.py, oracle/memswitch.py) == golden  — pins the oracle;
  * native math (include/warmserve.h ws_* planning) == golden, bit-exact;
  * native-backed Cluster (ledger-only pools) == golden after every op.
"""

import ctypes as C
import math

import pytest

from ledger_replay import ClusterBackend, OracleBackend, replay
from oracle import ledger as OL
from oracle import memswitch as OM


def _traces(traces, name=None):
    return [t for t in traces if name is None or t["name"] == name]


class TestOraclePinnedToReference:
    def test_every_trace_replays_on_oracle(self, ledger_traces):
        assert len(ledger_traces) > 300
        for t in ledger_traces:
            replay(t, OracleBackend(t["init"]))

    def test_required_layers_and_stall(self, plan_math):
        for w, par, L, a, b, bw, tok, k in plan_math["required"]:
            assert OL.required_prewarm_layers(w, par, L, a, b, bw, tok) == k
        for w, par, L, a, b, m, bw, tok, st in plan_math["stall"]:
            assert OL.catchup_stall_ms(w, par, L, a, b, m, bw, tok) == st  # bit-exact

    def test_reservation_and_pages(self, plan_math):
        for m, c, r, k, t in plan_math["reservation"]:
            assert OL.reservation_target(m, c, r, k) == t
        for w, par, page, pb, pp, lb in plan_math["pages"]:
            assert OL.partition_bytes(w, par) == pb
            assert OL.partition_pages(w, par, page) == pp
            assert OL.layer_bytes(w, par, 1) / 1 == pb  # sanity of the split helper

    def test_pipeline_and_kvmap(self, plan_math):
        for total, bw, mu, chunk, page, n, first, finish, stall in plan_math["pipeline"]:
            p = OM.pipelined_load(total, bw, mu, chunk, page)
            assert (p["n_chunks"], p["first_chunk_map_ms"], p["finish_ms"], p["stall_ms"]) == (
                n, first, finish, stall)
        for pages, mu, rate, st in plan_math["kvmap"]:
            assert OM.background_kv_mapping(pages, mu, rate) == st


class TestNativeMath:
    def test_required_layers_bit_exact(self, plan_math):
        from paper_2512_09472_b200 import _native as N

        k = C.c_int32()
        for w, par, L, a, b, bw, tok, want in plan_math["required"]:
            N.call("ws_required_prewarm_layers", w, par, L, a, b, bw, tok, C.byref(k))
            assert k.value == want

    def test_catchup_stall_bit_exact(self, plan_math):
        from paper_2512_09472_b200 import _native as N

        out = C.c_double()
        for w, par, L, a, b, m, bw, tok, want in plan_math["stall"]:
            N.call("ws_catchup_stall_ms", w, par, L, a, b, m, bw, tok, C.byref(out))
            assert out.value == want

    def test_reservation_target_bit_exact(self, plan_math):
        from paper_2512_09472_b200.cluster import reservation_target

        for m, c, r, k, want in plan_math["reservation"]:
            assert reservation_target(m, c, r, k) == want
        with pytest.raises(ValueError):
            reservation_target(100, 32, 33, 0)
        with pytest.raises(ValueError):
            reservation_target(100, 32, 0, 200)

    def test_pipelined_load_bit_exact(self, plan_math):
        from paper_2512_09472_b200.memswitch import background_kv_mapping, pipelined_load

        for total, bw, mu, chunk, page, n, first, finish, stall in plan_math["pipeline"]:
            p = pipelined_load(total, bw, mu, chunk, page)
            assert (p.n_chunks, p.first_chunk_map_ms, p.finish_ms, p.critical_path_stall_ms) == (
                n, first, finish, stall)
        for pages, mu, rate, want in plan_math["kvmap"]:
            assert background_kv_mapping(pages, mu, rate) == want

    def test_partition_pages(self, plan_math):
        from paper_2512_09472_b200.cluster import ModelSpec

        for w, par, page, pb, pp, lb in plan_math["pages"]:
            s = ModelSpec("m", w, par)
            assert (s.partition_bytes, s.partition_pages(page)) == (pb, pp)


class TestNativeLedgerReplay:
    @pytest.mark.parametrize("name", ["kat_ledger", "kat_servers", "config3", "engine_light_warmserve",
                                      "engine_heavy_warmserve", "engine_heavy_sllm_gpu",
                                      "engine_heavy_no_prewarm", "engine_grace"])
    def test_named_traces(self, ledger_traces, name):
        ts = _traces(ledger_traces, name)
        assert ts, name
        for t in ts:
            replay(t, ClusterBackend(t["init"]))

    def test_reference_lifecycle_walks(self, ledger_traces):
        walks = _traces(ledger_traces, "walk")
        assert len(walks) == 300
        for t in walks:
            replay(t, ClusterBackend(t["init"]))

    def test_config3_freed_bytes_match_survey(self, ledger_traces):
        t = _traces(ledger_traces, "config3")[0]
        freed = [op["ret"] for op in t["ops"] if op["op"] == "reclaim"][:4]
        assert freed == [5_419_040_768, 124_644_229_120, 36_861_640_704, 1_073_741_824]
