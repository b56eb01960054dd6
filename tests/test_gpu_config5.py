"""BASELINE config 5 on a real B200: the reference engine's decision log for
the 8-worker periodic trace (tests/golden/config5_trace.json.gz, recorded by
oracle/gen_config5_trace.py from the unmodified prewarmsim engine on this
framework's Cluster) replayed op by op on real UniversalWorkers
(tools/config5_live.py): prewarms copy real layers over PCIe, promotions run
activate_instance (switch + layer stream + prefill + first token), admissions
run real prefills, grace/release switch KV pages back. After every op the
worker's ledger must equal the engine's exactly (role, free / KV-mapped /
KV-capacity / KV-used pages, slots in insertion order, evicted models).
Logical GPU 0 (36 activations) and 4 (a background prewarm) under the
warmserve policy, GPU 1 under no_prewarm (every activation cold, then
evicted)."""

import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))


@pytest.fixture(scope="module")
def live(cuda_device):
    from config5_live import HostImages, load_trace

    trace = load_trace()
    return trace, HostImages(sorted(trace["models"]), cuda_device)


@pytest.mark.parametrize("policy,gpus", [("warmserve", [0, 4]), ("no_prewarm", [1])])
def test_config5_replay_on_real_workers(live, cuda_device, policy, gpus):
    from config5_live import run_live

    trace, images = live
    out = run_live(policy, gpus, cuda_device, trace, images)
    assert out["ledger_mismatches"] == 0, out["first_mismatches"]
    n_ops = sum(1 for o in trace["policies"][policy]["ops"] if o["gpu"] in gpus)
    assert out["ledger_checks"] == n_ops
    assert out["requests"] == sum(1 for a in trace["policies"][policy]["admissions"] if a["gpu"] in gpus)
    acts = out["activations"]
    assert acts["n"] > 0
    if policy == "no_prewarm":
        assert acts["cold"] == acts["n"] and acts["cold_ttft_ms_p50"] > acts["startup_ms_p50"] > 0
    else:
        assert acts["warm"] >= acts["n"] - 1
    assert out["activations"]["switch_us_p99"] < 1000.0
