"""Run the reference's OWN tests with this framework substituted in.

The reference's test_cluster.py (ledger KATs, role machine, 300 lifecycle
walks), test_memswitch.py (pipeline oracle properties), test_engine.py (the
engine driving our Cluster) and test_placement.py execute unmodified from a
/tmp copy, with tests/ref_shim.py swapping in paper_2512_09472_b200.cluster /
.memswitch. Skipped where /root/reference is absent (the GPU box).
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.reference


@pytest.fixture(scope="module")
def ref_tests(tmp_path_factory):
    if not REF.exists():
        pytest.skip("reference not present (GPU box)")
    dst = tmp_path_factory.mktemp("ref") / "tests"
    shutil.copytree(REF / "tests", dst)
    return dst


@pytest.mark.parametrize("module", ["test_cluster.py", "test_memswitch.py", "test_engine.py",
                                    "test_placement.py"])
def test_reference_module_passes_on_our_cluster(ref_tests, module):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests"), str(ROOT), str(REF / "src"), str(ref_tests)])
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-p", "ref_shim", "-p", "no:cacheprovider",
         str(ref_tests / module)],
        cwd=ref_tests, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout


def test_shim_really_substitutes(ref_tests):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests"), str(ROOT), str(REF / "src")])
    code = ("import ref_shim, prewarmsim.engine as e, prewarmsim.cluster as c;"
            "print(e.Cluster.__module__, c.Cluster.__module__, e.pipelined_load.__module__)")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.stdout.split() == ["paper_2512_09472_b200.cluster"] * 2 + ["paper_2512_09472_b200.memswitch"]


def test_measured_latency_engine_adapter(ref_tests):
    """§8f-1: the reference engine replays a desk workload on our Cluster with
    measured latencies; warm scale-ups cost exactly the measured switch."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(REF / "src"), str(ref_tests)])
    code = r'''
import json
import prewarmsim.engine as engine
from conftest import desk_config, desk_model, periodic_trace
from paper_2512_09472_b200 import models as M
from paper_2512_09472_b200.engine_adapter import Measured, run_measured
ma, mb = desk_model("a", initial_instances=1), desk_model("b", initial_instances=1)
cfg = desk_config([ma, mb]); cfg.cluster.gpus_per_server = 8
from prewarmsim.trace import Request
parts = periodic_trace("a", 2, cfg.sim.day_ms, 60_000, (1, 3, 5, 7), 2, ma, slack_ms=700.0) + \
        periodic_trace("b", 2, cfg.sim.day_ms, 60_000, (2, 3, 4), 3, mb, slack_ms=700.0)
reqs = [Request(f"r{i}", r.model_id, r.arrival, r.input_tokens, r.output_tokens)
        for i, r in enumerate(sorted(parts, key=lambda r: r.arrival))]
meas = Measured(prefill_ms=30.5, prompt_tokens=2048, switch_ms=0.124, stream_gb_s=55.5, map_ms_per_page=0.24)
shapes = {"a": M.TINY, "b": M.TINY}
rep = run_measured(engine, cfg, reqs, "warmserve", meas, shapes, reference_model="a")
warm = [x for x in rep.audit if x["kind"] == "scale_up" and x["warm"]]
print(json.dumps({"viol": len(rep.invariant_violations), "n": len(rep.records),
                  "warm_starts": sorted({round(x["breakdown"]["warm_start_ms"], 6) for x in warm})}))
'''
    r = subprocess.run([sys.executable, "-c", code], cwd=ref_tests, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    import json

    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["viol"] == 0 and out["n"] > 100
    assert out["warm_starts"] in ([], [0.124])
