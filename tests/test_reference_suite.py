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
