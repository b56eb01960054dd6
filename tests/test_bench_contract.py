"""bench.py contract checks that run without a GPU.

The reference arm (--impl reference) must not load this repo's package or
native library (the driver records which .so files it maps), and its
hard-coded model shapes must be the ones the GPU arm runs.
"""

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_shapes_match_models():
    import bench
    from paper_2512_09472_b200 import models as M

    for name, shape in bench.REF_SHAPES.items():
        cfg = M.ALL[name]
        for k, v in shape.items():
            assert getattr(cfg, k) == v, (name, k)


def test_reference_arm_never_imports_the_package():
    code = (
        "import sys, torch\n"
        "import bench\n"
        "shape = dict(bench.REF_SHAPES['llama3-8b'], layers=1, hidden=256, ffn=512, heads=4, kv_heads=2,\n"
        "             head_dim=64, vocab=1000)\n"
        "w = bench._ref_cpu_weights(shape)\n"
        "tok = bench._ref_cpu_prefill(shape, w, torch.randint(0, 1000, (64,)))\n"
        "led = bench._ref_ledger_ops(20)\n"
        "assert 0 <= tok < 1000 and led['promote_p50_us'] > 0\n"
        "bad = [m for m in sys.modules if m.startswith('paper_2512_09472_b200')]\n"
        "assert not bad, bad\n"
        "print('ok')\n"
    )
    out = subprocess.run([sys.executable, "-c", code], cwd=str(ROOT), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
