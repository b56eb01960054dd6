"""Prefill attention kernels alone (ws_attn_prefill) against a torch fp32
causal GQA reference on K/V written straight into the paged pool: the
paired-head persistent tcgen05 kernel (attn_tc2, even GQA groups), the
one-head tcgen05 kernel (odd groups: Qwen2.5's 7; head_dim 96 via the
cp.async gather: Phi-3), the legacy mma.sync kernel; full prompts, chunked
prefill (pos0 > 0), ragged tails (one-row last query tile, partial key
tiles). Bar: ||out - ref|| / ||ref|| < 1e-2 (bf16 P and output)."""

import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))

CASES = [
    ("llama3-8b", 2048, 0), ("llama3-8b", 1537, 0), ("llama3-8b", 300, 700), ("llama3-8b", 1, 2047),
    ("llama3-8b", 129, 0), ("qwen2.5-7b", 1000, 37), ("phi3-mini", 517, 0), ("tiny", 512, 0),
    ("llama3-70b-tp8", 640, 128),
]


@pytest.mark.parametrize("shape,rows,pos0", CASES)
@pytest.mark.parametrize("impl", [0, 1])
def test_attention_matches_fp32(cuda_device, shape, rows, pos0, impl):
    import torch
    from attn_bench import AttnRig

    rig = AttnRig(shape, pos0 + rows, seed=rows + pos0)
    try:
        q = torch.randn(rows, rig.H * rig.hd, generator=torch.Generator().manual_seed(3)).bfloat16().cuda()
        out = rig.run(q, rows, pos0, impl)
        torch.cuda.synchronize()
        ref = rig.reference(q, rows, pos0)
        rel = ((out.float().cpu() - ref).norm() / ref.norm()).item()
        assert rel < 1e-2, rel
        # deterministic: a second launch gives the same bits
        out2 = rig.run(q, rows, pos0, impl)
        assert torch.equal(out, out2)
    finally:
        rig.close()
