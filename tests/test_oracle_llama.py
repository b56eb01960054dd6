"""Pin the CPU fp32 logits oracle (oracle/llama_fp32.py) against HF
transformers' LlamaForCausalLM / Qwen2ForCausalLM on the same weights."""

import math

import pytest
import torch

from oracle import llama_fp32 as O
from paper_2512_09472_b200 import models as M


def _hf_llama(cfg, w):
    tr = pytest.importorskip("transformers")
    if cfg.qkv_bias:
        hc = tr.Qwen2Config(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
                            num_hidden_layers=cfg.layers, num_attention_heads=cfg.heads,
                            num_key_value_heads=cfg.kv_heads, rms_norm_eps=cfg.rms_eps,
                            rope_theta=cfg.rope_theta, max_position_embeddings=cfg.max_positions,
                            tie_word_embeddings=False, head_dim=cfg.head_dim)
        model = tr.Qwen2ForCausalLM(hc)
    else:
        hc = tr.LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
                            num_hidden_layers=cfg.layers, num_attention_heads=cfg.heads,
                            num_key_value_heads=cfg.kv_heads, rms_norm_eps=cfg.rms_eps,
                            rope_theta=cfg.rope_theta, max_position_embeddings=cfg.max_positions,
                            tie_word_embeddings=False, head_dim=cfg.head_dim, attention_bias=False,
                            mlp_bias=False)
        model = tr.LlamaForCausalLM(hc)
    model = model.float().eval()
    H, KV, hd = cfg.heads, cfg.kv_heads, cfg.head_dim
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"],
          "lm_head.weight": w["lm_head"]}
    for l in range(cfg.layers):
        p = f"model.layers.{l}."
        qkv = w[f"l{l}.wqkv"]
        sd[p + "self_attn.q_proj.weight"] = qkv[: H * hd]
        sd[p + "self_attn.k_proj.weight"] = qkv[H * hd: (H + KV) * hd]
        sd[p + "self_attn.v_proj.weight"] = qkv[(H + KV) * hd:]
        if cfg.qkv_bias:
            b = w[f"l{l}.bqkv"]
            sd[p + "self_attn.q_proj.bias"] = b[: H * hd]
            sd[p + "self_attn.k_proj.bias"] = b[H * hd: (H + KV) * hd]
            sd[p + "self_attn.v_proj.bias"] = b[(H + KV) * hd:]
        sd[p + "self_attn.o_proj.weight"] = w[f"l{l}.wo"]
        sd[p + "input_layernorm.weight"] = w[f"l{l}.attn_norm"]
        sd[p + "post_attention_layernorm.weight"] = w[f"l{l}.ffn_norm"]
        gate, up = O.split_gate_up(w[f"l{l}.wgu"], cfg.ffn)
        sd[p + "mlp.gate_proj.weight"] = gate
        sd[p + "mlp.up_proj.weight"] = up
        sd[p + "mlp.down_proj.weight"] = w[f"l{l}.wdown"]
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all("rotary" in k for k in missing), missing
    return model


@pytest.mark.parametrize("cfg", [M.TINY, M.TINY.with_(name="tinyq", qkv_bias=True, rope_theta=1e6, rms_eps=1e-6)])
def test_oracle_matches_transformers(cfg):
    from paper_2512_09472_b200.weights import synth_flat

    flat = synth_flat(cfg, seed=3, device="cpu")
    w = O.unpack(cfg, cfg.layout(), flat)
    toks = torch.randint(0, cfg.vocab, (64,), generator=torch.Generator().manual_seed(1))
    ours, _ = O.forward(cfg, w, toks)
    hf = _hf_llama(cfg, w)
    with torch.no_grad():
        ref = hf(toks[None]).logits[0]
    err = (ours - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-4, err


def test_oracle_incremental_decode_matches_full_prefill():
    from paper_2512_09472_b200.weights import synth_flat

    cfg = M.TINY
    w = O.unpack(cfg, cfg.layout(), synth_flat(cfg, seed=5, device="cpu"))
    toks = torch.randint(0, cfg.vocab, (40,), generator=torch.Generator().manual_seed(2))
    full, _ = O.forward(cfg, w, toks)
    _, past = O.forward(cfg, w, toks[:32])
    for i in range(32, 40):
        step, past = O.forward(cfg, w, toks[i:i + 1], pos0=i, past=past)
        assert torch.allclose(step[0], full[i], rtol=1e-4, atol=1e-4)
