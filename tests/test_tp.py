"""Tensor parallelism (config 4): shard math on CPU with a world_size-2 gloo
group, shard sizing against the reference's partition rule, and (GPU) the
native NCCL TP path at TP=1 against the single-GPU path."""

import os
import socket

import pytest
import torch

from oracle import llama_fp32 as O
from paper_2512_09472_b200 import models as M
from paper_2512_09472_b200 import tp as TP
from paper_2512_09472_b200.weights import synth_flat

TINY_TP = M.TINY.with_(name="tiny-tp", heads=4, kv_heads=2, ffn=1024)  # ffn/2 = 512 = 4 x 128


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_70b_shards_match_reference_partition(tp):
    """A rank's physical shard equals the reference's partition_bytes for a
    spec with weight_bytes = TP x shard (cluster.py:79-80), and the shards of
    the sharded tensors tile the full model."""
    from paper_2512_09472_b200.cluster import ModelSpec

    cfg = M.LLAMA3_70B
    s = TP.shard_config(cfg, tp)
    assert (s.heads, s.kv_heads, s.ffn, s.lm_head_rows) == (64 // tp, 8 // tp, 28672 // tp, 128256 // tp)
    shard = s.layout().total
    spec = ModelSpec(cfg.name, tp * shard, tp, layers=cfg.layers)
    assert spec.partition_bytes == shard
    d, V, L = cfg.hidden, cfg.vocab, cfg.layers
    replicated = V * d * 2 + (2 * L + 1) * d * 2  # embedding + norms on every rank
    per_layer = (cfg.qkv_dim * d + d * cfg.heads * cfg.head_dim + 3 * cfg.ffn * d) * 2
    assert shard == replicated + (L * per_layer + V * d * 2) // tp  # sharded layers + lm_head


def test_shard_flat_equals_synth_shard():
    full = synth_flat(TINY_TP, seed=4, device="cpu")
    for r in range(2):
        a = TP.shard_flat(TINY_TP, full, 2, r)
        b = TP.synth_shard(TINY_TP, 2, r, seed=4, device="cpu")
        assert torch.equal(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tp_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = TINY_TP
        full = synth_flat(cfg, seed=9, device="cpu")
        scfg = TP.shard_config(cfg, world)
        w = O.unpack(scfg, scfg.layout(), TP.shard_flat(cfg, full, world, rank))
        toks = torch.randint(0, cfg.vocab, (48,), generator=torch.Generator().manual_seed(3))

        def allreduce(t):
            dist.all_reduce(t)

        def allgather(t):
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t.contiguous())
            return torch.cat(parts, -1)

        got = O.forward_tp(scfg, w, toks, allreduce, allgather)
        if rank == 0:
            ref, _ = O.forward(cfg, O.unpack(cfg, cfg.layout(), full), toks)
            q.put(((got - ref).abs().max() / ref.abs().max()).item())
    finally:
        dist.destroy_process_group()


def test_tp2_gloo_shards_reproduce_full_model():
    """world_size-2 gloo group: each rank runs its Megatron shard, allreduce
    after O/down, allgather of the vocab-parallel lm_head == full model."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    err = q.get(timeout=10)
    assert err < 1e-4, err


@pytest.mark.gpu
def test_native_tp_path_at_tp1_matches_single_gpu(cuda_device):
    """The NCCL TP path (fp32 partials + allreduce + residual add, lm_head
    allgather + reorder) on a 1-rank communicator == the fused single-GPU path,
    and == the same path with the allreduces on the peer-memory kernel; the
    default bf16-partial NCCL path matches the oracle."""
    from paper_2512_09472_b200.weights import pinned_host_copy
    from paper_2512_09472_b200.worker import UniversalWorker

    cfg = TINY_TP
    host = pinned_host_copy(synth_flat(cfg, seed=2, device="cuda"))
    prompt = torch.randint(0, cfg.vocab, (300,), generator=torch.Generator().manual_seed(1), dtype=torch.int32)
    outs = []
    for use_tp in (False, True, "peer", "bf16"):
        w = UniversalWorker(cuda_device, pool_pages=64, max_tokens=512)
        grp = TP.TpGroup(0, 1, cuda_device, TP.TpGroup.unique_id()) if use_tp else None
        if use_tp == "peer":  # row-parallel allreduces through the peer-memory kernel
            grp.attach_peer(512 * cfg.hidden)
        w.register(cfg, host, tp=grp)
        if use_tp in (True, "peer"):
            w.set_tp_fp32(cfg.name, True)
        w.prewarm(cfg.name, layers=cfg.layers)
        r = w.activate_instance(cfg.name, prompt.pin_memory())
        outs.append((r.token, w.logits[: cfg.vocab].clone()))
        w.release()
        w.close()
        if grp:
            grp.close()
    assert outs[0][0] == outs[1][0] == outs[2][0]
    rel = ((outs[0][1] - outs[1][1]).norm() / outs[0][1].norm()).item()
    assert rel < 1e-3, rel
    assert torch.equal(outs[1][1], outs[2][1])  # one rank: both allreduces are the identity
    ref, _ = O.forward(cfg, O.unpack(cfg, cfg.layout(), host), prompt.long())
    rel_bf16 = ((outs[3][1].double().cpu() - ref[-1].double()).norm() / ref[-1].double().norm()).item()
    assert rel_bf16 < 2e-2 and outs[3][0] == int(ref[-1].argmax()), rel_bf16


def _tp_peer_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_09472_b200.weights import pinned_host_copy
        from paper_2512_09472_b200.worker import UniversalWorker

        torch.cuda.set_device(0)
        cfg = TINY_TP
        scfg = TP.shard_config(cfg, world)
        host = pinned_host_copy(TP.shard_flat(cfg, synth_flat(cfg, seed=6, device="cpu"), world, rank))
        grp = TP.TpGroup.peer_only(0, max(512 * cfg.hidden, cfg.vocab))
        w = UniversalWorker(0, pool_pages=64, max_tokens=512)
        w.register(scfg, host, tp=grp)
        w.prewarm(scfg.name, layers=scfg.layers)
        prompt = torch.randint(0, cfg.vocab, (300,), generator=torch.Generator().manual_seed(5), dtype=torch.int32)
        r = w.activate_instance(scfg.name, prompt.pin_memory())
        first = w.logits[: cfg.vocab].cpu().numpy()  # by value: the process exits before the reader
        w.release()
        # two decode steps on the same shards (row-parallel reduce-adds + lm_head gather per step)
        w.switch_memory(scfg.name)
        sq = w.open_seq(310)
        w.prefill(sq, prompt.cuda())
        tok, steps = r.token, []
        for i in range(2):
            logits, nxt = w.decode(torch.tensor([sq], dtype=torch.int32, device="cuda"),
                                   torch.tensor([300 + i], dtype=torch.int32, device="cuda"),
                                   torch.tensor([tok], dtype=torch.int32, device="cuda"), 301 + i)
            steps.append((tok, logits[0].float().cpu().numpy()))
            tok = int(nxt[0])
        w.close_seq(sq)
        q.put((rank, r.token, first, steps))
        w.release()
        w.close()
        grp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_tp2_peer_collectives_two_processes_match_oracle(cuda_device):
    """Config 4 end to end without NCCL: two ranks (two processes sharing one
    B200) run their Megatron shards of the prefill through the native path,
    the row-parallel partials reduced and the lm_head shards gathered over
    peer memory (CUDA IPC), then two decode steps; both ranks produce the
    same logits, which match the fp32 oracle of the full model."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(2):  # drain the queue before joining (a child exits only once its data is read)
            rank, tok, logits, steps = q.get(timeout=300)
            res[rank] = (tok, torch.from_numpy(logits), [(t, torch.from_numpy(x)) for t, x in steps])
    finally:
        for p in procs:
            p.join(60)
            if p.exitcode is None:
                p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert res[0][0] == res[1][0]
    assert torch.equal(res[0][1], res[1][1])
    cfg = TINY_TP
    weights = O.unpack(cfg, cfg.layout(), synth_flat(cfg, seed=6, device="cpu"))
    prompt = torch.randint(0, cfg.vocab, (300,), generator=torch.Generator().manual_seed(5), dtype=torch.int32)
    ref, past = O.forward(cfg, weights, prompt.long())

    def rel(a, b):
        return ((a.double() - b.double()).norm() / b.double().norm()).item()

    assert rel(res[0][1], ref[-1]) < 2e-2
    assert res[0][0] == int(ref[-1].argmax())
    for i, ((t0, l0), (t1, l1)) in enumerate(zip(res[0][2], res[1][2])):
        assert t0 == t1 and torch.equal(l0, l1)
        ref, past = O.forward(cfg, weights, [t0], pos0=300 + i, past=past)
        assert rel(l0, ref[0]) < 2e-2, (i, rel(l0, ref[0]))
