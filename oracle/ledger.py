"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference page ledger.

Restates, in plain Python, the algorithm of the reference's worker/cluster
state (``/root/reference/pkg/src/prewarmsim/cluster.py``). It is written as a
small state machine over plain dicts so that golden replays
(``tests/golden/*.json.gz``) can compare every counter after every op. Pinned
against outputs of the reference itself (see ``oracle/gen_golden.py``).

Every function cites the reference lines whose behaviour it restates.
"""

from __future__ import annotations

import math

# Role names and the legal edge set: cluster.py:16-30
IDLE, UNIVERSAL, DEDICATED, GRACE_ROLE = "idle", "universal", "dedicated", "dedicated_grace"
LEGAL_EDGES = frozenset(
    {
        (IDLE, UNIVERSAL),
        (UNIVERSAL, DEDICATED),
        (DEDICATED, GRACE_ROLE),
        (GRACE_ROLE, UNIVERSAL),
        (UNIVERSAL, IDLE),
        (IDLE, DEDICATED),
    }
)
# Instance states: cluster.py:33-37
STARTING, ACTIVE, GRACE, TERMINATED = "starting", "active", "grace", "terminated"


class OracleError(RuntimeError):
    """Mirrors ClusterError (cluster.py:40-41); message substrings match."""


# --------------------------------------------------------------------- math


def partition_bytes(weight_bytes: int, parallelism: int) -> int:
    """ceil(weight / parallelism) — cluster.py:79-80."""
    q, r = divmod(weight_bytes, parallelism)
    return q + (1 if r else 0)


def partition_pages(weight_bytes: int, parallelism: int, page_size: int) -> int:
    """ceil(partition / page) — cluster.py:82-83."""
    q, r = divmod(partition_bytes(weight_bytes, parallelism), page_size)
    return q + (1 if r else 0)


def layer_bytes(weight_bytes: int, parallelism: int, layers: int) -> float:
    """Uniform float split of the partition — cluster.py:85-88."""
    return partition_bytes(weight_bytes, parallelism) / layers


def _times(weight_bytes, parallelism, layers, prefill_a, prefill_b, bandwidth, ref_tokens):
    t_load = layer_bytes(weight_bytes, parallelism, layers) / bandwidth
    t_comp = (prefill_a * ref_tokens + prefill_b) / layers
    return t_load, t_comp


def required_prewarm_layers(
    weight_bytes, parallelism, layers, prefill_a, prefill_b, bandwidth, ref_tokens=512
) -> int:
    """Smallest k with (l-k)*t_load <= (l-1)*t_comp for every l in (k, L];
    L when none — cluster.py:145-166. The reference evaluates the products
    in this exact order, which matters for bit-exact float comparison."""
    if bandwidth <= 0:
        raise ValueError("bandwidth must be > 0")
    t_load, t_comp = _times(weight_bytes, parallelism, layers, prefill_a, prefill_b, bandwidth, ref_tokens)
    k = 1
    while k < layers:
        l = k + 1
        while l <= layers and (l - k) * t_load <= (l - 1) * t_comp:
            l += 1
        if l > layers:
            return k
        k += 1
    return layers


def catchup_stall_ms(
    weight_bytes, parallelism, layers, prefill_a, prefill_b, loaded, bandwidth, ref_tokens=512
) -> float:
    """max(0, max_{l>m} (l-m)*t_load - (l-1)*t_comp) — cluster.py:169-182."""
    if loaded >= layers:
        return 0.0
    t_load, t_comp = _times(weight_bytes, parallelism, layers, prefill_a, prefill_b, bandwidth, ref_tokens)
    worst = -math.inf
    for l in range(loaded + 1, layers + 1):
        v = (l - loaded) * t_load - (l - 1) * t_comp
        if v > worst:
            worst = v
    return worst if worst > 0.0 else 0.0


def reservation_target(capacity_bytes, max_batch, inflight, used_bytes) -> float:
    """Eq. 1: max(M*R/C, K + M/C) with range checks — cluster.py:185-197."""
    if inflight < 0 or inflight > max_batch:
        raise ValueError(f"inflight {inflight} outside [0, {max_batch}]")
    if used_bytes < 0 or used_bytes > capacity_bytes:
        raise ValueError(f"kv_used {used_bytes} outside [0, {capacity_bytes}]")
    a = capacity_bytes * inflight / max_batch
    b = used_bytes + capacity_bytes / max_batch
    return a if a >= b else b


# --------------------------------------------------------------------- ledger


def new_cluster(n_servers, gpus_per_server, pages_per_gpu, page_size):
    """Cluster.__init__ — cluster.py:203-230."""
    if n_servers < 1 or gpus_per_server < 1:
        raise ValueError("cluster needs at least one server and one GPU")
    gpus = []
    for gid in range(n_servers * gpus_per_server):
        gpus.append(
            dict(
                id=gid,
                server=gid // gpus_per_server,
                total=pages_per_gpu,
                role=IDLE,
                slots=[],  # ordered list of slot dicts (dict insertion order)
                kv_mapped=0,
                kv_used=0,
                kv_cap=0,
                inst=None,
            )
        )
    return dict(page=page_size, gpus=gpus, instances={}, next_slot=0, next_inst=0, transitions=[])


def slot_pages(g) -> int:
    return sum(s["pages"] for s in g["slots"])  # cluster.py:123-125


def free_pages(g) -> int:
    return g["total"] - slot_pages(g) - g["kv_mapped"]  # cluster.py:127-129


def _find(g, model):
    for s in g["slots"]:
        if s["model"] == model:
            return s
    return None


def _role(cl, g, new):
    """_set_role — cluster.py:235-243."""
    old = g["role"]
    if old == new:
        return
    if (old, new) not in LEGAL_EDGES:
        raise OracleError(f"gpu {g['id']}: {old} -> {new}")
    g["role"] = new
    cl["transitions"].append((g["id"], old, new))


def begin_prewarm(cl, gid, model, pages, required):
    """cluster.py:245-274."""
    g = cl["gpus"][gid]
    if g["role"] == DEDICATED:
        raise OracleError(f"gpu {gid} is dedicated; cannot prewarm")
    if _find(g, model) is not None:
        raise OracleError(f"gpu {gid} already holds a slot for {model}")
    if pages > free_pages(g):
        raise OracleError(f"gpu {gid}: insufficient pages (need {pages}, free {free_pages(g)})")
    slot = dict(id=cl["next_slot"], model=model, pages=pages, required=required, active=False)
    cl["next_slot"] += 1
    g["slots"].append(slot)
    if g["role"] == IDLE:
        _role(cl, g, UNIVERSAL)
    return slot


def evict_slot(cl, gid, model):
    """cluster.py:276-289."""
    g = cl["gpus"][gid]
    slot = _find(g, model)
    if slot is None:
        return None
    if slot["active"]:
        raise OracleError(f"gpu {gid}: cannot evict active slot for {model}")
    g["slots"].remove(slot)
    if g["role"] == UNIVERSAL and not g["slots"]:
        _role(cl, g, IDLE)
    return slot


def promote(cl, gids, model, parallelism, weight_bytes, max_batch, required):
    """promote_to_dedicated — cluster.py:291-342. Returns (inst_id, evicted)."""
    gs = [cl["gpus"][i] for i in gids]
    if len(gids) != parallelism:
        raise OracleError(f"{model} needs {parallelism} GPUs, got {len(gids)}")
    if len({g["server"] for g in gs}) != 1:
        raise OracleError("instance GPUs must reside on one server")
    for g in gs:
        if g["role"] in (DEDICATED, GRACE_ROLE):
            raise OracleError(f"gpu {g['id']} is dedicated to instance {g['inst']}")
        if g["role"] == UNIVERSAL and _find(g, model) is None:
            raise OracleError(f"gpu {g['id']} holds no slot for {model} and is not idle")
    want = partition_pages(weight_bytes, parallelism, cl["page"])
    iid = cl["next_inst"]
    cl["next_inst"] += 1
    evicted = []
    for g in gs:
        for other in [s["model"] for s in g["slots"] if s["model"] != model]:
            evict_slot(cl, g["id"], other)
            evicted.append((g["id"], other))
        slot = _find(g, model)
        if slot is None:
            slot = begin_prewarm(cl, g["id"], model, want, required)
        slot["active"] = True
        g["kv_cap"] = g["total"] - slot["pages"]
        if g["kv_cap"] <= 0:
            raise OracleError(f"gpu {g['id']}: weights leave no pages for KV cache")
        g["kv_mapped"] = g["kv_cap"]
        g["inst"] = iid
        _role(cl, g, DEDICATED)
    cl["instances"][iid] = dict(id=iid, model=model, gpus=tuple(gids), max_batch=max_batch, state=STARTING)
    return iid, evicted


def enter_grace(cl, iid):
    """cluster.py:344-349."""
    inst = cl["instances"][iid]
    if inst["state"] not in (ACTIVE, STARTING):
        raise OracleError(f"instance {iid} not active")
    inst["state"] = GRACE
    for gid in inst["gpus"]:
        _role(cl, cl["gpus"][gid], GRACE_ROLE)


def reclaim(cl, gid, inflight, max_batch, used_bytes) -> int:
    """reclaim_on_completion — cluster.py:351-365: floor-free whole pages
    above the Eq. 1 target; returns freed bytes."""
    g = cl["gpus"][gid]
    if g["role"] != GRACE_ROLE:
        raise OracleError(f"gpu {gid} is not draining")
    page = cl["page"]
    cap_bytes = g["kv_cap"] * page
    used = used_bytes if used_bytes < cap_bytes else cap_bytes
    g["kv_used"] = int(math.ceil(used / page))
    target = reservation_target(cap_bytes, max_batch, inflight, used)
    n = int(math.floor((g["kv_mapped"] * page - target) / page))
    if n < 0:
        n = 0
    g["kv_mapped"] -= n
    return n * page


def release(cl, iid, inflight=0):
    """release_instance — cluster.py:367-387."""
    inst = cl["instances"][iid]
    if inst["state"] != GRACE:
        raise OracleError(f"instance {iid} is not in grace")
    if inflight:
        raise OracleError(f"instance {iid} still has {inflight} inflight")
    for gid in inst["gpus"]:
        g = cl["gpus"][gid]
        g["kv_mapped"] = g["kv_used"] = g["kv_cap"] = 0
        g["inst"] = None
        s = _find(g, inst["model"])
        if s is not None:
            s["active"] = False
        _role(cl, g, UNIVERSAL)
    inst["state"] = TERMINATED
    return list(inst["gpus"])


def invariants(cl) -> list[str]:
    """Page-level subset of check_invariants — cluster.py:389-416."""
    out = []
    for g in cl["gpus"]:
        if slot_pages(g) + g["kv_mapped"] > g["total"]:
            out.append(f"gpu {g['id']}: pages over capacity")
        n_active = sum(1 for s in g["slots"] if s["active"])
        if g["role"] == IDLE and (g["slots"] or g["kv_mapped"]):
            out.append(f"gpu {g['id']}: idle but holds slots or KV")
        if g["role"] in (DEDICATED, GRACE_ROLE):
            if n_active != 1:
                out.append(f"gpu {g['id']}: {g['role']} with {n_active} active slots")
            if g["role"] == DEDICATED and g["kv_mapped"] <= 0:
                out.append(f"gpu {g['id']}: dedicated with no KV mapped")
        elif n_active:
            out.append(f"gpu {g['id']}: {g['role']} with an active slot")
    return out


def snapshot(cl) -> list:
    """Compact per-GPU state used by the golden replays:
    [role, free, kv_mapped, kv_used, kv_cap, inst, [[model, slot_id, pages, active], ...]]."""
    return [
        [
            g["role"],
            free_pages(g),
            g["kv_mapped"],
            g["kv_used"],
            g["kv_cap"],
            g["inst"],
            [[s["model"], s["id"], s["pages"], bool(s["active"])] for s in g["slots"]],
        ]
        for g in cl["gpus"]
    ]
