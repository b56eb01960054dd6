"""Replay golden Cluster-op traces (tests/golden/ledger_traces.json.gz) against
a backend and compare the page ledger after every op.

Backends: ``OracleBackend`` (oracle/ledger.py, CPU restatement) and
``ClusterBackend`` (paper_2512_09472_b200.cluster over native pools, ledger-only
or device-backed).
"""

from __future__ import annotations

from oracle import ledger as OL


class OracleBackend:
    def __init__(self, init):
        servers, per, pages, page, _bw = init
        self.cl = OL.new_cluster(servers, per, pages, page)

    def apply(self, op):
        cl = self.cl
        k = op["op"]
        if k == "begin_prewarm":
            return OL.begin_prewarm(cl, op["gpu"], op["model"], op["pages"], op["required"])["id"]
        if k == "evict_slot":
            s = OL.evict_slot(cl, op["gpu"], op["model"])
            return None if s is None else s["id"]
        if k == "promote":
            iid, ev = OL.promote(cl, op["gpus"], op["model"], op["parallelism"], op["weight"],
                                 op["max_batch"], op["required"])
            return [iid, [list(p) for p in ev]]
        if k == "enter_grace":
            return OL.enter_grace(cl, op["inst"])
        if k == "reclaim":
            return OL.reclaim(cl, op["gpu"], op["inflight"], op["max_batch"], op["used"])
        if k == "release":
            return OL.release(cl, op["inst"], op["inflight"])
        raise KeyError(k)

    def snapshot(self):
        return OL.snapshot(self.cl)

    errors = (OL.OracleError, ValueError)


class _Spec:
    def __init__(self, model_id, weight_bytes, parallelism, max_batch, layers):
        self.model_id = model_id
        self.weight_bytes = weight_bytes
        self.parallelism = parallelism
        self.max_batch = max_batch
        self.layers = layers

    def partition_pages(self, page_size):
        from paper_2512_09472_b200.cluster import _partition

        return _partition(self.weight_bytes, self.parallelism, page_size)[1]


class ClusterBackend:
    def __init__(self, init, devices=None):
        from paper_2512_09472_b200 import cluster as M

        servers, per, pages, page, bw = init
        self.M = M
        self.cl = M.Cluster(servers, per, pages, page, bw, devices=devices)
        self.errors = (M.ClusterError, ValueError)

    def apply(self, op):
        cl, M = self.cl, self.M
        k = op["op"]
        if k == "begin_prewarm":
            spec = _Spec(op["model"], 1, 1, 1, 1)
            return cl.begin_prewarm(cl.gpu(op["gpu"]), spec, op["pages"], op["required"]).slot_id
        if k == "evict_slot":
            s = cl.evict_slot(cl.gpu(op["gpu"]), op["model"])
            return None if s is None else s.slot_id
        if k == "promote":
            spec = _Spec(op["model"], op["weight"], op["parallelism"], op["max_batch"], op["layers"])
            inst, ev = cl.promote_to_dedicated(tuple(op["gpus"]), spec, op["required"])
            return [inst.instance_id, [list(p) for p in ev]]
        if k == "enter_grace":
            return cl.enter_grace(cl.instances[op["inst"]])
        if k == "reclaim":
            return cl.reclaim_on_completion(cl.gpu(op["gpu"]), op["inflight"], op["max_batch"], op["used"])
        if k == "release":
            inst = cl.instances[op["inst"]]
            inst.inflight = {f"r{i}" for i in range(op["inflight"])}
            try:
                return [g.gpu_id for g in cl.release_instance(inst)]
            finally:
                inst.inflight = set()
        raise KeyError(k)

    def snapshot(self):
        out = []
        for g in self.cl.gpus:
            c = g.counts()
            out.append([g.role.value, c.free_pages, c.kv_pages_mapped, c.kv_pages_used,
                        c.kv_capacity_pages, g.instance_id,
                        [[s.model_id, s.slot_id, s.mapped_pages, bool(s.active)] for s in g.slots.values()]])
        return out


def replay(trace, backend, check_roles=True):
    """Apply every op; assert return value, error text and full ledger match."""
    for i, op in enumerate(trace["ops"]):
        where = f"{trace.get('name')} op#{i} {op['op']}"
        want_err = op.get("err")
        try:
            got = backend.apply(op)
        except backend.errors as e:
            assert want_err is not None, f"{where}: unexpected error {e}"
            msg = str(e)
            want = want_err.split("ValueError: ", 1)[-1]
            key = want.split("(")[0].strip()
            assert key.split(":")[-1].strip() in msg or key in msg, f"{where}: error {msg!r} vs {want_err!r}"
        else:
            assert want_err is None, f"{where}: expected error {want_err!r}"
            assert got == op.get("ret"), f"{where}: ret {got!r} != {op.get('ret')!r}"
        assert backend.snapshot() == op["state"], f"{where}: ledger mismatch"
