"""Peer-HBM weight source.

A universal worker whose slot holds a model exports the physical handles
behind that slot (``ws_pool_export_slot``: POSIX fds of the pool's 128 MiB
handles); a worker in another process imports them (``ws_peer_map_import``)
and passes the mapping to ``UniversalWorker.activate_instance(source=...)``:
the layer streamer then copies layers k..L device-to-device from the peer's
HBM — over NVLink 5 / NVSwitch when the exporter is another GPU, where the
reference's own criterion gives k = 1 (cluster.py:145-166, >= 750 GB/s).

File descriptors cross the process boundary over a Unix domain socket in the
abstract namespace (SCM_RIGHTS; ``socket.send_fds`` / ``recv_fds``); the
slot's byte offset and handle sizes travel in the same message. The exporter
must keep the slot resident (not evicted) while any importer streams from it.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import socket

import torch

from . import _native as N
from .devmem import view


def export_slot(worker, name: str) -> tuple[list[int], list[int], int]:
    """(fds, handle byte sizes, slot offset in the first handle) of ``name``'s slot."""
    slot = worker.slot(name)
    cap = 4096
    fds = (C.c_int32 * cap)()
    sizes = (C.c_int64 * cap)()
    n, off = C.c_int64(), C.c_int64()
    N.call("ws_pool_export_slot", worker.gpu.pool, slot.slot_id, fds, sizes, cap, C.byref(n), C.byref(off))
    return list(fds[: n.value]), list(sizes[: n.value]), off.value


def _addr(tag: str) -> str:
    return "\0warmserve-peer-" + tag


def serve_export(worker, name: str, tag: str, n_clients: int = 1) -> None:
    """Hand ``name``'s slot handles to ``n_clients`` importers (blocking);
    this process's fd copies are closed afterwards."""
    fds, sizes, off = export_slot(worker, name)
    meta = json.dumps({"sizes": sizes, "offset": off, "bytes": worker.models[name].layout.total}).encode()
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(_addr(tag))
    srv.listen(n_clients)
    try:
        for _ in range(n_clients):
            conn, _ = srv.accept()
            with conn:
                conn.sendall(len(meta).to_bytes(4, "little"))
                socket.send_fds(conn, [meta], fds)
                conn.recv(1)  # importer done mapping
    finally:
        srv.close()
        for fd in fds:
            os.close(fd)


class PeerSource:
    """A peer's slot mapped into this process for ``device``: ``tensor`` is a
    uint8 view of the model image (the ``source=`` of activate_instance)."""

    def __init__(self, device: int, tag: str, timeout_s: float = 120.0):
        import time

        cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        t0 = time.monotonic()
        while True:
            try:
                cli.connect(_addr(tag))
                break
            except (ConnectionRefusedError, FileNotFoundError):
                if time.monotonic() - t0 > timeout_s:
                    raise
                time.sleep(0.05)
        with cli:
            n = int.from_bytes(cli.recv(4), "little")
            msg, fds, _, _ = socket.recv_fds(cli, n, 4096)
            meta = json.loads(msg)
            try:
                cfds = (C.c_int32 * len(fds))(*fds)
                sizes = (C.c_int64 * len(fds))(*meta["sizes"])
                va, h = C.c_void_p(), C.c_void_p()
                N.call("ws_peer_map_import", device, cfds, sizes, len(fds), C.byref(va), C.byref(h))
            finally:
                for fd in fds:
                    os.close(fd)
            cli.sendall(b"k")
        self._h = h
        self.device = device
        self.ptr = va.value + meta["offset"]
        self.nbytes = meta["bytes"]
        self.tensor = view(self.ptr, (self.nbytes,), torch.uint8, device)

    def close(self) -> None:
        if self._h:
            torch.cuda.synchronize(self.device)
            N.call("ws_peer_map_release", self._h)
            self._h = None


def can_access_peer(device: int, peer: int) -> bool:
    v = C.c_int32()
    N.call("ws_device_can_access_peer", device, peer, C.byref(v))
    return bool(v.value)
