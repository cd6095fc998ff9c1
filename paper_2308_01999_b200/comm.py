"""PyTorch-free control plane for the one-process-per-GPU layer (multigpu.py):
rendezvous, barriers, byte all-gathers (CUDA IPC handles) and float64
all-reduces over plain TCP sockets.

The data plane never goes through here: amplitudes move GPU to GPU over
NVLink through CUDA IPC mappings (dsv_exchange_masked).  What crosses the
sockets is a few hundred bytes per collective — handles, barrier tokens and
the float64 partial sums of norms, marginals and expectation values — so a
star around rank 0 is enough.  Reductions sum the per-rank values in rank
order on every rank (deterministic, identical on all ranks).

Rendezvous follows torchrun's environment (RANK, WORLD_SIZE, LOCAL_RANK,
MASTER_ADDR); the port is DSV_COMM_PORT, else MASTER_PORT + 1 (torchrun's
own store holds MASTER_PORT).
"""

from __future__ import annotations

import os
import socket
import struct
import time

import numpy as np

__all__ = ["SocketComm"]

_HDR = struct.Struct("<Q")


def _send(sock: socket.socket, payload: bytes) -> None:
    sock.sendall(_HDR.pack(len(payload)) + payload)


def _recv_exact(sock: socket.socket, n: int) -> bytes:
    buf = bytearray()
    while len(buf) < n:
        chunk = sock.recv(n - len(buf))
        if not chunk:
            raise ConnectionError("peer closed the control connection")
        buf += chunk
    return bytes(buf)


def _recv(sock: socket.socket) -> bytes:
    (n,) = _HDR.unpack(_recv_exact(sock, _HDR.size))
    return _recv_exact(sock, n)


class SocketComm:
    """rank / world / local_rank plus the collectives DistributedStateVector
    needs (barrier, all_gather_bytes, allreduce_sum, allreduce_max)."""

    backend = "socket"

    def __init__(self, rank: int | None = None, world: int | None = None, addr: str | None = None,
                 port: int | None = None, timeout: float = 300.0):
        env = os.environ
        self.rank = int(env.get("RANK", "0")) if rank is None else int(rank)
        self.world = int(env.get("WORLD_SIZE", "1")) if world is None else int(world)
        self.local_rank = int(env.get("LOCAL_RANK", str(self.rank)))
        addr = addr or env.get("MASTER_ADDR", "127.0.0.1")
        if port is None:
            port = int(env["DSV_COMM_PORT"]) if "DSV_COMM_PORT" in env else int(env.get("MASTER_PORT", "29500")) + 1
        self._peers: list[socket.socket] = []   # rank 0: one socket per rank 1..world-1
        self._root: socket.socket | None = None  # ranks > 0: the socket to rank 0
        if self.world <= 1:
            return
        if self.rank == 0:
            srv = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
            srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
            srv.bind((addr, port))
            srv.listen(self.world)
            srv.settimeout(timeout)
            peers: dict[int, socket.socket] = {}
            while len(peers) < self.world - 1:
                conn, _ = srv.accept()
                conn.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
                (r,) = struct.unpack("<i", _recv_exact(conn, 4))
                peers[r] = conn
            srv.close()
            self._peers = [peers[r] for r in range(1, self.world)]
        else:
            deadline = time.monotonic() + timeout
            while True:
                try:
                    s = socket.create_connection((addr, port), timeout=timeout)
                    break
                except OSError:
                    if time.monotonic() > deadline:
                        raise
                    time.sleep(0.05)
            s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            s.sendall(struct.pack("<i", self.rank))
            self._root = s

    # -- collectives ---------------------------------------------------------------------
    def all_gather_bytes(self, payload: bytes) -> list[bytes]:
        if self.world <= 1:
            return [bytes(payload)]
        if self.rank == 0:
            parts = [bytes(payload)] + [_recv(s) for s in self._peers]
            blob = b"".join(_HDR.pack(len(p)) + p for p in parts)
            for s in self._peers:
                _send(s, blob)
        else:
            _send(self._root, bytes(payload))
            blob = _recv(self._root)
        out, off = [], 0
        for _ in range(self.world):
            (n,) = _HDR.unpack_from(blob, off)
            off += _HDR.size
            out.append(blob[off:off + n])
            off += n
        return out

    def barrier(self) -> None:
        self.all_gather_bytes(b"")

    def allreduce_sum(self, arr) -> np.ndarray:
        a = np.ascontiguousarray(arr, dtype=np.float64)
        parts = self.all_gather_bytes(a.tobytes())
        total = np.zeros_like(a)
        for p in parts:  # rank order on every rank: deterministic and identical
            total += np.frombuffer(p, dtype=np.float64).reshape(a.shape)
        return total

    def allreduce_max(self, value: float) -> float:
        parts = self.all_gather_bytes(struct.pack("<d", float(value)))
        return max(struct.unpack("<d", p)[0] for p in parts)

    def close(self) -> None:
        for s in self._peers:
            s.close()
        if self._root is not None:
            self._root.close()
        self._peers, self._root = [], None
