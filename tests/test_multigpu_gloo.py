"""The one-process-per-GPU layer (paper_2308_01999_b200/multigpu.py) on CPU:
world_size 2 and 4 over gloo (TorchComm) and over the PyTorch-free socket
control plane (comm.SocketComm), with a NumPy segment double standing in for
the libdsv/NVLink segment.  Exercises the real host protocol — relocation
planning, partner roles, global-control predicates, the exchange sequence,
reductions and transfer accounting — and checks the gathered state against
the CPU oracle's single-segment run."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


class NumpySegment:
    """Host stand-in for NvlinkSegment: local ops by explicit index sets,
    exchanges by gloo send/recv of the half segments."""

    def __init__(self, comm, nloc, dtype):
        self.comm, self.nloc, self.dtype = comm, nloc, np.dtype(dtype)
        self.a = np.zeros(1 << nloc, dtype=self.dtype)
        if comm.rank == 0:
            self.a[0] = 1

    def _groups(self, bits, ctrls):
        n = self.nloc
        idx = np.arange(1 << n)
        ok = np.ones(idx.size, bool)
        for b, v in ctrls:
            ok &= ((idx >> b) & 1) == v
        for b in bits:
            ok &= ((idx >> b) & 1) == 0
        base = idx[ok]
        offs = np.array([sum(((j >> m) & 1) << b for m, b in enumerate(bits)) for j in range(1 << len(bits))])
        return base[None, :] + offs[:, None]

    def apply_matrix(self, m, bits, ctrls):
        g = self._groups(bits, ctrls)
        self.a[g] = np.asarray(m, self.dtype) @ self.a[g]

    def apply_genperm(self, perm, diag, bits, ctrls):
        g = self._groups(bits, ctrls)
        out = np.empty_like(self.a[g])
        out[np.asarray(perm)] = np.asarray(diag, self.dtype)[:, None] * self.a[g]
        self.a[g] = out

    def apply_matrix_phased(self, m, bits, cross, outside):
        idx = np.arange(self.a.size)
        ph = np.zeros(self.a.size)
        for mi, b, t in cross:
            ph += t * (((idx >> bits[mi]) & 1) & ((idx >> b) & 1))
        for b, t in outside:
            ph += t * ((idx >> b) & 1)
        self.a *= np.exp(1j * ph).astype(self.dtype)
        self.apply_matrix(m, bits, [])

    def swap_bits(self, pairs):
        idx = np.arange(self.a.size)
        dst = idx.copy()
        for x, y in pairs:
            d = ((idx >> x) ^ (idx >> y)) & 1
            dst ^= d * ((1 << x) | (1 << y))
        out = np.empty_like(self.a)
        out[dst] = self.a
        self.a = out

    def norm2(self):
        return float(np.sum(np.abs(self.a) ** 2))

    def marginal(self, bits):
        idx = np.arange(self.a.size)
        o = np.zeros_like(idx)
        for j, b in enumerate(bits):
            o |= ((idx >> b) & 1) << j
        return np.bincount(o, weights=np.abs(self.a) ** 2, minlength=1 << len(bits))

    def expect_pauli(self, factors):
        b = self.a.copy()
        idx = np.arange(b.size)
        for bit, p in factors:
            if p in "XY":
                b = b[idx ^ (1 << bit)]
                if p == "Y":
                    b = b * np.where((idx >> bit) & 1, 1j, -1j)
            elif p == "Z":
                b = b * np.where((idx >> bit) & 1, -1, 1)
        return complex(np.vdot(self.a, b))

    def download(self):
        return self.a.copy()

    def set_basis(self, index):
        self.a[:] = 0
        if index is not None:
            self.a[index] = 1

    def sync(self):
        pass

    def _sendrecv(self, partner, payload, low):
        if getattr(self.comm, "backend", "") == "socket":  # every rank is in one pair per round
            parts = self.comm.all_gather_bytes(np.ascontiguousarray(payload).tobytes())
            return np.frombuffer(parts[partner], dtype=np.complex128).copy()
        import torch

        out = torch.from_numpy(np.ascontiguousarray(payload).view(np.float64).copy())
        buf = torch.empty_like(out)
        if low:
            dist.send(out, partner)
            dist.recv(buf, partner)
        else:
            dist.recv(buf, partner)
            dist.send(out, partner)
        return buf.numpy().view(self.dtype)

    def exchange_masked(self, partner, lbits, pat_low, pat_high, i_am_low):
        idx = np.arange(self.a.size)
        mask = sum(1 << b for b in lbits)
        mine = idx[(idx & mask) == (pat_low if i_am_low else pat_high)]
        self.a[mine] = self._sendrecv(partner, self.a[mine].astype(np.complex128), i_am_low).astype(self.dtype)

    def exchange_all(self, partner, i_am_low):
        if partner == self.comm.rank:
            if getattr(self.comm, "backend", "") == "socket":
                self.comm.all_gather_bytes(b"")  # stay in step with the pairs that do exchange
            return
        self.a = self._sendrecv(partner, self.a.astype(np.complex128), self.comm.rank < partner).astype(self.dtype)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, kind="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    if kind == "gloo":
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sv_oracle as O
        from paper_2308_01999_b200 import gates as G
        from paper_2308_01999_b200.circuits import gen_qft, random_gate_sequence, to_gates
        from paper_2308_01999_b200.multigpu import DistributedStateVector, TorchComm

        if kind == "gloo":
            comm = TorchComm()
        else:  # the PyTorch-free control plane (comm.py)
            from paper_2308_01999_b200.comm import SocketComm

            comm = SocketComm(rank, world, "127.0.0.1", port)
        n = 7
        rng = np.random.default_rng(11)
        gates = to_gates(gen_qft(n)) + random_gate_sequence(n, 25, rng, max_arity=2)
        gates.append(G.x(6, controls=((5, 1),)))
        gates.append(G.DenseGate(G.random_unitary(4, rng), (6, 0), controls=((5, 0),)))
        dsv = DistributedStateVector(n, np.complex128, comm, segment_factory=NumpySegment)
        dsv.run(gates)
        probs = dsv.probabilities([6, 0, 3])
        obs = [G.PauliString(((0, "Z"), (5, "X"), (6, "Y")), 0.5), G.PauliString(((6, "Z"),))]
        ev = dsv.expectation(obs)
        norm = dsv.norm_squared()
        state = dsv.gather_logical()
        stats = dsv.stats.as_dict()
        # fold-fuser ops (phased windows with global outside qubits, relabel swaps)
        from paper_2308_01999_b200.fusion_fold import fuse_fold

        folded = fuse_fold(to_gates(gen_qft(n)), 3)
        dsv.reset()
        before = dsv.stats.num_reorders
        dsv.run(folded.ops)
        fold_reorders = dsv.stats.num_reorders - before
        fstate = dsv.gather_logical()
        if rank == 0:
            want = O.run_circuit(gates, n)
            fwant = O.run_circuit(to_gates(gen_qft(n)), n)
            # |0> placement: the global bits start on the qubits targeted last -> one reorder
            q.put({"fold_err": float(np.abs(fstate - fwant).max()), "fold_reorders": fold_reorders})
            res = {
                "state_err": float(np.abs(state - want).max()),
                "prob_err": float(np.abs(probs - O.marginal(want, n, [6, 0, 3])).max()),
                "ev_err": abs(ev - sum(O.expectation_pauli(want, n, p.factors, p.coefficient) for p in obs)),
                "norm": norm,
                "reorders": stats["num_reorders"],
            }
            q.put(res)
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put({"error": repr(e)})
        raise
    finally:
        if kind == "gloo":
            dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["gloo", "socket"])
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_protocol_over_gloo(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, kind)) for r in range(world)]
    for p in procs:
        p.start()
    fold = q.get(timeout=240)
    assert "error" not in fold, fold
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert "error" not in res, res
    assert fold["fold_err"] < 1e-12
    assert fold["fold_reorders"] == 1
    assert res["state_err"] < 1e-12
    assert res["prob_err"] < 1e-12
    assert res["ev_err"] < 1e-12
    assert abs(res["norm"] - 1.0) < 1e-12
    assert res["reorders"] > 0
