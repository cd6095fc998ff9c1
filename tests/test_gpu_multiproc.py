"""The real multi-process segment backend (CUDA IPC mappings + the in-place
exchange kernel) with two and four processes.  On a one-GPU box all ranks
share cuda:0 — the IPC/exchange code path is identical to the NVLink case,
only the peer memory is local.  Control plane: the PyTorch-free SocketComm
(comm.py) that multigpu.py uses by default."""

import os
import socket

import multiprocessing as mp

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, dtype_name):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), DSV_COMM_PORT=str(port))
    comm = None
    try:
        from oracle import sv_oracle as O
        from paper_2308_01999_b200 import gates as G
        from paper_2308_01999_b200.circuits import gen_qft, random_gate_sequence, to_gates
        from paper_2308_01999_b200.fusion import FusionConfig, fuse
        from paper_2308_01999_b200.comm import SocketComm
        from paper_2308_01999_b200.multigpu import DistributedStateVector

        dtype = np.dtype(dtype_name)
        comm = SocketComm()
        n = 12
        rng = np.random.default_rng(5)
        gates = fuse(to_gates(gen_qft(n)), FusionConfig(4, 6)).gates
        gates += random_gate_sequence(n, 30, rng, max_arity=3)
        gates.append(G.x(n - 1, controls=((n - 2, 1),)))
        dsv = DistributedStateVector(n, dtype, comm)
        dsv.run(gates)
        probs = dsv.probabilities([n - 1, 0])
        obs = [G.PauliString(((0, "Z"), (n - 2, "X"), (n - 1, "Y")), 0.5)]
        ev = dsv.expectation(obs)
        state = dsv.gather_logical()
        if rank == 0:
            want = O.run_circuit(gates, n, dtype=np.complex128)
            q.put({"state_err": float(np.abs(state - want).max()),
                   "prob_err": float(np.abs(probs - O.marginal(want, n, [n - 1, 0])).max()),
                   "ev_err": abs(ev - O.expectation_pauli(want, n, obs[0].factors, 0.5)),
                   "reorders": dsv.stats.num_reorders})
    except Exception as e:
        q.put({"error": repr(e)})
        raise
    finally:
        if comm is not None:
            comm.close()


@pytest.mark.parametrize("world,dtype", [(2, "complex128"), (4, "complex64")])
def test_ipc_exchange_multiprocess(world, dtype, gpu_available):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, dtype)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert "error" not in res, res
    tol = 1e-12 if dtype == "complex128" else 1e-5
    assert res["state_err"] < tol
    assert res["prob_err"] < tol
    assert res["ev_err"] < tol
    assert res["reorders"] > 0
