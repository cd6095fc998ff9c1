"""One process per GPU: a 2^n state vector sharded over P = 2^g B200s by its
top g index bits (the reference's SegmentedStateVector with one segment per
GPU, distsim.py:69-277, made multi-process).

* Local gates (all targets local) run on every rank with no communication;
  a gate whose global control bits disagree with the rank's bits is skipped
  (distsim.py:232-244).
* A global target is relocated first with the reference's victim rule
  (plan.relocation_pairs; ties toward the highest local bit).  The (global,
  local) pairs of one reorder run together as 2^q - 1 rounds of pairwise
  masked exchanges (plan.exchange_rounds), each ONE in-place pass over
  NVLink: each rank maps its partner's segment through CUDA IPC and both
  ranks swap half of the exchanged amplitudes each, reading and writing both
  HBMs directly (peer loads/stores, no staging buffer — 34q c128 on 2 GPUs
  leaves no room for one).  No NCCL on amplitude data.  The torch-free
  single-process engine (one host thread, all GPUs) is shard.py; this module
  is the torchrun (one process per GPU) form.
* Reductions (norm, marginals, Pauli expectations) reduce per rank on the
  GPU and all-reduce a handful of float64s over the control plane: by
  default the PyTorch-free SocketComm (comm.py, TCP star around rank 0,
  rank-order sums); TorchComm (torch.distributed, NCCL / gloo) plugs in the
  same way.

The segment backend is pluggable so the host protocol (planning, roles,
predicates, reductions) is tested on CPU with world_size=2 gloo and a NumPy
segment double (tests/test_multigpu_gloo.py); on GPUs the backend is libdsv.
"""

from __future__ import annotations

import math
import os
from collections.abc import Sequence

import numpy as np

from .core import InvalidArgumentError, check_swap_pairs
from .gates import Gate, PauliString, PermutationGate
from .plan import (TransferStats, decompose_swap, exchange_rounds, initial_placement, localize_phased, relabel,
                   relocation_pairs, segment_selected, split_controls, swap_transfer)


class TorchComm:
    """torch.distributed plumbing (rendezvous, barriers, tiny all-reduces)."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.backend = dist.get_backend()
        self.local_rank = int(os.environ.get("LOCAL_RANK", self.rank))

    def barrier(self) -> None:
        if self.backend == "nccl":
            self.dist.barrier(device_ids=[self.local_rank])
        else:
            self.dist.barrier()

    def allreduce_sum(self, arr: np.ndarray) -> np.ndarray:
        t = self.torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
        if self.backend == "nccl":
            t = t.to(f"cuda:{self.local_rank}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy()

    def allreduce_max(self, value: float) -> float:
        t = self.torch.tensor([float(value)], dtype=self.torch.float64)
        if self.backend == "nccl":
            t = t.to(f"cuda:{self.local_rank}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.cpu()[0])

    def all_gather_bytes(self, payload: bytes) -> list[bytes]:
        out: list = [None] * self.world
        self.dist.all_gather_object(out, payload)
        return out


class NvlinkSegment:
    """libdsv segment on this rank's GPU + IPC mappings of partner segments."""

    def __init__(self, comm, nloc: int, dtype, device: int):
        from . import _native as N

        self.N = N
        self.comm = comm
        self.device = device
        self.seg = N.NativeState(nloc, dtype, device)
        if comm.rank != 0:
            self.seg.set_zero()
        handles = comm.all_gather_bytes(self.seg.ipc_handle())
        self._handles = handles
        self._peers: dict[int, object] = {}
        self.nloc, self.dtype = nloc, np.dtype(dtype)

    def _peer(self, r: int):
        if r not in self._peers:
            self._peers[r] = self.N.NativeState.open_peer(self.device, self.nloc, self.dtype, self._handles[r])
        return self._peers[r]

    # local ops
    def apply_matrix(self, m, bits, ctrls):
        self.seg.apply_matrix(m, bits, ctrls)

    def apply_genperm(self, perm, diag, bits, ctrls):
        self.seg.apply_genperm(perm, diag, bits, ctrls)

    def apply_matrix_phased(self, m, bits, cross, outside):
        self.seg.apply_matrix_phased(m, bits, cross, outside)

    def swap_bits(self, pairs):
        self.seg.swap_bits(pairs)

    def norm2(self) -> float:
        return self.seg.norm2()

    def marginal(self, bits):
        return self.seg.marginal(bits)

    def expect_pauli(self, factors) -> complex:
        return self.seg.expect_pauli(factors)

    def download(self) -> np.ndarray:
        return self.seg.download()

    def upload(self, arr):
        self.seg.upload(arr)

    def set_basis(self, index: int | None):
        if index is None:
            self.seg.set_zero()
        else:
            self.seg.set_basis(index)

    def sync(self):
        self.seg.sync()

    # exchanges over NVLink (both partners call; each does half)
    def exchange_masked(self, partner: int, lbits, pat_low: int, pat_high: int, i_am_low: bool):
        """One round of a batched (global, local) swap between this rank and
        `partner`: low[off | pat_low] <-> high[off | pat_high], each rank
        running one half of the offsets over the peer mapping."""
        self.seg.sync()
        self.comm.barrier()
        peer = self._peer(partner)
        if i_am_low:
            self.seg.exchange_masked(peer, lbits, pat_low, pat_high, 0, 2)
            self.seg.sync()
        else:
            peer.exchange_masked(self.seg, lbits, pat_low, pat_high, 1, 2)
            peer.sync()
        self.comm.barrier()

    def exchange_all(self, partner: int, i_am_low: bool):
        self.seg.sync()
        self.comm.barrier()
        if i_am_low:
            self.seg.exchange_all(self._peer(partner))
            self.seg.sync()
        self.comm.barrier()


class DistributedStateVector:
    """2^n amplitudes over `world` processes (world = 2^g), one segment each."""

    def __init__(self, num_qubits: int, dtype=np.complex64, comm=None, segment_factory=None):
        if comm is None:
            from .comm import SocketComm

            comm = SocketComm()
        self.comm = comm
        world = self.comm.world
        g = int(round(math.log2(world)))
        if 1 << g != world:
            raise InvalidArgumentError(f"world size {world} is not a power of two")
        if not 0 <= g < num_qubits:
            raise InvalidArgumentError("need fewer global bits than qubits")
        self.num_qubits = num_qubits
        self.global_bits = g
        self.local_bits = num_qubits - g
        self.rank = self.comm.rank
        self.dtype = np.dtype(dtype)
        if segment_factory is None:
            from . import _native as N

            dev = getattr(self.comm, "local_rank", self.rank) % max(1, N.device_count())
            self.seg = NvlinkSegment(self.comm, self.local_bits, self.dtype, dev)
        else:
            self.seg = segment_factory(self.comm, self.local_bits, self.dtype)
        self.qubit_map = list(range(num_qubits))
        self.stats = TransferStats()
        self._basis0 = True  # a fresh segment set is |0...0>

    # -- layout --------------------------------------------------------------------------
    def reset(self) -> None:
        """|0...0> with the identity qubit map."""
        self.seg.set_basis(0 if self.rank == 0 else None)
        self.qubit_map = list(range(self.num_qubits))
        self._basis0 = True

    def _place_for(self, gates) -> None:
        """|0...0> is invariant under any relabelling of index bits: choose
        the qubit map before the first gate (plan.initial_placement)."""
        self.qubit_map = initial_placement(gates, self.num_qubits, self.local_bits)

    def distributed_index_bit_swap(self, pairs: Sequence[tuple[int, int]]) -> None:
        check_swap_pairs(pairs)
        for a, b in pairs:
            if a >= self.num_qubits or b >= self.num_qubits:
                raise InvalidArgumentError(f"bit pair ({a}, {b}) exceeds {self.num_qubits} bits")
        pairs = [(int(a), int(b)) for a, b in pairs]
        dec = decompose_swap(pairs, self.local_bits)
        if dec.local_pairs:
            self.seg.swap_bits(dec.local_pairs)
        # all (global, local) pairs at once: 2^q - 1 rounds, every rank in
        # exactly one pair per round (plan.exchange_rounds)
        for _, s, t, lbits, pat_s, pat_t in exchange_rounds(dec.global_local, self.comm.world):
            if self.rank in (s, t):
                self.seg.exchange_masked(t if self.rank == s else s, lbits, pat_s, pat_t, i_am_low=self.rank == s)
        for j1, j2 in dec.global_global:
            if ((self.rank >> j1) ^ (self.rank >> j2)) & 1:
                partner = self.rank ^ ((1 << j1) | (1 << j2))
                self.seg.exchange_all(partner, i_am_low=self.rank < partner)
            else:
                # keep the collective barrier sequence aligned across ranks
                self.seg.exchange_all(self.rank, i_am_low=False)
        ex, moved, intra, inter = swap_transfer(pairs, self.local_bits, self.global_bits, self.comm.world)
        if ex:
            self.stats.num_reorders += 1
            self.stats.num_messages += 2 * ex
            self.stats.amplitudes_moved += moved
            self.stats.amplitudes_moved_intra_worker += intra
            self.stats.amplitudes_moved_inter_worker += inter
        self.qubit_map = relabel(self.qubit_map, pairs)

    # -- gates -------------------------------------------------------------------------------
    def apply(self, g: Gate, upcoming=()) -> None:
        from .fusion_fold import PhasedDenseGate, QubitSwap

        self._basis0 = False
        if isinstance(g, QubitSwap):  # relabel only: no data moves on any rank
            self.qubit_map[g.a], self.qubit_map[g.b] = self.qubit_map[g.b], self.qubit_map[g.a]
            return
        if len(g.targets) > self.local_bits:
            raise InvalidArgumentError(f"gate arity {len(g.targets)} exceeds local capacity {self.local_bits}")
        pairs = relocation_pairs(self.qubit_map, self.local_bits, [self.qubit_map[q] for q in g.targets], upcoming,
                                 prefer_high=True)
        if pairs:
            self.distributed_index_bit_swap(pairs)
        if isinstance(g, PhasedDenseGate):
            m, tb, cross, outside = localize_phased(g, self.qubit_map, self.local_bits, self.rank, self.dtype)
            self.seg.apply_matrix_phased(m, tb, cross, outside)
            return
        tbits = [self.qubit_map[q] for q in g.targets]
        loc, glob = split_controls(self.qubit_map, self.local_bits, g.controls)
        if not segment_selected(self.rank, glob):
            return
        if isinstance(g, PermutationGate):
            self.seg.apply_genperm(g.permutation, np.asarray(g.diagonal, dtype=self.dtype), tbits, loc)
        else:
            self.seg.apply_matrix(np.asarray(g.matrix, dtype=self.dtype), tbits, loc)

    def run(self, gates) -> None:
        gates = list(gates)
        if getattr(self, "_basis0", False) and self.global_bits > 0:
            self._place_for(gates)
        for i, g in enumerate(gates):
            self.apply(g, gates[i + 1:])

    # -- reductions ------------------------------------------------------------------------------
    def norm_squared(self) -> float:
        return float(self.comm.allreduce_sum(np.array([self.seg.norm2()]))[0])

    def probabilities(self, qubits: Sequence[int]) -> np.ndarray:
        if len(set(qubits)) != len(qubits):
            raise InvalidArgumentError("qubits must be distinct")
        bits = [self.qubit_map[q] for q in qubits]
        loc_pos = [j for j, b in enumerate(bits) if b < self.local_bits]
        local = self.seg.marginal([bits[j] for j in loc_pos]) if loc_pos else np.array([self.seg.norm2()])
        out = np.zeros(1 << len(bits))
        glob_val = 0
        for j, b in enumerate(bits):
            if b >= self.local_bits and (self.rank >> (b - self.local_bits)) & 1:
                glob_val |= 1 << j
        for o_loc, p in enumerate(local):
            o = glob_val
            for t, j in enumerate(loc_pos):
                o |= ((o_loc >> t) & 1) << j
            out[o] += p
        return self.comm.allreduce_sum(out)

    def expectation(self, paulis: Sequence[PauliString]) -> complex:
        total = 0.0 + 0.0j
        for pauli in paulis:
            flip = [self.qubit_map[q] for q, p in pauli.factors if p in "XY"]
            pairs = relocation_pairs(self.qubit_map, self.local_bits, flip, [], prefer_high=True)
            if pairs:
                self.distributed_index_bit_swap(pairs)
            local, sign = [], 1.0
            for q, p in pauli.factors:
                bit = self.qubit_map[q]
                if bit < self.local_bits:
                    local.append((bit, p))
                elif p == "Z" and (self.rank >> (bit - self.local_bits)) & 1:
                    sign = -sign
            v = sign * self.seg.expect_pauli(local)
            red = self.comm.allreduce_sum(np.array([v.real, v.imag]))
            total += pauli.coefficient * complex(red[0], red[1])
        return total

    def gather_logical(self) -> np.ndarray | None:
        """Logical-order state on rank 0 (tests only; O(2^n) host memory)."""
        local = self.seg.download()
        parts = self.comm.all_gather_bytes(local.tobytes())
        if self.rank != 0:
            return None
        phys = np.concatenate([np.frombuffer(p, dtype=self.dtype) for p in parts])
        n = self.num_qubits
        idx = np.arange(1 << n, dtype=np.int64)
        src = np.zeros_like(idx)
        for q, bit in enumerate(self.qubit_map):
            src |= ((idx >> q) & 1) << bit
        return phys[src]


# ---- benchmark leg (bench.py --gpus N under torchrun, DSV_BENCH_MULTIPROC=1) -----------------

def bench_main(args, metric, n_qubits, fusion, published, workload, ClockSampler, peaks, cpu_cores):
    """One process per GPU, PyTorch-free: SocketComm control plane, CUDA IPC
    data plane, device time max over ranks (bench.py contract)."""
    import json
    import time

    from . import _native as N
    from .comm import SocketComm

    comm = SocketComm()
    ndev = max(1, N.device_count())
    local_dev = comm.local_rank % ndev  # > 1 rank per GPU only for functional runs on a 1-GPU box
    gates, ops, fuse_s = workload(getattr(args, "fusion", "fold"))
    dsv = DistributedStateVector(n_qubits, np.complex64, comm)
    seg = dsv.seg.seg

    def step():
        dsv.reset()
        dsv.run(ops)
        dsv.seg.sync()

    for _ in range(args.warmup):
        step()
    comm.barrier()
    seg.prof_reset()
    seg.prof_enable(True)
    clocks = ClockSampler(local_dev).start()
    launches0 = N.launch_count()
    comm.barrier()
    t0 = time.perf_counter()
    seg.event_record(0)
    for _ in range(args.steps):
        step()
    seg.event_record(1)
    comm.barrier()
    wall = time.perf_counter() - t0
    ms_dev = seg.event_elapsed(0, 1)
    # exchanges and barriers sit between device events on different streams:
    # the step time is the wall time between barriers, max over ranks
    ms_total = comm.allreduce_max(max(ms_dev, wall * 1000.0))
    clk = clocks.stop()
    prof = seg.prof_read()
    seg.prof_enable(False)
    launches = N.launch_count() - launches0
    launches_all = int(comm.allreduce_sum(np.array([float(launches)]))[0])
    ms_step = ms_total / args.steps
    value = len(gates) / (ms_step / 1000.0)
    p = dsv.probabilities([0, 1, 2, 3])
    # e2e through the public API, host wall clock, max over ranks: fuse on the
    # host (every rank), reset to |0>, run with P2P swaps, probabilities read-back
    from .fusion_fold import fuse_fold

    e2e = []
    for i in range(3):
        comm.barrier()
        t0 = time.perf_counter()
        ops2 = fuse_fold(gates, 5).ops if getattr(args, "fusion", "fold") == "fold" else ops
        dsv.reset()
        dsv.run(ops2)
        p = dsv.probabilities([0, 1, 2, 3])
        dt = comm.allreduce_max(time.perf_counter() - t0)
        if i > 0:
            e2e.append(dt)
    e2e_s = sorted(e2e)[len(e2e) // 2]
    gate_bytes = sum(int(getattr(g, "matrix", np.zeros(0)).size) * 8 for g in ops)
    if comm.rank == 0:
        pk = peaks()
        dom_name, dom_v = max(((k, v) for k, v in prof.items() if k != "exchange"), key=lambda kv: kv[1]["ms"])
        achieved = dom_v["bytes"] / (dom_v["ms"] / 1000.0) / 1e9
        line = {
            "metric": metric, "value": value, "unit": "gates/s", "n_gpus": comm.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64",
            "data": "synthetic (QFT-33 circuit generated on the host, state starts at |0>)",
            "config": {"workload": "qft33_c64_fused_k5", "n_qubits": n_qubits, "circuit_gates": len(gates),
                       "fused_ops": len(ops), "fusion": getattr(args, "fusion", "fold"),
                       "global_bits": dsv.global_bits, "l2": "segment >= 8 GiB >> 126 MB L2",
                       "parallelism": f"sv-shard{comm.world}: one process per GPU (SocketComm control plane, "
                                      "CUDA IPC masked exchanges over NVLink)"},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": None},
            "transfer_stats": dsv.stats.as_dict(),
            "e2e": {"value": len(gates) / e2e_s, "unit": "gates/s", "seconds_per_step": e2e_s,
                    "h2d_bytes_per_step": gate_bytes, "d2h_bytes_per_step": p.nbytes,
                    "path": "fuse_fold + DistributedStateVector.reset/run + probabilities([0..3]), "
                            "wall clock, max over ranks"},
            "gpu_launches": launches_all,
            "clocks": clk,
            "check_prob_sum": float(p.sum()),
        }
        print(json.dumps(line), flush=True)
    comm.barrier()
    comm.close()
