"""The simulate CLI (paper_2308_01999_b200/cli.py), mirroring the reference's
tests/test_cli.py TestSimulate cases for the state-vector engines."""

import json

import numpy as np
import pytest

from paper_2308_01999_b200.cli import main


def run_json(capsys, *argv):
    code = main(list(argv))
    out = capsys.readouterr().out
    return code, json.loads(out)


def masked(report):
    report = dict(report)
    report.pop("timings", None)
    return report


def test_qft_33_dry_run(capsys):
    code, rep = run_json(capsys, "simulate", "--circuit", "qft", "--n", "33", "--dry-run")
    assert code == 0
    assert rep["counters"]["gates"] == 577
    assert rep["schema_version"] == 1 and rep["command"] == "simulate"


def test_out_of_scope_engine_is_an_error(capsys):
    assert main(["simulate", "--circuit", "qft", "--n", "4", "--engine", "mps"]) == 2
    err = json.loads(capsys.readouterr().err)
    assert err["error"] == "invalid-argument" and "mps" in err["detail"]


def test_invalid_argument_exit_code_and_json(capsys):
    """The reference prints {"error": "invalid-argument", "detail": ...} and
    exits 2 (cli.py:606-610); --verify limits are checked before any work."""
    assert main(["simulate", "--circuit", "qft", "--n", "30", "--verify"]) == 2
    err = json.loads(capsys.readouterr().err)
    assert err == {"error": "invalid-argument", "detail": "--verify limited to n <= 20"}
    assert main(["simulate", "--circuit", "qft", "--n", "4", "--gpus", "0"]) == 2


def test_workers_default_from_environment(monkeypatch):
    from paper_2308_01999_b200.cli import build_parser

    monkeypatch.setenv("DUETSIM_WORKERS", "3")
    args = build_parser().parse_args(["simulate", "--circuit", "qft", "--n", "4"])
    assert args.workers == 3


@pytest.mark.gpu
class TestSimulateGPU:
    @pytest.fixture(autouse=True)
    def _gpu(self, gpu_available):
        return gpu_available

    def test_qft_20_gate_count_and_norm(self, capsys):
        code, rep = run_json(capsys, "simulate", "--circuit", "qft", "--n", "20", "--engine", "sv")
        assert code == 0
        assert rep["counters"]["gates"] == 20 + 190 + 10
        assert abs(rep["counters"]["norm"] - 1.0) < 1e-10
        assert rep["timings"]["kernels"]  # per-kernel-class device times

    def test_sv_dist_engine_matches_and_reports_transfers(self, capsys):
        code, rep = run_json(capsys, "simulate", "--circuit", "qft", "--n", "8", "--engine", "sv-dist",
                             "--global-bits", "2", "--workers", "2", "--verify")
        assert code == 0
        assert rep["verification"]["passed"]
        assert "transfer_stats" in rep["counters"]

    def test_fusion_flags(self, capsys):
        code, rep = run_json(capsys, "simulate", "--circuit", "qft", "--n", "8", "--engine", "sv",
                             "--max-fused-gate-size", "4", "--max-fused-diagonal-gate-size", "6", "--verify")
        assert code == 0
        assert rep["counters"]["fused_gates"] < rep["counters"]["gates"]
        assert rep["verification"]["passed"]

    def test_fold_fusion_c64_on_the_tensor_path(self, capsys):
        code, rep = run_json(capsys, "simulate", "--circuit", "qft", "--n", "18", "--dtype", "c64",
                             "--fusion", "fold:5", "--verify")
        assert code == 0
        assert rep["verification"]["passed"]
        assert rep["counters"]["data_passes"] == 4
        assert "dense_tc" in rep["timings"]["kernels"]

    def test_qaoa_ring_simulation(self, capsys):
        code, rep = run_json(capsys, "simulate", "--circuit", "qaoa", "--n", "6", "--engine", "sv", "--verify")
        assert code == 0
        assert rep["counters"]["gates"] == 6 + 2 * (6 + 6)
        assert rep["verification"]["passed"]

    def test_deterministic_reports_modulo_timings(self, capsys):
        args = ("simulate", "--circuit", "qv", "--n", "6", "--engine", "sv", "--seed", "5")
        _, rep1 = run_json(capsys, *args)
        _, rep2 = run_json(capsys, *args)
        assert masked(rep1) == masked(rep2)

    def test_streamed_digest_matches_full(self, capsys, monkeypatch):
        """Large states stream the digest and norm chunk by chunk: same values."""
        from paper_2308_01999_b200 import cli
        from paper_2308_01999_b200.statevec import StateVector

        args = ("simulate", "--circuit", "qv", "--n", "12", "--engine", "sv", "--seed", "3", "--dtype", "c64")
        _, full = run_json(capsys, *args)
        monkeypatch.setattr(cli, "STREAM_QUBITS", 4)
        monkeypatch.setattr(StateVector, "DUMP_CHUNK", 1 << 7)
        _, streamed = run_json(capsys, *args)
        assert streamed["digest"] == full["digest"]
        assert abs(streamed["counters"]["norm"] - full["counters"]["norm"]) < 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(5))
def test_reports_match_the_reference_cli(capsys, case, gpu_available):
    """The GPU CLI against the reference CLI's own reports for the same
    arguments (tests/golden/cli.pkl.gz, made by oracle/gen_golden.py):
    counters (gates, fused_gates, transfer_stats), exit code, verification,
    the norm to 1e-12 and — for QFT from |0>, whose rounded amplitudes sit
    far from rounding boundaries — the digest itself."""
    from conftest import golden

    ref = golden("cli")[case]
    code, rep = run_json(capsys, *ref["argv"])
    assert code == ref["code"]
    want = ref["report"]
    for key in ("gates", "fused_gates", "transfer_stats"):
        assert rep["counters"].get(key) == want["counters"].get(key), key
    assert abs(rep["counters"]["norm"] - want["counters"]["norm"]) <= 1e-12
    if "qft" in ref["argv"]:
        assert rep["digest"] == want["digest"]
    if want.get("verification") is not None:
        assert rep["verification"]["passed"] == want["verification"]["passed"]
        assert rep["verification"]["max_error"] <= 1e-10


@pytest.mark.gpu
def test_gpus_flag_shards_and_verifies(capsys, gpu_available):
    code, rep = run_json(capsys, "simulate", "--circuit", "qv", "--n", "12", "--dtype", "c128", "--gpus", "4",
                         "--verify")
    assert code == 0
    assert rep["verification"]["passed"]
    assert rep["params"]["gpus"] == 4
    assert rep["counters"]["transfer_stats"]["num_reorders"] > 0


@pytest.mark.gpu
def test_cluster_fusion_flag(capsys, gpu_available):
    code, rep = run_json(capsys, "simulate", "--circuit", "qv", "--n", "12", "--dtype", "c128", "--fusion", "auto:4",
                         "--verify")
    assert code == 0
    assert rep["verification"]["passed"]
    assert rep["counters"]["data_passes"] < rep["counters"]["gates"]
