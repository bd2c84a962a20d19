"""CPU tests of the host-side logic added in round 2: bench.py's multi-GPU launch, the staging / sharding entry
points' argument checks (no device needed), the oracle's threading (bitwise the single-threaded result), and the
full-shape parity helpers' comparison logic."""
import importlib.util
import os
import sys

import numpy as np
import pytest

import oracle
from paper_2510_14471_b200 import api, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_bench_gpus_n_relaunches_under_torchrun(monkeypatch):
    """--gpus N without a torchrun environment re-executes bench.py as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1; with WORLD_SIZE set it runs in place."""
    bench = load_bench()
    calls = []

    def fake_exec(prog, argv):
        calls.append(argv)
        raise SystemExit(0)

    monkeypatch.setattr(os, "execvp", fake_exec)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit):
        bench.main()
    argv = calls[0]
    assert argv[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "127.0.0.1" in argv
    assert argv[-3:] == ["--gpus", "4", "--steps", "2"][-3:] and os.path.abspath(bench.__file__) in argv
    # inside the launched ranks WORLD_SIZE is set: no second relaunch
    calls.clear()
    monkeypatch.setenv("WORLD_SIZE", "4")
    ran = []
    monkeypatch.setattr(bench, "run_ours", lambda a: ran.append(a.gpus))
    bench.main()
    assert not calls and ran == [4]


def test_bench_reference_arm_rank0_only(monkeypatch, capsys):
    """Under torchrun the reference arm runs on rank 0 only; the other ranks exit without work."""
    bench = load_bench()
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    bench.main()
    assert capsys.readouterr().out == ""


def test_row_partition_covers_rows():
    for M, P in ((1000, 2), (3000, 3), (1_000_000, 8), (100, 3)):
        parts = [api.row_partition(M, P, r) for r in range(P)]
        assert parts[0][0] == 0
        for (a0, m0), (a1, _) in zip(parts, parts[1:]):
            assert a0 + m0 == a1
        assert parts[-1][0] + parts[-1][1] == M


def test_host_pointer_layouts():
    """stage / from_host_sharded accept column-major numpy arrays or (cols, rows) row-major torch / numpy arrays."""
    import torch
    X = np.asfortranarray(np.random.default_rng(0).standard_normal((40, 7)))
    assert api._host_ptr(X, (40, 7)) == X.ctypes.data
    T = torch.from_numpy(np.ascontiguousarray(X.T))
    assert api._host_ptr(T, (40, 7)) == T.data_ptr()
    with pytest.raises(api.DimensionMismatch):
        api._host_ptr(np.ascontiguousarray(X), (40, 7))  # C-ordered (40, 7) is not column-major
    with pytest.raises(api.DimensionMismatch):
        api._host_ptr(X.astype(np.float32), (40, 7))


def test_oracle_threads_bitwise():
    """The OpenMP restatement is bitwise the single-threaded one (independent per-block / per-tile outputs)."""
    p = synth.make_problem(4, M=700, G=12)
    cfg = oracle.make_config(tol_rel=p.tol_rel, max_iter=40)
    n0 = oracle.threads()
    try:
        oracle.set_threads(1)
        a = oracle.solve(p, cfg=cfg, beta_true=p.beta)
        oracle.set_threads(max(2, os.cpu_count() or 2))
        b = oracle.solve(p, cfg=cfg, beta_true=p.beta)
    finally:
        oracle.set_threads(n0)
    assert a.iterations == b.iterations
    assert np.array_equal(a.b, b.b)
    assert np.array_equal(a.trace["c"], b.trace["c"])
    assert np.array_equal(a.trace["aug_residual_norm"], b.trace["aug_residual_norm"])


def test_witness_compare_logic():
    """oracle.witness.compare: the strict bar is same iterations, same termination and b to 1e-10."""
    from oracle import witness

    class Sol:
        def __init__(self, it, term, b):
            self.iterations, self.b = it, b
            self.termination = type("T", (), {"name": term})()

    class G:
        def __init__(self, it, term, b, c):
            self.solution = Sol(it, term, b)
            self.trace = type("Tr", (), {"rows": {"c": np.asarray(c)}})()

    class O:
        def __init__(self, it, term, b, c):
            self.iterations, self.termination, self.b = it, term, b
            self.trace = {"c": np.asarray(c)}

    b = np.arange(1.0, 6.0)
    ok = witness.compare(G(5, "Converged", b * (1 + 1e-12), [3.0, 2.0, 1.0]), O(5, "Converged", b, [3.0, 2.0, 1.0]))
    assert ok["strict"] and ok["rel_b"] < 1e-11
    bad = witness.compare(G(6, "Converged", b, [3.0]), O(5, "Converged", b, [3.0]))
    assert not bad["strict"]
    far = witness.compare(G(5, "Converged", b * (1 + 1e-8), [3.0]), O(5, "Converged", b, [3.0]))
    assert not far["strict"]


def test_no_device_creation_fails_loudly():
    """Without a CUDA device every creation path fails with the no-device status (no CPU fallback)."""
    if api.device_count() > 0:
        pytest.skip("a CUDA device is present")
    p = synth.make_problem(0)
    with pytest.raises(api.GlsError):
        api.sur_preconditioner(api.sur_from_problem(p))
    with pytest.raises(api.GlsError):
        api.GpuSurPreconditioner.from_host_sharded(p.G, p.M, p.M, p.nb, p.X, p.Y, p.omega, b"\0" * 128, 0, 1)
    with pytest.raises(api.GlsError):
        api.LocalGroup(2)
