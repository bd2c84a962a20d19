"""Formats row: include/gls_b200/io.hpp against the reference's own writers and
readers (proj/src/io.cpp:16-244, driven by tests/cpp/bin/ref_io linked with oracle/_ref): byte-identical
trace CSV and problem directories, round trips both ways, and the binary SUR / MVRGLM files.  CPU only."""
import filecmp
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_2510_14471_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin")


@pytest.fixture(scope="module")
def tools(have_ref):
    if not os.path.exists(os.path.join(BIN, "test_io")) or not os.path.exists(os.path.join(BIN, "ref_io")):
        from paper_2510_14471_b200 import build as B
        B.build()
        B.build_cpp_tests()
    if not os.path.exists(os.path.join(BIN, "ref_io")):
        pytest.skip("ref_io not built (needs the reference headers at build time)")
    return True


def run(name, *args):
    p = subprocess.run([os.path.join(BIN, name), *map(str, args)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr


def same_tree(a, b):
    cmp = filecmp.dircmp(a, b)
    assert not cmp.left_only and not cmp.right_only and not cmp.diff_files, (cmp.left_only, cmp.right_only,
                                                                               cmp.diff_files)
    for sub in cmp.common_dirs:
        same_tree(os.path.join(a, sub), os.path.join(b, sub))


def write_sur_bin(path, p):
    with open(path, "wb") as f:
        f.write(b"GLSSUR1\0")
        np.array([p.G, p.M], dtype=np.int64).tofile(f)
        np.asarray(p.nb, dtype=np.int64).tofile(f)
        for a in (p.X, p.Y, p.omega):
            np.asfortranarray(a, dtype=np.float64).ravel(order="F").tofile(f)


def read_sur_bin(path):
    raw = open(path, "rb").read()
    assert raw[:8] == b"GLSSUR1\0"
    G, M = np.frombuffer(raw, np.int64, 2, 8)
    nb = np.frombuffer(raw, np.int64, G, 24)
    n = int(nb.sum())
    d = np.frombuffer(raw, np.float64, offset=24 + 8 * G)
    X = d[:M * n].reshape(M, n, order="F")
    Y = d[M * n:M * n + M * G].reshape(M, G, order="F")
    om = d[M * n + M * G:].reshape(G, G, order="F")
    return nb, X, Y, om


def write_mv_bin(path, p):
    roff, ridx = p.csr()
    with open(path, "wb") as f:
        f.write(b"GLSMV1\0\0")
        np.array([p.G, p.M0, p.N0, p.k], dtype=np.int64).tofile(f)
        for a in (p.Z0, p.Y, p.omega):
            np.asfortranarray(a, dtype=np.float64).ravel(order="F").tofile(f)
        roff.tofile(f)
        ridx[:p.k].tofile(f)


def test_sur_dir_byte_identical_and_round_trips(tools, tmp_path):
    p = synth.random_sur(3, 17, [2, 4, 3], seed=61)
    p.X[0, 0] = 1e-300
    p.X[1, 1] = -0.0
    p.Y[2, 1] = 123456789.123456789
    src = tmp_path / "in.glssur"
    write_sur_bin(src, p)
    rdir, odir, bdir = tmp_path / "ref", tmp_path / "ours", tmp_path / "bin_back"
    run("ref_io", "save-sur", src, rdir)                 # the reference's writer
    run("test_io", "copy-sur", rdir, odir)               # our reader on its files, then our writer
    same_tree(rdir, odir)                                # ... byte-identical
    run("ref_io", "load-sur", odir, tmp_path / "back.glssur")   # the reference's reader on our files
    nb, X, Y, om = read_sur_bin(tmp_path / "back.glssur")
    assert np.array_equal(nb, p.nb) and np.array_equal(X, p.X) and np.array_equal(Y, p.Y)
    assert np.array_equal(om, p.omega)
    assert np.signbit(X[1, 1]) and X[0, 0] == 1e-300     # -0 and tiny normals survive %.17g (subnormals do not:
                                                          # std::stod rejects them, in the reference as here)
    run("test_io", "bin", rdir, tmp_path / "p.glssur", bdir)    # GLSSUR1 round trip is exact
    same_tree(rdir, bdir)
    assert (tmp_path / "p.glssur").read_bytes() == src.read_bytes()


def test_mvrglm_dir_byte_identical_and_round_trips(tools, tmp_path):
    p = synth.random_mv(4, 20, 5, seed=62)
    src = tmp_path / "in.glsmv"
    write_mv_bin(src, p)
    rdir, odir, bdir = tmp_path / "ref", tmp_path / "ours", tmp_path / "bin_back"
    run("ref_io", "save-mv", src, rdir)
    run("test_io", "copy-mv", rdir, odir)
    same_tree(rdir, odir)
    run("ref_io", "load-mv", odir, tmp_path / "back.glsmv")
    assert (tmp_path / "back.glsmv").read_bytes() == src.read_bytes()
    run("test_io", "bin-mv", rdir, tmp_path / "p.glsmv", bdir)
    same_tree(rdir, bdir)
    assert (tmp_path / "p.glsmv").read_bytes() == src.read_bytes()


def test_trace_csv_byte_identical(tools, tmp_path):
    o = oracle.solve(synth.random_sur(3, 20, [2, 3, 2], seed=63))
    rows = o.trace.copy()
    rows["rmse"][1::2] = np.nan                  # unsampled rows: empty rmse cell
    rows["rmse"][0] = 0.1
    raw = tmp_path / "rows.raw"
    rows.tofile(raw)
    run("ref_io", "trace", raw, tmp_path / "ref.csv")
    run("test_io", "trace", raw, tmp_path / "ours.csv")
    assert (tmp_path / "ref.csv").read_bytes() == (tmp_path / "ours.csv").read_bytes()
    lines = (tmp_path / "ref.csv").read_text().splitlines()
    assert lines[0] == "iter,c_i,aug_residual_norm,dual_feas_norm,rmse,elapsed_ns" and len(lines) == len(rows) + 1
