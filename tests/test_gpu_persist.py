"""Factor caching: save / load of the whole GPU factorization (SLBGPU01) and
stage two in the reference's SweepFactorization layout (SLBSWP01, stage_two.hpp:200-232 with
DenseLU dense.hpp:71-87), read back here by a restatement of the reference's reader."""
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import paper_2211_07572_b200 as S

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_sweep(path):
    """SweepFactorization::deserialize restated: (lu blocks, 0-based pivots, sub, super)."""
    with open(path, "rb") as fh:
        assert fh.read(8) == b"SLBSWP01"
        (k,) = struct.unpack("<Q", fh.read(8))

        def dense():
            r, c = struct.unpack("<QQ", fh.read(16))
            return np.frombuffer(fh.read(8 * r * c), np.float64).reshape(c, r).T

        lus, pivs = [], []
        for _ in range(k):
            a = dense()
            lus.append(a)
            pivs.append(np.frombuffer(fh.read(8 * a.shape[0]), np.int64) - 1)
        sub = [dense() for _ in range(k - 1)]
        sup = [dense() for _ in range(k - 1)]
        assert fh.read(1) == b""
    return lus, pivs, sub, sup


def lu_product(a, piv):
    n = a.shape[0]
    L = np.tril(a, -1) + np.eye(n)
    U = np.triu(a)
    m = L @ U
    for i in range(n - 1, -1, -1):  # undo the row interchanges (LAPACK order)
        m[[i, piv[i]]] = m[[piv[i], i]]
    return m


@pytest.fixture(scope="module")
def problem():
    sysg = S.assemble_fd5(S.helmholtz_bump_problem(96, 64, 50.0))
    fact = S.factorize(sysg, S.SolverConfig(b=11, keep_T=True))
    f = np.column_stack([sysg.rhs, S.gaussian_matrix(sysg.dim(), 2, 9)])
    return sysg, fact, f


def test_save_load_bitwise(problem, tmp_path):
    sysg, fact, f = problem
    u1 = S.solve(fact, f)
    path = tmp_path / "fact.slbgpu"
    fact.save(path)
    g = S.load(path)
    assert (g.n1, g.n2, g.b) == (fact.n1, fact.n2, fact.b)
    assert g.storage_scalars() == fact.storage_scalars()
    assert np.array_equal(S.solve(g, f), u1)
    # another process loads and solves (factor once, solve many across processes)
    np.save(tmp_path / "f.npy", f)
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_2211_07572_b200 as S; "
            "g = S.load(%r); np.save(%r, S.solve(g, np.load(%r)))" %
            (ROOT, str(path), str(tmp_path / "u.npy"), str(tmp_path / "f.npy")))
    subprocess.run([sys.executable, "-c", code], check=True, timeout=300)
    assert np.array_equal(np.load(tmp_path / "u.npy"), u1)


def test_export_sweep_reference_layout(problem, tmp_path):
    sysg, fact, f = problem
    path = tmp_path / "sweep.slbswp"
    fact.export_sweep(path)
    lus, pivs, sub, sup = read_sweep(path)
    k = fact.stats.interfaces
    assert len(lus) == k and len(sub) == k - 1
    for j in range(k - 1):  # couplings are the reduced blocks themselves
        assert np.array_equal(sub[j], fact.T_block("sub", j))
        assert np.array_equal(sup[j], fact.T_block("super", j))
    # S_0 = T_00 and S_1 = T_11 - sub_0 S_0^{-1} super_0 (stage_two.hpp:135-147) from the stored LU
    t00 = fact.T_block("diag", 0)
    assert np.linalg.norm(lu_product(lus[0], pivs[0]) - t00) <= 1e-12 * np.linalg.norm(t00)
    s1 = fact.T_block("diag", 1) - sub[0] @ np.linalg.solve(t00, sup[0])
    assert np.linalg.norm(lu_product(lus[1], pivs[1]) - s1) <= 1e-11 * np.linalg.norm(s1)
    # imported back onto the GPU it solves the reduced system as the original handle does
    sw = S.import_sweep(path)
    red = fact.reduce_rhs(f)
    assert np.array_equal(sw.solve(red), fact.sweep_solve(red))


def test_bad_files_rejected(problem, tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTMAGIC" + b"\0" * 64)
    with pytest.raises(S.Error, match="magic"):
        S.load(bad)
    with pytest.raises(S.Error, match="magic"):
        S.import_sweep(bad)
    _, fact, _ = problem
    good = tmp_path / "fact.slbgpu"
    fact.save(good)
    trunc = tmp_path / "trunc"
    trunc.write_bytes(good.read_bytes()[:4096])
    with pytest.raises(S.Error, match="truncated|expected"):
        S.load(trunc)
