"""Pin the CPU oracle against the reference's own known-answer tests.

Values come from tests/golden/reference_known_answers.json (extracted from
/root/reference/proj/tests by tests/golden/make_known_answers.py); the
tolerances are the ones the reference tests use (cited per test).
"""
import numpy as np
import pytest

import oracle as O


def test_bessel_table(known):  # proj/tests/test_problem.cpp:203-217
    assert O.bessel_j0(0.0) == 1.0
    assert O.bessel_j0(-3.25) == O.bessel_j0(3.25)
    rows = known["bessel_j0_table"] + known["bessel_j0_table_2"] + known["bessel_j0_table_3"]
    for t, v in zip(rows[0::2], rows[1::2]):
        assert abs(O.bessel_j0(t) - v) <= 1e-13


def test_reference_solutions(known):  # proj/tests/test_problem.cpp:184-201
    assert abs(O.true_solution_poisson(0.9, 0.5)) <= 1e-15
    assert O.true_solution_poisson(-0.1, 1.5) == 0.0
    assert abs(O.true_solution_poisson(0.5, 0.5) - np.log(0.6)) <= 1e-15
    assert O.true_solution_helmholtz(0.3, 0.8, 0.0) == 1.0
    assert abs(O.true_solution_helmholtz(0.9, 0.5, 1.0) - known["helmholtz_true_0p9_0p5_k1"][0]) <= 1e-14
    assert abs(O.true_solution_helmholtz(0.9, 0.5, 2.404825557695773)) <= 1e-13


def test_kappa_from_ppw(known):  # proj/tests/test_problem.cpp:219-229
    assert O.kappa_from_ppw(250.0, 512) == pytest.approx(known["kappa_from_ppw_250_512"][0], rel=1e-6)
    assert O.kappa_from_ppw(10.0, 512) == 2.0 * 3.14159265358979323846 * 513.0 / 10.0
    with pytest.raises(O.ConfigError):
        O.kappa_from_ppw(0.0, 512)
    with pytest.raises(O.ConfigError):
        O.kappa_from_ppw(10.0, 1)


def test_choose_b(known):  # proj/tests/test_driver.cpp:54-78
    cs = {"choose_b_c0p5": 0.5, "choose_b_c0p6": 0.6, "choose_b_c0p54": 0.54,
          "choose_b_clamp_hi": 0.6, "choose_b_clamp_lo": 0.05}
    for key, c in cs.items():
        n1, n2, b = known[key]
        assert O.choose_b(int(n1), int(n2), 0, c) == b
    n1, n2, b = known["choose_b_explicit"]
    assert O.choose_b(int(n1), int(n2), 17, 0.05) == b
    with pytest.raises(O.ConfigError):
        O.choose_b(100, 7, 0, 0.6)
    with pytest.raises(O.ConfigError):
        O.choose_b(100, 64, 0, 0.0)
    with pytest.raises(O.ConfigError):
        O.choose_b(100, 64, 0, 2.5)
    assert O.choose_b(100, 64, 0, 2.0) > 0


def test_partition_geometries(known):  # proj/tests/test_partition.cpp:49-120
    ints, ifcs = O.partition(7, 5, 3)
    assert ints.tolist() == [[0, 3], [4, 3]] and ifcs.tolist() == [[3, 1]]
    ints, ifcs = O.partition(9, 4, 3)
    assert ifcs[:, 0].tolist() == [3, 7] and ints[-1, 1] == 1
    ints, ifcs = O.partition(1000, 1000, 50)
    assert len(ifcs) == known["partition_1000_50_ifc"][0]
    assert len(ints) == known["partition_1000_50_int"][0]
    assert ints[-1, 1] == known["partition_1000_50_lastw"][0]
    ints, ifcs = O.partition(8, 3, 3)
    assert len(ifcs) == 2 and len(ints) == 2 and ifcs[1, 0] == 7
    for bad in [(10, 4, 0), (10, 4, 9), (10, 4, 20), (2, 4, 1), (10, 0, 3)]:
        with pytest.raises(O.ConfigError):
            O.partition(*bad)


def test_hand_built_9x9(known):  # proj/tests/test_problem.cpp:66-94
    d, o = known["hand9x9_diag_off"]
    s = O.assemble(3, 3, 0.25, 0.0, O.COEF_ONE, O.DIR_ZERO, 1.0)
    a = s.dense()
    ref = np.zeros((9, 9))
    for i in range(3):
        for j in range(3):
            r = i * 3 + j
            ref[r, r] = d
            for ii, jj in ((i - 1, j), (i + 1, j), (i, j - 1), (i, j + 1)):
                if 0 <= ii < 3 and 0 <= jj < 3:
                    ref[r, ii * 3 + jj] = o
    assert np.abs(a - ref).max() == 0.0
    assert np.abs(s.rhs - 1.0).max() == 0.0


def test_dirichlet_fold(known):  # proj/tests/test_problem.cpp:96-108
    s = O.assemble(3, 3, 0.25, 0.0, O.COEF_ONE, O.DIR_X_PLUS_Y, 7.0)
    assert s.rhs[0] == known["dirichlet_fold_corner"][0]
    assert s.rhs[4] == known["dirichlet_fold_interior"][0]


def test_variable_coefficient_diagonal():  # proj/tests/test_problem.cpp:110-123
    s = O.assemble(4, 4, 0.2, 2.0, O.COEF_LINEAR_X2Y, O.DIR_ZERO, 0.0)
    a = s.dense()
    x, y = 2.0 * 0.2, 3.0 * 0.2
    assert a[1 * 4 + 2, 1 * 4 + 2] == 4.0 / (0.2 * 0.2) - 4.0 * (x + 2.0 * y)
    assert a[1 * 4 + 2, 2 * 4 + 2] == -1.0 / (0.2 * 0.2)


def test_assembly_rejects_invalid():  # proj/tests/test_problem.cpp:125-140
    with pytest.raises(O.ConfigError):
        O.assemble(4, 1, 0.2)
    with pytest.raises(O.ConfigError):
        O.assemble(4, 6, 0.2)
    with pytest.raises(O.ConfigError):
        O.assemble(4, 4, 0.0)
    with pytest.raises(O.OracleError):
        O.assemble(4, 4, 0.2, 1.0, O.COEF_NEG_ONE)


@pytest.mark.parametrize("n", [16, 32, 64])
def test_poisson_relerr_true_through_slablu(known, n):  # proj/tests/test_driver.cpp:235-252
    s = O.assemble_canned(O.POISSON_LOG, n, n)
    fact = O.factorize(s, b=4)
    u = fact.solve(s.rhs)
    res, err = O.error_report(s, u, O.sample_dirichlet(O.POISSON_LOG, n, n))
    assert err == pytest.approx(known[f"poisson_relerr_true_slablu_b4_n{n}"][0], rel=1e-4)
    assert err == pytest.approx(known[f"poisson_relerr_true_dense_n{n}"][0], rel=1e-5)
    assert res < 1e-12


def _dense_T(s, ints, ifcs, j, k):
    a = s.dense()
    n2 = s.n2
    oj, ok = ifcs[j, 0] * n2, ifcs[k, 0] * n2
    t = a[oj:oj + n2, ok:ok + n2].copy()

    def sub(strip):
        off, m = ints[strip, 0] * n2, ints[strip, 1] * n2
        t[:] -= a[oj:oj + n2, off:off + m] @ np.linalg.solve(a[off:off + m, off:off + m], a[off:off + m, ok:ok + n2])
    if j == k:
        sub(j)
        if j + 1 < len(ints):
            sub(j + 1)
    else:
        sub(max(j, k))
    return t


def test_T_blocks_vs_dense_schur():  # proj/tests/test_stage_one.cpp:138-178
    s = O.assemble_canned(O.POISSON_LOG, 32, 32)
    ints, ifcs = O.partition(32, 32, 4)
    assert len(ifcs) == 6
    fact = O.factorize(s, b=4, keep_T=True)
    for j, k in [(0, 0), (2, 2), (5, 5), (0, 1), (1, 0), (3, 4), (4, 3)]:
        want = _dense_T(s, ints, ifcs, j, k)
        got = fact.T_block("diag", j) if j == k else (fact.T_block("super", j) if k == j + 1 else fact.T_block("sub", k))
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


@pytest.mark.parametrize("n1,n2,b,kappa", [(48, 48, 4, 0.0), (8, 8, 3, 0.0), (9, 8, 4, 0.0), (33, 17, 5, 8.0)])
def test_end_to_end_vs_dense(n1, n2, b, kappa):  # proj/tests/test_stage_one.cpp:296-328
    s = O.assemble_canned(O.HELMHOLTZ if kappa > 0 else O.POISSON_LOG, n1, n2, kappa)
    f = np.column_stack([s.rhs, O.gaussian_matrix(s.dim, 1, 41)[:, 0]])
    u_ref = np.linalg.solve(s.dense(), f)
    u = O.factorize(s, b=b).solve(f)
    assert np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref) < 1e-10
    assert np.linalg.norm(s.matvec(u) - f) / np.linalg.norm(f) < 1e-11


@pytest.mark.parametrize("n", [32, 48])
def test_acceptance_criterion_1(n):  # proj/tests/acceptance.cpp:54-83
    kappa = O.kappa_from_ppw(15.0, n)
    for kind, k in ((O.POISSON_LOG, 0.0), (O.HELMHOLTZ, kappa)):
        s = O.assemble_canned(kind, n, n, k)
        u_star = np.linalg.solve(s.dense(), s.rhs)
        for b in (3, 4, 8):
            u = O.factorize(s, b=b).solve(s.rhs)[:, 0]
            assert np.abs(u - u_star).max() / np.abs(u_star).max() <= 1e-10


def test_storage_and_degenerate():  # proj/tests/test_driver.cpp:80-146
    s = O.assemble_canned(O.POISSON_LOG, 32, 32)
    f = O.factorize(s, b=4)
    assert f.storage_stage2 == (f.k + 2 * (f.k - 1)) * 32 * 32
    s2 = O.assemble_canned(O.POISSON_LOG, 16, 8)
    f2 = O.factorize(s2, b=20)
    assert f2.single_slab
    u = f2.solve(s2.rhs)
    assert np.linalg.norm(u[:, 0] - np.linalg.solve(s2.dense(), s2.rhs)) < 1e-10 * np.linalg.norm(u)


def test_chunked_rhs_and_threads_bitwise():
    s = O.assemble_canned(O.HELMHOLTZ, 40, 24, 9.0)
    a = O.factorize(s, b=5, keep_T=True)
    b = O.factorize(s, b=5, threads=4, chunk=7, keep_T=True)
    for j in range(a.k):
        assert np.array_equal(a.T_block("diag", j), b.T_block("diag", j))
    assert np.array_equal(a.solve(s.rhs), b.solve(s.rhs))


def test_singular_slab_reported_with_index():  # proj/tests/test_stage_one.cpp:121-136
    s = O.assemble_canned(O.POISSON_LOG, 12, 8)
    ints, _ = O.partition(12, 8, 3)
    off, m = ints[1, 0] * 8, ints[1, 1] * 8
    v = s.values.copy()
    for r in range(off, off + m):
        for p in range(s.row_ptr[r], s.row_ptr[r + 1]):
            if off <= s.col_idx[p] < off + m:
                v[p] = 0.0
    s2 = O.system_from_csr(12, 8, s.h, s.row_ptr, s.col_idx, v, s.rhs)
    with pytest.raises(O.SingularMatrixError) as e:
        O.factorize(s2, b=3)
    assert e.value.index == 1


def test_scipy_cross_check_helmholtz_bump():
    """Independent cross-check: oracle vs scipy sparse LU on a bump problem."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    n1, n2 = 60, 40
    kappa = O.kappa_from_ppw(10.0, n2)
    s = O.assemble_canned(O.HELMHOLTZ_BUMP, n1, n2, kappa)
    a = sp.csr_matrix((s.values, s.col_idx, s.row_ptr), shape=(s.dim, s.dim))
    u_ref = spla.spsolve(a.tocsc(), s.rhs)
    u = O.factorize(s, b=7).solve(s.rhs)[:, 0]
    assert np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref) < 1e-10
