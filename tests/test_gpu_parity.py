"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle.

Tolerances follow the reference's own tests: reduced blocks <= 1e-12
relative Frobenius (proj/tests/test_stage_one.cpp:151), end-to-end solutions
<= 1e-10 relative (test_stage_one.cpp:321, north_star), residual <= 1e-11.
Index maps are bit-exact (tests/test_abi.py).
"""
import numpy as np
import pytest

import oracle as O
import paper_2211_07572_b200 as S

pytestmark = pytest.mark.gpu

KINDS = {0: S.poisson_log_problem, 1: S.helmholtz_problem, 2: S.helmholtz_bump_problem}


def spec_of(kind, n1, n2, kappa):
    return KINDS[kind](n1, n2) if kind == 0 else KINDS[kind](n1, n2, kappa)


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def backward_error(sys_g, u, f):
    """Normwise backward error ||Au - f|| / (||A||_inf ||u|| + ||f||) (2-norms for vectors)."""
    rows = np.repeat(np.arange(sys_g.dim()), np.diff(sys_g.row_ptr))
    a_inf = np.bincount(rows, weights=np.abs(sys_g.values)).max()
    return np.linalg.norm(sys_g.matvec(u) - f) / (a_inf * np.linalg.norm(u) + np.linalg.norm(f))


@pytest.mark.parametrize("kind,n1,n2,b,kappa", [
    (0, 32, 32, 4, 0.0),       # test_stage_one.cpp:138 geometry
    (1, 33, 17, 5, 8.0),
    (2, 64, 40, 7, 60.0),
    (1, 48, 48, 8, 40.0),
])
def test_T_blocks_match_oracle(kind, n1, n2, b, kappa):
    sys_g = S.assemble_fd5(spec_of(kind, n1, n2, kappa))
    sys_o = O.assemble_canned(kind, n1, n2, kappa)
    fg = S.factorize(sys_g, S.SolverConfig(b=b, keep_T=True))
    fo = O.factorize(sys_o, b=b, keep_T=True)
    k = fg.stats.interfaces
    assert k == fo.k
    for j in range(k):
        assert relerr(fg.T_block("diag", j), fo.T_block("diag", j)) < 1e-12
    for j in range(k - 1):
        assert relerr(fg.T_block("super", j), fo.T_block("super", j)) < 1e-12
        assert relerr(fg.T_block("sub", j), fo.T_block("sub", j)) < 1e-12


@pytest.mark.parametrize("n1,n2,b,kappa", [(48, 48, 4, 0.0), (8, 8, 3, 0.0), (9, 8, 4, 0.0), (33, 17, 5, 8.0),
                                           (40, 24, 6, 12.0)])
def test_end_to_end_vs_oracle_and_dense(n1, n2, b, kappa):  # test_stage_one.cpp:296-328
    kind = 1 if kappa > 0 else 0
    sys_g = S.assemble_fd5(spec_of(kind, n1, n2, kappa))
    sys_o = O.assemble_canned(kind, n1, n2, kappa)
    f = np.column_stack([sys_g.rhs, S.gaussian_matrix(sys_g.dim(), 1, 41)[:, 0]])
    u = S.solve(S.factorize(sys_g, S.SolverConfig(b=b)), f)
    u_o = O.factorize(sys_o, b=b).solve(f)
    u_d = np.linalg.solve(sys_o.dense(), f)
    assert relerr(u, u_o) < 1e-10
    assert relerr(u, u_d) < 1e-10
    assert np.linalg.norm(sys_g.matvec(u) - f) / np.linalg.norm(f) < 1e-11


def test_reduce_rhs_matches_oracle():
    sys_g = S.assemble_fd5(S.helmholtz_problem(24, 12, 5.0))
    sys_o = O.assemble_canned(1, 24, 12, 5.0)
    f = np.column_stack([sys_g.rhs, S.gaussian_matrix(sys_g.dim(), 1, 17)[:, 0]])
    rg = S.factorize(sys_g, S.SolverConfig(b=3)).reduce_rhs(f)
    ro = O.factorize(sys_o, b=3).reduce_rhs(f)
    assert relerr(rg, ro) < 1e-12


def test_cfg1_poisson_255_b31_matches_oracle():
    """configs[0]: 255x255 Poisson, b = 31 (the reference CPU oracle config)."""
    sys_g = S.assemble_fd5(S.poisson_log_problem(255, 255))
    sys_o = O.assemble_canned(0, 255, 255)
    fact = S.factorize(sys_g, S.SolverConfig(b=31, keep_T=True))
    assert fact.stats.strips == 8 and fact.stats.interfaces == 7
    fo = O.factorize(sys_o, b=31, threads=8, keep_T=True)
    for j in range(7):
        assert relerr(fact.T_block("diag", j), fo.T_block("diag", j)) < 1e-12
    u = S.solve(fact, sys_g.rhs)
    u_o = fo.solve(sys_o.rhs)
    assert relerr(u, u_o) < 1e-10
    rep = S.error_report(sys_g, u, S.sample_solution(0, 255, 255))
    assert rep.relerr_res < 1e-10
    assert fact.storage_stage2 == fo.storage_stage2


@pytest.mark.parametrize("n", [16, 32, 64])
def test_poisson_golden_relerr_true(known, n):  # test_driver.cpp:235-252
    sys_g = S.assemble_fd5(S.poisson_log_problem(n, n))
    u = S.solve(S.factorize(sys_g, S.SolverConfig(b=4)), sys_g.rhs)
    rep = S.error_report(sys_g, u, S.sample_solution(0, n, n))
    assert rep.relerr_true == pytest.approx(known[f"poisson_relerr_true_slablu_b4_n{n}"][0], rel=1e-4)


def test_acceptance_criterion_1():  # acceptance.cpp:54-83
    worst = 0.0
    for n in (32, 48):
        kappa = S.kappa_from_ppw(15.0, n)
        for kind, k in ((0, 0.0), (1, kappa)):
            sys_g = S.assemble_fd5(spec_of(kind, n, n, k))
            u_star = np.linalg.solve(O.assemble_canned(kind, n, n, k).dense(), sys_g.rhs)
            for b in (3, 4, 8):
                u = S.solve(S.factorize(sys_g, S.SolverConfig(b=b)), sys_g.rhs)[:, 0]
                worst = max(worst, np.abs(u - u_star).max() / np.abs(u_star).max())
    assert worst <= 1e-10


def test_degenerate_whole_grid():  # test_driver.cpp:124-146
    sys_g = S.assemble_fd5(S.poisson_log_problem(16, 8))
    fact = S.factorize(sys_g, S.SolverConfig(b=20))
    assert fact.single_slab()
    u = S.solve(fact, sys_g.rhs)[:, 0]
    u_d = np.linalg.solve(O.assemble_canned(0, 16, 8).dense(), sys_g.rhs)
    assert relerr(u, u_d) < 1e-10


def test_consistent_rhs_and_zero_rhs():  # test_driver.cpp:110-122
    sys_g = S.assemble_fd5(S.helmholtz_problem(48, 32, 9.0))
    fact = S.factorize(sys_g, S.SolverConfig(b=5))
    w = S.gaussian_matrix(sys_g.dim(), 2, 7)
    u = S.solve(fact, sys_g.matvec(w))
    assert relerr(u, w) < 1e-10
    assert np.linalg.norm(S.solve(fact, np.zeros((sys_g.dim(), 3)))) == 0.0


def test_factor_once_solve_many_bitwise():  # test_driver.cpp:148-161
    sys_g = S.assemble_fd5(S.helmholtz_bump_problem(64, 48, 30.0))
    fact = S.factorize(sys_g, S.SolverConfig(b=6))
    f = S.gaussian_matrix(sys_g.dim(), 3, 5)
    u1 = S.solve(fact, f)
    u2 = S.solve(fact, f)
    assert np.array_equal(u1, u2)
    fact2 = S.factorize(sys_g, S.SolverConfig(b=6))
    assert np.array_equal(S.solve(fact2, f), u1)


def test_many_rhs_chunks():
    sys_g = S.assemble_fd5(S.helmholtz_problem(40, 32, 20.0))
    fact = S.factorize(sys_g, S.SolverConfig(b=6))
    f = S.gaussian_matrix(sys_g.dim(), 70, 3)  # > one 64-column sweep chunk
    u = S.solve(fact, f)
    u_o = O.factorize(O.assemble_canned(1, 40, 32, 20.0), b=6).solve(f)
    assert relerr(u, u_o) < 1e-10


def test_singular_slab_reported():  # test_stage_one.cpp:121-136
    sys_g = S.assemble_fd5(S.poisson_log_problem(12, 8))
    part = S.partition(12, 8, 3)
    off, m = part.interior_offset(1), part.interior_size(1)
    v = sys_g.values.copy()
    for r in range(off, off + m):
        for p in range(sys_g.row_ptr[r], sys_g.row_ptr[r + 1]):
            if off <= sys_g.col_idx[p] < off + m:
                v[p] = 0.0
    bad = S.SparseSystem(sys_g.row_ptr, sys_g.col_idx, v, sys_g.rhs, 12, 8, sys_g.h)
    with pytest.raises(S.SingularMatrixError) as e:
        S.factorize(bad, S.SolverConfig(b=3))
    assert e.value.index == 1


def test_nonsymmetric_operator_full_sweep():
    """A nonsymmetric interior takes the full backward sweep (no mirror)."""
    sys_g = S.assemble_fd5(S.helmholtz_problem(30, 20, 7.0))
    v = sys_g.values.copy()
    rng = np.random.default_rng(3)
    v *= 1.0 + 0.05 * rng.standard_normal(v.shape)
    ns = S.SparseSystem(sys_g.row_ptr, sys_g.col_idx, v, sys_g.rhs, 30, 20, sys_g.h)
    fact = S.factorize(ns, S.SolverConfig(b=4, keep_T=True))
    assert fact.stats.symmetric_strips == 0
    so = O.system_from_csr(30, 20, sys_g.h, ns.row_ptr, ns.col_idx, v, ns.rhs)
    fo = O.factorize(so, b=4, keep_T=True)
    for j in range(fact.stats.interfaces):
        assert relerr(fact.T_block("diag", j), fo.T_block("diag", j)) < 1e-12
    u = S.solve(fact, ns.rhs)
    assert relerr(u, fo.solve(ns.rhs)) < 1e-10


def test_cfg2_scale_properties():
    """configs[1] at full size (1000^2, 10 ppw Helmholtz, b=60): size-independent checks."""
    n = 1000
    kappa = S.kappa_from_ppw(10.0, n)
    sys_g = S.assemble_fd5(S.helmholtz_problem(n, n, kappa))
    fact = S.factorize(sys_g, S.SolverConfig(b=60, compression=S.CompressionChoice.dense))
    assert fact.stats.strips == 17 and fact.stats.interfaces == 16
    w = S.gaussian_matrix(sys_g.dim(), 1, 11)
    f = sys_g.matvec(w)
    u = S.solve(fact, f)
    res = np.linalg.norm(sys_g.matvec(u) - f) / np.linalg.norm(f)
    fwd = relerr(u, w)
    eta0 = backward_error(sys_g, u[:, 0], f[:, 0])
    print(f"cfg2: residual {res:.3e}, forward error {fwd:.3e}, backward error {eta0:.3e}")
    assert eta0 < 1e-13                     # backward stable
    assert fwd < 1e-4                       # conditioning-limited at 10 ppw (cond ~1e9)
    u1 = S.solve(fact, sys_g.rhs)[:, 0]
    rep = S.error_report(sys_g, u1, S.sample_solution(1, n, n, kappa))
    eta = backward_error(sys_g, u1, sys_g.rhs)
    print(f"cfg2: relerr_res {rep.relerr_res:.3e}, relerr_true {rep.relerr_true:.3e}, backward error {eta:.3e}")
    # kappa_from_ppw(10, 1000) sits near a discrete resonance (relerr_true ~ 1e5, so
    # ||u|| >> ||u_true||); the normwise backward error is the solver-quality bound.
    assert eta < 1e-13


@pytest.mark.parametrize("n,b", [(120, 12), (200, 20)])
def test_ten_ppw_helmholtz_vs_oracle(n, b):
    """10 ppw (the benchmark's wavelength density) at oracle-feasible sizes."""
    kappa = S.kappa_from_ppw(10.0, n)
    sys_g = S.assemble_fd5(S.helmholtz_bump_problem(n, n, kappa))
    sys_o = O.assemble_canned(2, n, n, kappa)
    fact = S.factorize(sys_g, S.SolverConfig(b=b, keep_T=True))
    fo = O.factorize(sys_o, b=b, threads=8, keep_T=True)
    for j in range(0, fact.stats.interfaces, 3):
        assert relerr(fact.T_block("diag", j), fo.T_block("diag", j)) < 1e-11
    u = S.solve(fact, sys_g.rhs)[:, 0]
    u_o = fo.solve(sys_o.rhs)[:, 0]
    eta_g = backward_error(sys_g, u, sys_g.rhs)
    eta_o = backward_error(sys_g, u_o, sys_g.rhs)
    d = relerr(u, u_o)
    print(f"10ppw n={n}: diff vs oracle {d:.3e}, backward error gpu {eta_g:.3e} oracle {eta_o:.3e}")
    assert eta_g < 1e-14 and eta_g < 10 * eta_o + 1e-16
    assert d < 1e-10


def test_forward_shortcut_matches_full_operator(monkeypatch):
    """Levels without cross-level pivoting use Fbot t = -diag(Lsub) y (schur.cu); the full
    [Ainv ; Fbot] operator must give the same T blocks and solution."""
    n1, n2, b, kappa = 96, 64, 11, 50.0
    sys_g = S.assemble_fd5(S.helmholtz_bump_problem(n1, n2, kappa))
    fa = S.factorize(sys_g, S.SolverConfig(b=b, keep_T=True))
    monkeypatch.setenv("SLB_NO_FSC", "1")
    fb = S.factorize(sys_g, S.SolverConfig(b=b, keep_T=True))
    for j in range(fa.stats.interfaces):
        assert relerr(fa.T_block("diag", j), fb.T_block("diag", j)) < 1e-12
    ua, ub = S.solve(fa, sys_g.rhs), S.solve(fb, sys_g.rhs)
    assert relerr(ua, ub) < 1e-12


def test_backward_columns_match_full_operator(monkeypatch):
    """U13 != 0 levels stream only the x_{l+1} half of H and apply the x_{l+2} half through the
    few columns of the rows pivoted up (Usup diagonal); the explicit H must give the same blocks."""
    n1, n2, b, kappa = 96, 64, 11, 50.0
    sys_g = S.assemble_fd5(S.helmholtz_bump_problem(n1, n2, kappa))
    f = np.column_stack([sys_g.rhs] + [S.gaussian_matrix(sys_g.dim(), 1, 5 + c)[:, 0] for c in range(11)])
    fa = S.factorize(sys_g, S.SolverConfig(b=b, keep_T=True))
    ua = S.solve(fa, f)  # 12 RHS: the 64-column sweep kernel
    monkeypatch.setenv("SLB_NO_BSC", "1")
    fb = S.factorize(sys_g, S.SolverConfig(b=b, keep_T=True))
    ub = S.solve(fb, f)
    for j in range(fa.stats.interfaces):
        assert relerr(fa.T_block("diag", j), fb.T_block("diag", j)) < 1e-12
        if j + 1 < fa.stats.interfaces:
            assert relerr(fa.T_block("super", j), fb.T_block("super", j)) < 1e-12
    assert relerr(ua, ub) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,nrhs", [(1, 1), (37, 3), (64, 1), (100, 8), (333, 2), (1000, 5), (4000, 1), (700, 12), (129, 16), (2000, 64),
                                    (257, 2), (4500, 2)])
def test_stage_two_getrs_vs_numpy(n, nrhs):
    """The stage-two solve applies S_j^{-1} from its LU factors (stage_two.hpp:176-186,
    DenseLU::solve dense.hpp:48-61): chained getrs, 8-column chains (+ a remainder chain).
    Checked against numpy's LAPACK solve of the same matrix (relative 1e-10)."""
    import ctypes
    from paper_2211_07572_b200 import _lib
    L = _lib.lib()
    P = ctypes.POINTER(ctypes.c_double)
    L.slablu_gpu_debug_getrs.restype = ctypes.c_int
    L.slablu_gpu_debug_getrs.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, ctypes.c_int, ctypes.c_int, P]
    rng = np.random.default_rng(n * 31 + nrhs)
    A = np.asfortranarray(rng.standard_normal((n, n)) + 0.0)
    B = np.asfortranarray(rng.standard_normal((n, nrhs)))
    X = np.zeros((n, nrhs), order="F")
    t = np.zeros(1)
    assert L.slablu_gpu_debug_getrs(n, nrhs, A.ctypes.data_as(P), B.ctypes.data_as(P), X.ctypes.data_as(P), 3, 0,
                                    t.ctypes.data_as(P)) == 0
    ref = np.linalg.solve(A, B)
    cond = np.linalg.cond(A)
    assert np.linalg.norm(X - ref) / np.linalg.norm(ref) <= max(1e-10, 1e-14 * cond)
    assert np.linalg.norm(A @ X - B) / (np.linalg.norm(A) * np.linalg.norm(X)) <= 1e-13


@pytest.mark.gpu
@pytest.mark.timeout(120)
def test_stage_two_getrs_nonfinite_rhs_terminates():
    """Blocks of the chained getrs are published as data against a sentinel NaN pattern;
    NaN/Inf right-hand sides must propagate (canonicalised NaN), never stall the chain."""
    import ctypes
    from paper_2211_07572_b200 import _lib
    L = _lib.lib()
    P = ctypes.POINTER(ctypes.c_double)
    L.slablu_gpu_debug_getrs.restype = ctypes.c_int
    L.slablu_gpu_debug_getrs.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, ctypes.c_int, ctypes.c_int, P]
    n, nrhs = 300, 3
    rng = np.random.default_rng(7)
    A = np.asfortranarray(rng.standard_normal((n, n)))
    B = np.asfortranarray(rng.standard_normal((n, nrhs)))
    B[5, 0] = np.nan
    B[7, 1] = np.inf
    B.view(np.uint64)[11, 2] = np.uint64(0xFFFFFFFFFFFFFFFF)  # the sentinel pattern itself
    X = np.zeros((n, nrhs), order="F")
    t = np.zeros(1)
    assert L.slablu_gpu_debug_getrs(n, nrhs, A.ctypes.data_as(P), B.ctypes.data_as(P), X.ctypes.data_as(P), 2, 0,
                                    t.ctypes.data_as(P)) == 0
    assert np.isnan(X).any(axis=0).all()
