"""Parity at the benchmark configurations (BASELINE.json configs[1..3]).

The whole oracle factorization is out of reach at these sizes (the reference's
dense mode is ~2e14 flop at cfg3), so parity is staged, following the
reference's own stage-one tests (proj/tests/test_stage_one.cpp:138-178,
208-294) and the verify oracle's staged elimination check
(proj/include/slablu/verify.hpp:402-428): individual slabs are factored by the
oracle (oracle.Slab = factor_one_interior + dgbtrf) and every per-slab term the
GPU engine produces is compared on the same inputs:

  reduce_rhs   f_j - to_R A_jj^-1 f_j - to_L A_(j+1)^-1 f_(j+1)   (stage_one.hpp:415-433)
  T columns    A_jk - sum to_X A_ii^-1 from_Y e_q                  (stage_one.hpp:258-299)
  recover      A_ii^-1 (f_i - from_L u_L - from_R u_R)            (stage_one.hpp:438-462)

cfg2 (1000^2, 10 ppw) is compared with a committed oracle fixture
(tests/golden/make_cfg2_fixture.py); near its discrete resonance the solution
of ANY backward-stable solver differs from the exact one by ~cond*eps, so the
fixture also carries the extended-precision refined solution u* (SURVEY §7
hard part 6) and the GPU is held to the oracle's own distance from u*.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2211_07572_b200 as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.abspath(__file__))


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _csr_block(sys_g, r0, nr, c0, cols):
    """Dense columns `cols` (offsets from c0) of rows r0..r0+nr of the CSR."""
    out = np.zeros((nr, len(cols)))
    pos = {c0 + int(c): k for k, c in enumerate(cols)}
    for r in range(nr):
        for p in range(sys_g.row_ptr[r0 + r], sys_g.row_ptr[r0 + r + 1]):
            k = pos.get(int(sys_g.col_idx[p]))
            if k is not None:
                out[r, k] = sys_g.values[p]
    return out


@pytest.fixture(scope="module")
def cfg3():
    """configs[2] on one GPU: 4000^2 bump Helmholtz, 10 ppw, b = 150 (27 strips, 26 interfaces)."""
    n, b = 4000, 150
    kappa = S.kappa_from_ppw(10.0, n)
    sys_g = S.assemble_fd5(S.helmholtz_bump_problem(n, n, kappa))
    sys_o = O.system_from_csr(n, n, sys_g.h, sys_g.row_ptr, sys_g.col_idx, sys_g.values, sys_g.rhs)
    # refine = 0: the staged chain and the parity below are those of one unrefined solve
    fact = S.factorize(sys_g, S.SolverConfig(b=b, keep_T=True, refine=0, compression=S.CompressionChoice.dense))
    assert fact.stats.strips == 27 and fact.stats.interfaces == 26
    O.set_blas_threads(os.cpu_count() or 1)
    slabs = {}

    def slab(i):
        if i not in slabs:
            slabs[i] = O.Slab(sys_o, b, i)
        return slabs[i]

    f = np.column_stack([sys_g.rhs, S.gaussian_matrix(sys_g.dim(), 1, 2024)[:, 0]])
    return dict(n=n, b=b, sys_g=sys_g, sys_o=sys_o, fact=fact, slab=slab, f=f, part=fact.part)


@pytest.mark.timeout(1800)
def test_cfg3_reduce_rhs_vs_oracle_slabs(cfg3):
    """Reduced right-hand side at interfaces 0, 12, 25 (each from its two slabs), 2 RHS."""
    fact, f, n2 = cfg3["fact"], cfg3["f"], cfg3["n"]
    red = fact.reduce_rhs(f)
    worst = 0.0
    for j in (0, 12, 25):
        off = cfg3["part"].interface_offset(j)
        left, right = cfg3["slab"](j), cfg3["slab"](j + 1)
        assert left.right_ifc == j and right.left_ifc == j
        ref = f[off:off + n2] - left.contrib(f)[1] - right.contrib(f)[0]   # stage_one.hpp:423-432
        e = relerr(red[j * n2:(j + 1) * n2], ref)
        print(f"cfg3 reduce_rhs interface {j}: rel diff {e:.3e}")
        worst = max(worst, e)
    # measured 0.9e-12 .. 1.3e-11 across kernel versions (the reference's own 1e-12 bar is set on
    # 32^2 grids, test_stage_one.cpp:151; here the slab solves run over 4000 levels of a 10-ppw
    # Helmholtz operator, and the rounding order of the band LU differs from dgbtrf's)
    assert worst < 5e-11


@pytest.mark.timeout(1800)
def test_cfg3_T_columns_vs_oracle_slabs(cfg3):
    """16 sampled columns of diag[0], diag[25], super[12], sub[12] (reference block order
    stage_one.hpp:400-409: T_jj = A_jj - strip j (R,R) - strip j+1 (L,L); T_{j,j+1} from strip j+1
    (to_left, from_right); T_{j+1,j} from strip j+1 (to_right, from_left))."""
    fact, sys_g, n2 = cfg3["fact"], cfg3["sys_g"], cfg3["n"]
    part = cfg3["part"]
    cols = np.unique(np.concatenate([[0, 1, n2 // 2, n2 - 2, n2 - 1], np.linspace(3, n2 - 4, 11).astype(int)]))
    worst = 0.0
    for j in (0, 25):
        off = part.interface_offset(j)
        direct = _csr_block(sys_g, off, n2, off, cols)
        ref = direct - cfg3["slab"](j).T_columns("right", cols)[1] - cfg3["slab"](j + 1).T_columns("left", cols)[0]
        e = relerr(fact.T_block("diag", j)[:, cols], ref)
        print(f"cfg3 diag[{j}] sampled columns: rel diff {e:.3e}")
        worst = max(worst, e)
    j = 12
    s13 = cfg3["slab"](13)
    sup_ref = _csr_block(sys_g, part.interface_offset(j), n2, part.interface_offset(j + 1), cols) - \
        s13.T_columns("right", cols)[0]
    sub_ref = _csr_block(sys_g, part.interface_offset(j + 1), n2, part.interface_offset(j), cols) - \
        s13.T_columns("left", cols)[1]
    for which, ref in (("super", sup_ref), ("sub", sub_ref)):
        e = relerr(fact.T_block(which, j)[:, cols], ref)
        print(f"cfg3 {which}[{j}] sampled columns: rel diff {e:.3e}")
        worst = max(worst, e)
    assert worst < 1e-11  # measured 1.1e-12 .. 2.4e-12


@pytest.mark.timeout(1800)
def test_cfg3_recover_and_solution_vs_oracle_slabs(cfg3):
    """Solution on strips 0, 13, 26 = the oracle's recover_interiors from the GPU's interface
    values (1e-10, north_star), plus the staged ABI (reduce -> sweep_solve -> recover) equal to
    the fused solve.  Unrefined solve (refine = 0): relerr_res ~2e-9 (explicit level inverses);
    one refinement step brings it to ~2e-13 (checked in test_cfg3_refined_residual)."""
    fact, f, sys_g, n2 = cfg3["fact"], cfg3["f"], cfg3["sys_g"], cfg3["n"]
    part = cfg3["part"]
    u = S.solve(fact, f)
    res = np.linalg.norm(sys_g.matvec(u) - f, axis=0) / np.linalg.norm(f, axis=0)
    print(f"cfg3 relerr_res (unrefined) {res}")
    assert res.max() < 1e-8
    k = fact.stats.interfaces
    u_ifc = np.vstack([u[part.interface_offset(j):part.interface_offset(j) + n2] for j in range(k)])
    worst = 0.0
    for i in (0, 13, 26):
        sl = cfg3["slab"](i)
        ref = sl.recover(f, u_ifc)
        off = part.interior_offset(i)
        e = relerr(u[off:off + sl.width * n2], ref)
        print(f"cfg3 strip {i} (w={sl.width}): rel diff vs oracle recover {e:.3e}")
        worst = max(worst, e)
    assert worst < 1e-10
    # staged entry points chain to the same answer as the solve
    f1 = f[:, :1]
    us = fact.recover(f1, fact.sweep_solve(fact.reduce_rhs(f1)))
    assert relerr(us, u[:, :1]) < 1e-13


@pytest.mark.timeout(900)
def test_cfg3_refined_residual(cfg3):
    """SolverConfig.refine = 1 (the default): one step of iterative refinement against the CSR."""
    sys_g, f = cfg3["sys_g"], cfg3["f"]
    cfg3["fact"].close()  # one 80 GB factorization at a time
    fact = S.factorize(sys_g, S.SolverConfig(b=cfg3["b"], refine=1, compression=S.CompressionChoice.dense))
    u = S.solve(fact, f)
    res = np.linalg.norm(sys_g.matvec(u) - f, axis=0) / np.linalg.norm(f, axis=0)
    print(f"cfg3 relerr_res (refine=1) {res}")
    assert res.max() < 1e-10


def test_cfg2_vs_oracle_fixture():
    """configs[1] (1000^2 Helmholtz, 10 ppw, b=60, dense) against the committed oracle solution.

    kappa_from_ppw(10, 1000) sits next to a discrete resonance: the oracle's own solution is
    cond*eps away from the exact discrete solution u* (extended-precision refinement in the
    fixture).  The GPU solution must be as close to u* as the oracle's, and within the
    conditioning bound of the oracle's solution."""
    z = np.load(os.path.join(ROOT, "golden", "cfg2_oracle_fixture.npz"))
    n = int(z["n"])
    kappa = S.kappa_from_ppw(10.0, n)
    assert kappa == float(z["kappa"])
    sys_g = S.assemble_fd5(S.helmholtz_problem(n, n, kappa))
    assert int(sys_g.values.size) == int(z["nnz"])
    for refine in (0, 1):
        fact = S.factorize(sys_g, S.SolverConfig(b=60, compression=S.CompressionChoice.dense, refine=refine))
        u = S.solve(fact, sys_g.rhs)[:, 0]
        idx = z["idx"]
        u_star, u_orc = z["u_star_sub"], z["u_oracle_sub"]
        e_gpu = relerr(u[idx], u_star)
        e_orc = float(z["oracle_err_full"])
        d = relerr(u[idx], u_orc)
        full = abs(np.linalg.norm(u) / float(z["u_star_norm"]) - 1.0)
        res = np.linalg.norm(sys_g.matvec(u).ravel() - sys_g.rhs) / np.linalg.norm(sys_g.rhs)
        print(f"cfg2 refine={refine}: |u-u*|/|u*| {e_gpu:.3e} (oracle {e_orc:.3e}), vs oracle {d:.3e}, "
              f"norm ratio dev {full:.2e}, relerr_res {res:.2e}")
        res_orc = float(z["residual_history"][0])  # the oracle's own relerr_res (~1.5e-7 here)
        assert res <= max(1e-10, 10.0 * res_orc)
        assert e_gpu <= max(1e-10, 10.0 * e_orc)
        assert d <= 1.5 * (e_gpu + e_orc) + 1e-10


@pytest.mark.parametrize("kind,kappa,res_tol,lo,hi", [
    (0, 0.0, 1e-10, 1e-7, 2e-6),      # test_driver.cpp:314-323
    (1, 27.12, 1e-9, 3e-4, 1e-2),     # test_driver.cpp:325-335
])
def test_reference_accuracy_windows_1000(kind, kappa, res_tol, lo, hi):
    """The reference's slow-suite accuracy windows at 1000^2, b = 60 (automatic -> hbs, as there)."""
    spec = S.poisson_log_problem(1000, 1000) if kind == 0 else S.helmholtz_problem(1000, 1000, kappa)
    rep = S.run_problem(spec, S.SolverConfig(b=60))
    print(f"1000^2 kind {kind}: relerr_res {rep['relerr_res']:.3e} relerr_true {rep['relerr_true']:.3e}")
    assert rep["relerr_res"] < res_tol
    assert lo < rep["relerr_true"] < hi
    if kind == 0:
        assert rep["hbs_max_rank"] > 0  # automatic -> hbs: interfaces wide enough to compress


def test_acceptance_criteria_5_to_7():
    """acceptance.cpp:228-290: 512^2 Poisson window, O(h^2) refinement ratios, 250-ppw Helmholtz."""
    rep = S.run_problem(S.poisson_log_problem(512, 512), S.SolverConfig())
    assert rep["relerr_res"] <= 1e-10 and 5e-7 <= rep["relerr_true"] <= 2e-5        # criterion 5
    errs = [S.run_problem(S.poisson_log_problem(n, n), S.SolverConfig())["relerr_true"] for n in (64, 128, 256, 512)]
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    print(f"criterion 6 ratios {ratios}")
    assert all(3.4 <= r <= 4.6 for r in ratios)                                        # criterion 6
    kappa = S.kappa_from_ppw(250.0, 512)
    rep = S.run_problem(S.helmholtz_problem(512, 512, kappa), S.SolverConfig())
    assert rep["relerr_res"] <= 1e-9 and 1e-4 <= rep["relerr_true"] <= 3e-2           # criterion 7


@pytest.mark.timeout(1800)
def test_cfg4_batched_64_rhs():
    """configs[3]: 2000^2 Helmholtz 10 ppw, b = 100, a 64-column right-hand side (BASELINE.json
    north_star, batched solve).  The batched solve equals column-by-column solves, every column's
    residual is at direct accuracy, and the reduced right-hand side of the batch matches the
    oracle's slabs at an interior interface (stage_one.hpp:415-433)."""
    n, b = 2000, 100
    kappa = S.kappa_from_ppw(10.0, n)
    sys_g = S.assemble_fd5(S.helmholtz_problem(n, n, kappa))
    N = sys_g.dim()
    fact = S.factorize(sys_g, S.SolverConfig(b=b, refine=0, compression=S.CompressionChoice.dense))
    F = np.column_stack([sys_g.rhs, S.gaussian_matrix(N, 63, 4242)])
    U = S.solve(fact, F)
    for c in (0, 7, 8, 31, 63):  # column c alone, and its 8-column task neighbours in the batch
        uc = S.solve(fact, F[:, c:c + 1])[:, 0]
        e = relerr(U[:, c], uc)
        # 8-column DMMA tasks vs the 1-column DFMA kernel: different summation order, amplified
        # by the conditioning of the 10-ppw Helmholtz operator (measured 1.0e-11 on column 0)
        assert e < 1e-9, (c, e)
    R = np.column_stack([sys_g.matvec(U[:, c]).ravel() for c in range(0, 64, 9)]) - F[:, 0:64:9]
    res = np.linalg.norm(R, axis=0) / np.linalg.norm(F[:, 0:64:9], axis=0)
    print(f"cfg4 64-RHS unrefined residuals: max {res.max():.2e}")
    assert res.max() < 1e-8  # unrefined; refine = 1 brings it to ~1e-13 (bench relerr_res)
    # staged parity of the batch's reduced right-hand side at interface 9 (8 sampled columns)
    sys_o = O.system_from_csr(n, n, sys_g.h, sys_g.row_ptr, sys_g.col_idx, sys_g.values, sys_g.rhs)
    O.set_blas_threads(os.cpu_count() or 1)
    cols = [0, 1, 7, 8, 9, 33, 62, 63]
    red = fact.reduce_rhs(F[:, cols])
    j = 9
    off = fact.part.interface_offset(j)
    left, right = O.Slab(sys_o, b, j), O.Slab(sys_o, b, j + 1)
    ref = F[off:off + n][:, cols] - left.contrib(F[:, cols])[1] - right.contrib(F[:, cols])[0]
    e = relerr(red[j * n:(j + 1) * n], ref)
    print(f"cfg4 reduce_rhs interface {j}, 8 of 64 columns: rel diff {e:.3e}")
    assert e < 1e-11
