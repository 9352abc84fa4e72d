"""Randomized HBS compression on the GPU (hbs.cu) against the reference's own HBS tests.

Ports test_hbs.cpp:175-372 (compression of dense operators through the dense sampler),
test_stage_one.cpp:347-369 (compressed vs dense reduction at 1e-9), test_driver.cpp:163-184
(the compressed factorization path and the automatic dispatch, driver.hpp:125-130) and
acceptance criterion 4 (acceptance.cpp:153-200).  Random matrices come from numpy here (the
reference's come from mt19937_64); every assertion is a property the reference asserts.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2211_07572_b200 as S

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def csr(sysm):
    n = sysm.dim()
    return sp.csr_matrix((sysm.values, sysm.col_idx, sysm.row_ptr), shape=(n, n))


def interface_schur_dense(n, b):
    """test_hbs.cpp:70-86: one interface between two b-wide Poisson slabs, formed densely."""
    A = csr(S.assemble_fd5(S.poisson_log_problem(n, n))).tocsc()
    iface, w = b * n, b * n
    t = A[iface:iface + n, iface:iface + n].toarray()
    for j0 in (0, iface + n):
        ajj = A[j0:j0 + w, j0:j0 + w].toarray()
        aij = A[iface:iface + n, j0:j0 + w].toarray()
        aji = A[j0:j0 + w, iface:iface + n].toarray()
        t -= aij @ np.linalg.solve(ajj, aji)
    return t


def test_diagonal_operator_zero_width():
    """test_hbs.cpp:213-226."""
    rng = np.random.default_rng(11)
    m = np.diag(1.0 + np.abs(rng.standard_normal(96)))
    h, st = S.hbs_compress(m, 16, 2)
    assert st.final_rank == 0
    assert np.linalg.norm(h - m) <= 1e-13 * np.linalg.norm(m)
    assert st.residual_estimate <= 1e-13


def test_global_rank_one_offdiagonal():
    """test_hbs.cpp:228-245: rank-one coupling recovered within a rank-1 budget."""
    n = 64
    rng = np.random.default_rng(13)
    m = np.zeros((n, n))
    for k in range(8):
        sl = slice(8 * k, 8 * k + 8)
        m[sl, sl] = rng.standard_normal((8, 8)) + 10.0 * np.eye(8)
    m += np.outer(rng.standard_normal(n), rng.standard_normal(n))
    h, st = S.hbs_compress(m, 8, 1, S.CompressOptions(1e-10, 1e-12, 5))
    assert rel(h, m) <= 1e-12
    assert st.final_rank <= 1


def test_interface_schur_complement_exact_rank():
    """test_hbs.cpp:247-280: rank 2b+2 off-diagonal blocks; a 2b budget fails loudly."""
    b = 4
    t = interface_schur_dense(64, b)
    r = 2 * b + 2
    h, st = S.hbs_compress(t, 16, r, S.CompressOptions(1e-10, 1e-12, 7))
    assert rel(h, t) <= 1e-10
    assert st.products_normal <= 4 * r + 16 and st.products_adjoint <= 4 * r + 16
    with pytest.raises(S.CompressionError) as e:
        S.hbs_compress(t, 16, 2 * b, S.CompressOptions(1e-10, 1e-12, 7))
    assert e.value.residual_estimate > 1e-10


def test_infeasible_rank_bound_rejected():
    """test_hbs.cpp:282-293."""
    with pytest.raises(S.CompressionError):
        S.hbs_compress(np.eye(128), 64, 8)
    with pytest.raises(S.ConfigError):
        S.hbs_compress(np.eye(4), 9, 2)


def test_adaptive_doubles_to_needed_rank():
    """test_hbs.cpp:307-341."""
    n, true_rank = 96, 5
    rng = np.random.default_rng(31)
    m = 20.0 * np.eye(n) + rng.standard_normal((n, true_rank)) @ rng.standard_normal((n, true_rank)).T
    h, st = S.hbs_compress_adaptive(m, 12, 2, 64, S.CompressOptions(1e-10, 1e-12, 37))
    assert rel(h, m) <= 1e-10
    assert st.rounds <= 3
    assert st.final_rank <= 10
    assert st.products_normal <= 4 * 8 + 16 and st.products_adjoint <= 4 * 8 + 16
    _, one = S.hbs_compress_adaptive(m, 12, 6, 64, S.CompressOptions(1e-10, 1e-12, 37))
    assert one.rounds == 1


def test_adaptive_reports_failure_at_ceiling():
    """test_hbs.cpp:343-359."""
    n = 96
    rng = np.random.default_rng(41)
    m = 20.0 * np.eye(n) + rng.standard_normal((n, 20)) @ rng.standard_normal((n, 20)).T
    with pytest.raises(S.CompressionError) as e:
        S.hbs_compress_adaptive(m, 12, 2, 8, S.CompressOptions(1e-10, 1e-12, 43))
    assert e.value.residual_estimate > 1e-10 and np.isfinite(e.value.residual_estimate)


def test_residual_monotone_in_rank_budget():
    """test_hbs.cpp:374-397 (lower median over 10 seeds)."""
    n = 64
    rng = np.random.default_rng(61)
    q1 = np.linalg.qr(rng.standard_normal((n, 16)))[0]
    q2 = np.linalg.qr(rng.standard_normal((n, 16)))[0]
    m = 50.0 * np.eye(n) + q1 @ np.diag(0.5 ** np.arange(16)) @ q2.T

    def med(r):
        out = sorted(rel(S.hbs_compress(m, 16, r, S.CompressOptions(2.0, 1e-15, seed))[0], m) for seed in range(10))
        return out[4]

    assert med(8) <= med(4)


def test_seed_determinism():
    """Same seed, same result bit for bit (the reference's replay contract, hbs_compress.hpp:40)."""
    t = interface_schur_dense(64, 4)
    a, _ = S.hbs_compress(t, 16, 10, S.CompressOptions(1e-10, 1e-12, 53))
    b, _ = S.hbs_compress(t, 16, 10, S.CompressOptions(1e-10, 1e-12, 53))
    assert np.array_equal(a, b)


def _reduced(fact):
    K = len(fact.part.interfaces)
    out = [fact.T_block("diag", j) for j in range(K)]
    for j in range(K - 1):
        out += [fact.T_block("super", j), fact.T_block("sub", j)]
    return out


def test_compressed_reduction_matches_dense():
    """test_stage_one.cpp:347-369: every compressed block within 1e-9 of the dense one."""
    sysm = S.assemble_fd5(S.poisson_log_problem(64, 64))
    dense = S.factorize(sysm, S.SolverConfig(b=4, keep_T=True, compression=S.CompressionChoice.dense))
    comp = S.factorize(sysm, S.SolverConfig(b=4, keep_T=True, compression=S.CompressionChoice.hbs,
                                            hbs_leaf_size=16, seed=7))
    assert comp.config.compression == S.CompressionChoice.hbs
    assert 0 < comp.hbs_max_rank <= 16
    for tc, td in zip(_reduced(comp), _reduced(dense)):
        assert rel(tc, td) < 1e-9


def test_acceptance_criterion_4():
    """acceptance.cpp:153-200: tol 1e-12 / trunc 1e-14 -> every block within 1e-10."""
    sysm = S.assemble_fd5(S.poisson_log_problem(64, 64))
    dense = S.factorize(sysm, S.SolverConfig(b=4, keep_T=True, compression=S.CompressionChoice.dense))
    comp = S.factorize(sysm, S.SolverConfig(b=4, keep_T=True, compression=S.CompressionChoice.hbs,
                                            hbs_leaf_size=16, hbs_tol=1e-12, hbs_trunc_rel=1e-14))
    worst = max(rel(tc, td) for tc, td in zip(_reduced(comp), _reduced(dense)))
    print(f"criterion 4 worst block {worst:.2e}")
    assert worst <= 1e-10


def test_compressed_factorization_solves():
    """test_driver.cpp:163-184: hbs path solves to 1e-9; automatic stays dense on small interfaces."""
    sysm = S.assemble_fd5(S.poisson_log_problem(64, 64))
    fact = S.factorize(sysm, S.SolverConfig(b=4, compression=S.CompressionChoice.hbs, hbs_leaf_size=16))
    assert fact.config.compression == S.CompressionChoice.hbs
    assert fact.hbs_max_rank > 0
    u = S.solve(fact, sysm.rhs)[:, 0]
    u_ref = sp.linalg.spsolve(csr(sysm).tocsc(), sysm.rhs)
    assert rel(u, u_ref) < 1e-9
    plain = S.factorize(sysm, S.SolverConfig(b=4))
    assert plain.config.compression == S.CompressionChoice.dense
    assert plain.hbs_max_rank == 0


def test_automatic_dispatch_picks_hbs_on_long_interfaces():
    """driver.hpp:125-130: n2 >= 512 and b >= 16 -> hbs; the solution stays at direct accuracy."""
    sysm = S.assemble_fd5(S.poisson_log_problem(512, 512))
    fact = S.factorize(sysm, S.SolverConfig(b=40))
    assert fact.config.compression == S.CompressionChoice.hbs
    assert fact.hbs_max_rank > 0
    u = S.solve(fact, sysm.rhs)[:, 0]
    r = csr(sysm) @ u - sysm.rhs
    assert np.linalg.norm(r) / np.linalg.norm(sysm.rhs) < 1e-10
    print(f"512^2 b=40 automatic: hbs_max_rank {fact.hbs_max_rank}, t_hbs {fact.stats.t_hbs:.3f} s, "
          f"t_stage1 {fact.t_stage1:.3f} s")
    small_b = S.factorize(sysm, S.SolverConfig(b=10))
    assert small_b.config.compression == S.CompressionChoice.dense
