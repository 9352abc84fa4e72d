"""Stage two on caller-built block-tridiagonal systems (sweep_build, stage_two.hpp:126-232),
ported from proj/tests/test_stage_two.cpp: dense agreement, linearity, residual, the
two-thousand scale, exact storage, the singular-block index and the validation rules."""
import numpy as np
import pytest

import paper_2211_07572_b200 as S

pytestmark = pytest.mark.gpu


def random_system(k, m, seed):
    """Diagonally dominant random blocks (test_stage_two.cpp random_system)."""
    rng = np.random.default_rng(seed)
    diag = [rng.standard_normal((m, m)) + 4.0 * m * np.eye(m) for _ in range(k)]
    sup = [rng.standard_normal((m, m)) for _ in range(k - 1)]
    sub = [rng.standard_normal((m, m)) for _ in range(k - 1)]
    return S.BlockTridiagonal(diag, sup, sub)


def test_sweep_matches_dense():  # test_stage_two.cpp:124-135
    t = random_system(4, 8, 29)
    f = np.random.default_rng(31).standard_normal((32, 3))
    expect = np.linalg.solve(t.to_dense(), f)
    u = S.sweep_build(t).solve(f)
    assert np.linalg.norm(u - expect) <= 1e-11 * np.linalg.norm(expect)


def test_linear_in_rhs():  # :137-146
    fact = S.sweep_build(random_system(5, 6, 37))
    rng = np.random.default_rng(41)
    f1, f2 = rng.standard_normal(30), rng.standard_normal(30)
    lhs = fact.solve(2.5 * f1 - 0.75 * f2)
    rhs = 2.5 * fact.solve(f1) - 0.75 * fact.solve(f2)
    assert np.linalg.norm(lhs - rhs) <= 1e-11 * np.linalg.norm(rhs)


def test_residual_stacked_rhs():  # :148-158
    t = random_system(6, 16, 43)
    f = np.random.default_rng(47).standard_normal((96, 3))
    u = S.sweep_build(t).solve(f)
    assert np.linalg.norm(t.to_dense() @ u - f) <= 1e-11 * np.linalg.norm(f)


def test_two_thousand_scale():  # :160-171
    t = random_system(16, 128, 53)
    f = np.random.default_rng(59).standard_normal(16 * 128)
    expect = np.linalg.solve(t.to_dense(), f)
    u = S.sweep_build(t).solve(f)[:, 0]
    assert np.linalg.norm(u - expect) <= 1e-10 * np.linalg.norm(expect)


def test_storage_counted_exactly():  # :170-176
    k, m = 5, 12
    assert S.sweep_build(random_system(k, m, 61)).storage_scalars() == k * m * m + 2 * (k - 1) * m * m


def test_singular_block_named():  # :178-192 (S_1 = I - I I^-1 I = 0)
    eye = np.eye(4)
    t = S.BlockTridiagonal([eye] * 3, [eye] * 2, [eye] * 2)
    with pytest.raises(S.SingularMatrixError) as e:
        S.sweep_build(t)
    assert e.value.index == 1


def test_malformed_rejected():  # :194-216
    with pytest.raises(S.ConfigError):
        S.sweep_build(S.BlockTridiagonal([], [], []))
    t = random_system(3, 4, 67)
    t.diag[1] = np.zeros((5, 5))
    with pytest.raises(S.ConfigError):
        S.sweep_build(t)
    t = random_system(3, 4, 71)
    t.sub = t.sub[:1]
    with pytest.raises(S.ConfigError):
        S.sweep_build(t)
    for bad in (np.nan, np.inf):
        t = random_system(3, 4, 73)
        t.super[0][1, 2] = bad
        with pytest.raises(S.Error, match="non-finite"):
            S.sweep_build(t)


def test_blocks_beyond_4096_rows():
    """Stage-two envelope: blocks of 5000 rows (the panel cluster holds two rows per thread beyond
    4096).  Residual of the block-tridiagonal solve, computed blockwise."""
    k, m = 2, 5000
    rng = np.random.default_rng(71)
    diag = [rng.standard_normal((m, m)) + 2.0 * np.sqrt(m) * np.eye(m) for _ in range(k)]
    sup = [rng.standard_normal((m, m)) for _ in range(k - 1)]
    sub = [rng.standard_normal((m, m)) for _ in range(k - 1)]
    t = S.BlockTridiagonal(diag, sup, sub)
    f = rng.standard_normal(k * m)
    u = S.sweep_build(t).solve(f)[:, 0]
    r = np.concatenate([diag[0] @ u[:m] + sup[0] @ u[m:] - f[:m], sub[0] @ u[:m] + diag[1] @ u[m:] - f[m:]])
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(f)
