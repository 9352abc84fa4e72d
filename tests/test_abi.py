"""CPU-side checks of the drop-in boundary (no compute calls need a GPU).

- libslablu_gpu.so loads and exports every entry point declared in
  include/slablu_gpu.h;
- the host-side maps (choose_b, partition) are bit-exact with the oracle and
  the reference's known answers;
- assemble_fd5 produces a CSR bitwise identical to the oracle's restatement;
- with no CUDA device, compute entry points fail loudly (no CPU fallback).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2211_07572_b200 as S
from paper_2211_07572_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "slablu_gpu.h")).read()
    return sorted(set(re.findall(r"\b(slablu_gpu_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(L, name), name
    assert set(syms) == set(_lib.EXPORTS)


def test_choose_b_matches_known_answers(known):
    for key, c in {"choose_b_c0p5": 0.5, "choose_b_c0p6": 0.6, "choose_b_c0p54": 0.54,
                   "choose_b_clamp_hi": 0.6, "choose_b_clamp_lo": 0.05}.items():
        n1, n2, b = known[key]
        assert S.choose_b(int(n1), int(n2), S.SolverConfig(c=c)) == b
    n1, n2, b = known["choose_b_explicit"]
    assert S.choose_b(int(n1), int(n2), S.SolverConfig(b=17, c=0.05)) == b
    for bad in (dict(n1=100, n2=7), dict(n1=100, n2=64, c=0.0), dict(n1=100, n2=64, c=2.5)):
        with pytest.raises(S.ConfigError):
            S.choose_b(bad["n1"], bad["n2"], S.SolverConfig(c=bad.get("c", 0.6)))


@pytest.mark.parametrize("n1", [5, 11, 16, 37, 101, 257, 1000, 4000])
def test_partition_bit_exact_with_oracle(n1):
    for b in sorted({1, 2, 3, 7, 31, 50, 60, 100, 150, n1 - 2}):
        if b < 1 or b > n1 - 2:
            continue
        p = S.partition(n1, 6, b)
        oi, of = O.partition(n1, 6, b)
        assert [(s.first_col, s.width) for s in p.interiors] == [tuple(x) for x in oi.tolist()]
        assert [(s.first_col, s.width) for s in p.interfaces] == [tuple(x) for x in of.tolist()]
    for bad in [(10, 4, 0), (10, 4, 9), (2, 4, 1), (10, 0, 3)]:
        with pytest.raises(S.ConfigError):
            S.partition(*bad)


@pytest.mark.parametrize("kind,n1,n2,kappa", [(0, 40, 24, 0.0), (1, 33, 17, 8.0), (2, 64, 48, 31.4),
                                               (2, 255, 255, 160.85)])
def test_assembly_bitwise_equals_oracle(kind, n1, n2, kappa):
    spec = [S.poisson_log_problem, None, None][kind]
    spec = S.poisson_log_problem(n1, n2) if kind == 0 else (
        S.helmholtz_problem(n1, n2, kappa) if kind == 1 else S.helmholtz_bump_problem(n1, n2, kappa))
    sys_g = S.assemble_fd5(spec)
    sys_o = O.assemble_canned(kind, n1, n2, kappa)
    assert np.array_equal(sys_g.row_ptr, sys_o.row_ptr)
    assert np.array_equal(sys_g.col_idx, sys_o.col_idx)
    assert np.array_equal(sys_g.values, sys_o.values)
    assert np.array_equal(sys_g.rhs, sys_o.rhs)


def test_generic_spec_callbacks_match_hand_matrix(known):
    spec = S.ProblemSpec(3, 3, 0.25, 0.0, body_load=lambda x, y: 1.0)
    s = S.assemble_fd5(spec)
    d, o = known["hand9x9_diag_off"]
    assert s.values.max() == d and s.values.min() == o
    spec2 = S.ProblemSpec(3, 3, 0.25, 0.0, dirichlet_data=lambda x, y: x + y, body_load=lambda x, y: 7.0)
    s2 = S.assemble_fd5(spec2)
    assert s2.rhs[0] == known["dirichlet_fold_corner"][0]
    assert s2.rhs[4] == known["dirichlet_fold_interior"][0]
    with pytest.raises(S.ConfigError):
        S.assemble_fd5(S.ProblemSpec(4, 6, 0.2))
    with pytest.raises(S.Error):
        S.assemble_fd5(S.ProblemSpec(4, 4, 0.2, 1.0, coefficient_field=lambda x, y: -1.0))


def test_bessel_and_gaussian_match_oracle(known):
    rows = known["bessel_j0_table"] + known["bessel_j0_table_2"] + known["bessel_j0_table_3"]
    for t, v in zip(rows[0::2], rows[1::2]):
        assert S.bessel_j0(t) == O.bessel_j0(t)
        assert abs(S.bessel_j0(t) - v) <= 1e-13
    assert np.array_equal(S.gaussian_matrix(50, 3, 41), O.gaussian_matrix(50, 3, 41))
    assert S.kappa_from_ppw(10.0, 512) == O.kappa_from_ppw(10.0, 512)


def test_no_cpu_fallback_without_device():
    if S.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    sysm = S.assemble_fd5(S.poisson_log_problem(16, 16))
    with pytest.raises(S.Error, match="no CUDA device"):
        S.factorize(sysm, S.SolverConfig(b=4))
    # the other compute entry points fail the same way (HBS compression, stage two on caller
    # blocks): no CPU path behind any of them
    with pytest.raises(S.Error, match="no CUDA device"):
        S.hbs_compress(np.eye(32), 8, 4)
    eye = np.eye(4)
    with pytest.raises(S.Error, match="no CUDA device"):
        S.sweep_build(S.BlockTridiagonal([eye] * 2, [eye], [eye]))
