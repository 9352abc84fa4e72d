"""On-device assembly and validation: the canned problems assembled by a kernel
against the host assemble_fd5 (problem.hpp:78-132), the manufactured solutions, and error_report
(problem.hpp:160-196) on the device against a numpy restatement."""
import numpy as np
import pytest

import paper_2211_07572_b200 as S

pytestmark = pytest.mark.gpu


def host_spec(kind, n1, n2, kappa):
    return (S.poisson_log_problem(n1, n2) if kind == 0 else S.helmholtz_problem(n1, n2, kappa) if kind == 1
            else S.helmholtz_bump_problem(n1, n2, kappa))


@pytest.mark.parametrize("kind,n1,n2,ppw", [(0, 16, 16, None), (1, 37, 23, 12.0), (2, 64, 48, 10.0),
                                            (0, 255, 255, None), (2, 1000, 1000, 10.0)])
def test_device_assembly_matches_host(kind, n1, n2, ppw):
    kappa = 0.0 if ppw is None else S.kappa_from_ppw(ppw, n2)
    hs = S.assemble_fd5(host_spec(kind, n1, n2, kappa))
    rp, ci, v, rhs = S.assemble_canned_device(kind, n1, n2, kappa)
    assert np.array_equal(rp.cpu().numpy(), hs.row_ptr)          # index maps bit-exact
    assert np.array_equal(ci.cpu().numpy(), hs.col_idx)
    dv = v.cpu().numpy()
    assert np.max(np.abs(dv - hs.values) / np.abs(hs.values)) <= 4e-16   # same operation order
    if kind != 2:
        assert np.array_equal(dv, hs.values)
    dr = rhs.cpu().numpy()
    scale = np.max(np.abs(hs.rhs))
    tol = 1e-14 if kind == 0 else 1e-12                           # log vs J0 boundary data
    assert np.max(np.abs(dr - hs.rhs)) <= tol * scale


@pytest.mark.parametrize("kind,n", [(0, 64), (1, 200)])
def test_device_sample_solution(kind, n):
    kappa = 0.0 if kind == 0 else S.kappa_from_ppw(10.0, n)
    d = S.sample_solution_device(kind, n, n, kappa).cpu().numpy()
    h = S.sample_solution(kind, n, n, kappa)
    assert np.max(np.abs(d - h)) <= 1e-12


def test_device_error_report_and_golden():
    """Device assembly -> factorize -> solve -> error_report, all on the GPU; relerr_true equals the
    reference's golden value (test_driver.cpp:247-252, n = 32 Poisson, b = 4)."""
    import torch
    n = 32
    rp, ci, v, rhs = S.assemble_canned_device(0, n, n)
    fact = S.factorize_device(n, n, rp, ci, v, S.SolverConfig(b=4))
    u = torch.empty(1, n * n, dtype=torch.float64, device=rhs.device)
    S.solve_device(fact, rhs.reshape(1, -1), u)
    ut = S.sample_solution_device(0, n, n)
    rep = S.error_report_device(n * n, rp, ci, v, rhs, u, ut)
    assert rep.relerr_true == pytest.approx(4.961321e-04, rel=1e-4)
    assert rep.relerr_res < 1e-12
    # numpy restatement of problem.hpp:177-188 on the same (device-assembled) data; the residual
    # sits at round-off, where summation order alone moves it by ~1e-16
    import scipy.sparse as sp
    a = sp.csr_matrix((v.cpu().numpy(), ci.cpu().numpy(), rp.cpu().numpy()), shape=(n * n, n * n))
    uh, fh = u.cpu().numpy().ravel(), rhs.cpu().numpy()
    res = np.linalg.norm(a @ uh - fh) / np.linalg.norm(fh)
    ref_true = np.linalg.norm(uh - ut.cpu().numpy()) / np.linalg.norm(ut.cpu().numpy())
    assert abs(rep.relerr_res - res) <= 5e-16
    assert rep.relerr_true == pytest.approx(ref_true, rel=1e-12)
    hs = S.assemble_fd5(S.poisson_log_problem(n, n))
    # host-buffer entry point, zero right-hand side: absolute norm flagged
    z = np.zeros(n * n)
    rep0 = S.error_report(hs, z, z, z)
    assert rep0.residual_norm_is_absolute and rep0.solution_norm_is_absolute and rep0.relerr_res == 0.0
