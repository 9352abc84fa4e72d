"""GPU: the engine's strip-sharded factorization/solve as G
logical shards on one device, messages as device copies
(distributed.factorize_logical / solve_logical), against the unsharded
engine and the oracle."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2211_07572_b200 as S
from paper_2211_07572_b200 import distributed as D

pytestmark = pytest.mark.gpu


def _shards(sysm, n1, n2, b, G):
    dev = torch.device("cuda", 0)
    rp = torch.from_numpy(sysm.row_ptr).to(dev)
    ci = torch.from_numpy(sysm.col_idx).to(dev)
    v = torch.from_numpy(sysm.values).to(dev)
    cfg = S.SolverConfig(b=b, compression=S.CompressionChoice.dense)
    return [D.Shard(n1, n2, rp, ci, v, cfg, r, G) for r in range(G)], dev


@pytest.mark.parametrize("kind,n1,n2,b,kappa,G,nrhs", [
    (0, 40, 10, 3, 0.0, 2, 1),      # trailing interface
    (1, 64, 40, 7, 30.0, 3, 2),
    (2, 120, 60, 9, 40.0, 4, 1),
    (1, 64, 40, 7, 30.0, 8, 3),     # one strip per rank
    (1, 64, 40, 7, 30.0, 1, 1),     # one shard = the whole problem through the shard entry points
])
def test_logical_shards_match_oracle(kind, n1, n2, b, kappa, G, nrhs):
    spec = (S.poisson_log_problem(n1, n2) if kind == 0 else
            S.helmholtz_problem(n1, n2, kappa) if kind == 1 else S.helmholtz_bump_problem(n1, n2, kappa))
    sysm = S.assemble_fd5(spec)
    shards, dev = _shards(sysm, n1, n2, b, G)
    D.factorize_logical(shards)
    N = sysm.dim()
    f = np.column_stack([sysm.rhs] + [S.gaussian_matrix(N, 1, 3 + c)[:, 0] for c in range(nrhs - 1)])
    ft = torch.from_numpy(np.ascontiguousarray(f.T)).to(dev)
    parts = [torch.zeros_like(ft) for _ in range(G)]
    D.solve_logical(shards, ft, parts)
    u = sum(p for p in parts).cpu().numpy().T
    # every unknown written by exactly one shard
    written = sum((p != 0).to(torch.int32) for p in parts).cpu().numpy()
    assert written.max() <= 1
    fo = O.factorize(O.assemble_canned(kind, n1, n2, kappa), b=b)
    uo = fo.solve(f)
    assert np.linalg.norm(u - uo) / np.linalg.norm(uo) < 1e-10
    # the unsharded engine (direct solve) agrees too
    fg = S.factorize(sysm, S.SolverConfig(b=b, refine=0))
    ug = S.solve(fg, f)
    assert np.linalg.norm(u - ug) / np.linalg.norm(ug) < 1e-10
    for sh in shards:
        sh.close()


def test_logical_shards_refined_backward_error():
    n1, n2, b, kappa, G = 200, 120, 15, 80.0, 3
    sysm = S.assemble_fd5(S.helmholtz_bump_problem(n1, n2, kappa))
    shards, dev = _shards(sysm, n1, n2, b, G)
    D.factorize_logical(shards)
    ft = torch.from_numpy(sysm.rhs).to(dev).reshape(1, -1)
    u0 = D.solve_logical_refined(shards, ft, refine=0).cpu().numpy().ravel()
    u1 = D.solve_logical_refined(shards, ft, refine=1).cpu().numpy().ravel()
    rows = np.repeat(np.arange(sysm.dim()), np.diff(sysm.row_ptr))
    a_inf = np.bincount(rows, weights=np.abs(sysm.values)).max()

    def berr(u):
        return np.linalg.norm(sysm.matvec(u) - sysm.rhs) / (a_inf * np.linalg.norm(u) + np.linalg.norm(sysm.rhs))
    assert berr(u1) < 1e-15
    assert berr(u1) <= berr(u0)
    for sh in shards:
        sh.close()


def test_sharded_factorization_refuses_plain_solve():
    sysm = S.assemble_fd5(S.poisson_log_problem(40, 10))
    shards, dev = _shards(sysm, 40, 10, 3, 2)
    D.factorize_logical(shards)
    from paper_2211_07572_b200._lib import lib
    from paper_2211_07572_b200.slablu import _check
    f = torch.zeros((1, 400), dtype=torch.float64, device=dev)
    with pytest.raises(S.ConfigError):
        _check(lib().slablu_gpu_solve_device(shards[0]._h, f.data_ptr(), 400, 1, f.data_ptr(), 400))
    with pytest.raises(S.ConfigError):  # backward before forward
        shards[1].solve_backward(None, shards[1].new_message(1), torch.zeros((1, 400), dtype=torch.float64, device=dev))
