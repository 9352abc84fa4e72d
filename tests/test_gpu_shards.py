"""GPU: the engine's strip-sharded factorization/solve with the partitioned
stage two as G logical shards on one device, messages as
device copies (distributed.factorize_logical / solve_logical), and as two
processes over gloo, against the unsharded engine and the oracle."""
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
    (1, 64, 40, 7, 30.0, 8, 3),     # one strip per rank (empty interiors: adjacent separators)
    (2, 160, 80, 9, 50.0, 2, 1),    # long interior chains
    (0, 31, 8, 6, 0.0, 4, 2),       # rank 0 without interfaces, a thin last strip
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


def _mp_worker(rank, world, port, n1, n2, b, kappa, outdir):
    import os
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)  # both processes on the one GPU; messages staged through the host
        sysm = S.assemble_fd5(S.helmholtz_bump_problem(n1, n2, kappa))
        dev = torch.device("cuda", 0)
        rp, ci, v = (torch.from_numpy(x).to(dev) for x in (sysm.row_ptr, sysm.col_idx, sysm.values))
        sh = D.Shard(n1, n2, rp, ci, v, S.SolverConfig(b=b, compression=S.CompressionChoice.dense), rank, world)
        ex = D.TorchExchange(staged=True)
        D.factorize_dist(sh, ex)
        ft = torch.from_numpy(sysm.rhs).to(dev).reshape(1, -1)
        u = torch.zeros_like(ft)
        D.solve_dist(sh, ft, u, ex)
        uh = u.cpu()
        dist.all_reduce(uh)  # disjoint supports: the sum is the assembled solution
        if rank == 0:
            np.save(os.path.join(outdir, "u.npy"), uh.numpy().ravel())
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_engine_multiprocess_gloo(tmp_path):
    """The engine's shard entry points driven by distributed.factorize_dist / solve_dist in two
    processes (gloo, host-staged messages; both ranks share the one GPU of the test box, and no
    kernel waits on another process: every exchange is host-mediated)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n1, n2, b, kappa = 120, 60, 9, 40.0
    mp.spawn(_mp_worker, args=(2, port, n1, n2, b, kappa, str(tmp_path)), nprocs=2, join=True)
    u = np.load(tmp_path / "u.npy")
    so = O.assemble_canned(2, n1, n2, kappa)
    uo = O.factorize(so, b=b).solve(so.rhs)[:, 0]
    assert np.linalg.norm(u - uo) / np.linalg.norm(uo) < 1e-10


def test_shards_compression_choice():
    """A shard holds partial separator blocks, so it cannot compress them: compression = hbs is
    rejected (UnsupportedError) and automatic resolves to dense even on long interfaces."""
    n1 = n2 = 512
    sysm = S.assemble_fd5(S.poisson_log_problem(n1, n2))
    dev = torch.device("cuda", 0)
    rp = torch.from_numpy(sysm.row_ptr).to(dev)
    ci = torch.from_numpy(sysm.col_idx).to(dev)
    v = torch.from_numpy(sysm.values).to(dev)
    with pytest.raises(S.UnsupportedError):
        D.Shard(n1, n2, rp, ci, v, S.SolverConfig(b=40, compression=S.CompressionChoice.hbs), 0, 2)
    sh = D.Shard(n1, n2, rp, ci, v, S.SolverConfig(b=40), 0, 2)  # automatic, n2 >= 512, b >= 16
    assert int(sh.stats.compression) == 1
    sh.close()
