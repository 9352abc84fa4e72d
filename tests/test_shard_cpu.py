"""Multi-GPU host logic on CPU: shard ranges (Python == C ABI) and the partitioned
factorize/solve protocol (local elimination + separator sweep) over
torch.distributed gloo, world_size 2 to 4, with the numpy shard backend
(tests/shard_cpu.py), checked against the oracle's unsharded solve
(SURVEY.md §8(e))."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2211_07572_b200 as S
from paper_2211_07572_b200 import distributed as D


@pytest.mark.parametrize("n1,n2,b", [(40, 10, 3), (64, 40, 7), (255, 255, 31), (4000, 4000, 150), (39, 8, 4)])
def test_shard_ranges_match_abi(n1, n2, b):
    part = S.partition(n1, n2, b)
    Sg, K = part.interior_count(), part.interface_count()
    for G in range(1, min(Sg, 8) + 1):
        cover_s, cover_j = [], []
        for r in range(G):
            plan = D.shard_plan(n1, n2, b, r, G)
            assert (plan.s_begin, plan.s_end, plan.j_begin, plan.j_end) == D.shard_ranges(Sg, K, r, G)
            assert (plan.n_strips, plan.n_interfaces) == (Sg, K)
            cover_s += list(range(plan.s_begin, plan.s_end))
            cover_j += list(range(plan.j_begin, plan.j_end))
        assert cover_s == list(range(Sg))  # every strip on exactly one rank
        assert cover_j == list(range(K))   # every interface owned by exactly one rank


def test_shard_plan_rejects_too_many_ranks():
    part = S.partition(40, 10, 3)
    with pytest.raises(S.ConfigError):
        D.shard_plan(40, 10, 3, 0, part.interior_count() + 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n1, n2, b, kappa, nrhs, outdir):
    from shard_cpu import CpuShard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        sysm = S.assemble_fd5(S.helmholtz_problem(n1, n2, kappa) if kappa else S.poisson_log_problem(n1, n2))
        part = S.partition(n1, n2, b)
        geo = ([(g.first_col, g.width) for g in part.interiors], [(g.first_col, g.width) for g in part.interfaces])
        sh = CpuShard(n1, n2, sysm.row_ptr, sysm.col_idx, sysm.values, b, rank, world, geo)
        ex = D.TorchExchange()
        D.factorize_dist(sh, ex)
        f = np.column_stack([sysm.rhs] + [S.gaussian_matrix(sysm.dim(), 1, 7 + c)[:, 0] for c in range(nrhs - 1)])
        ft = torch.from_numpy(np.ascontiguousarray(f.T))
        u = torch.zeros_like(ft)
        D.solve_dist(sh, ft, u, ex)
        dist.all_reduce(u)  # disjoint supports: the sum is the assembled solution
        if rank == 0:
            np.save(os.path.join(outdir, "u.npy"), u.numpy().T)
            np.save(os.path.join(outdir, "f.npy"), f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n1,n2,b,kappa,nrhs", [(2, 40, 10, 3, 0.0, 1), (3, 40, 10, 3, 12.0, 2),
                                                      (2, 39, 8, 4, 0.0, 1), (4, 40, 10, 3, 9.0, 1),
                                                      (4, 31, 8, 6, 0.0, 2)])
def test_partitioned_protocol_gloo(tmp_path, world, n1, n2, b, kappa, nrhs):
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = here + os.pathsep + os.environ.get("PYTHONPATH", "")
    mp.spawn(_worker, args=(world, _free_port(), n1, n2, b, kappa, nrhs, str(tmp_path)), nprocs=world, join=True)
    u = np.load(tmp_path / "u.npy")
    f = np.load(tmp_path / "f.npy")
    kind = 1 if kappa else 0
    so = O.assemble_canned(kind, n1, n2, kappa)
    fo = O.factorize(so, b=b)
    uo = fo.solve(f)
    assert np.linalg.norm(u - uo) / np.linalg.norm(uo) < 1e-10
