"""CPU (numpy) backend with the method set of paper_2211_07572_b200.distributed.Shard.

Test infrastructure only: it restates, densely and for small grids, what the
engine's shard entry points compute (engine.cu shard_sweep_impl /
shard_solve_fwd_impl / shard_solve_bwd_impl) so that the multi-process
orchestration (distributed.factorize_dist / solve_dist over gloo) can be
checked on CPU against the oracle's unsharded solve.  Block definitions follow
stage_one.hpp:284-297 (T blocks), :415-462 (reduce / recover) and
stage_two.hpp:131-188 (sweep)."""
import numpy as np
import scipy.sparse as sp
import torch

from paper_2211_07572_b200.distributed import shard_ranges


class CpuShard:
    def __init__(self, n1, n2, row_ptr, col_idx, values, b, rank, nranks, partition):
        self.n1, self.n2, self.N = n1, n2, n1 * n2
        self.rank, self.nranks = rank, nranks
        A = sp.csr_matrix((values, col_idx, row_ptr), shape=(self.N, self.N)).toarray()
        self.A = A
        ints, ifcs = partition
        self.Sg, self.K = len(ints), len(ifcs)
        s0, s1, j0, j1 = shard_ranges(self.Sg, self.K, rank, nranks)
        self.s0, self.s1, self.j0, self.j1 = s0, s1, j0, j1
        self.sidx = [np.arange(c * n2, (c + w) * n2) for c, w in ints]
        self.iidx = [np.arange(c * n2, (c + 1) * n2) for c, _ in ifcs]
        K = self.K
        self.Ainv = {s: np.linalg.inv(A[np.ix_(self.sidx[s], self.sidx[s])]) for s in range(s0, s1)}

        def side(s, X):  # interface index on side X (0 left, 1 right) of strip s, or None
            j = s - 1 if X == 0 else s
            return j if 0 <= j < K else None

        def contrib(s, X, Y):
            jx, jy = side(s, X), side(s, Y)
            if s not in self.Ainv or jx is None or jy is None:
                return 0.0
            ix, iy, si = self.iidx[jx], self.iidx[jy], self.sidx[s]
            return A[np.ix_(ix, si)] @ self.Ainv[s] @ A[np.ix_(si, iy)]

        self.Tdiag, self.Tsup, self.Tsub = {}, {}, {}
        for j in range(max(0, s0 - 1), min(K, s1)):
            blk = A[np.ix_(self.iidx[j], self.iidx[j])].copy() if j0 <= j < j1 else np.zeros((n2, n2))
            blk = blk - contrib(j, 1, 1)
            if j + 1 < self.Sg:
                blk = blk - contrib(j + 1, 0, 0)
            self.Tdiag[j] = blk
        for j in range(max(0, s0 - 1), min(K - 1, s1 - 1)):
            self.Tsup[j] = A[np.ix_(self.iidx[j], self.iidx[j + 1])] - contrib(j + 1, 0, 1)
            self.Tsub[j] = A[np.ix_(self.iidx[j + 1], self.iidx[j])] - contrib(j + 1, 1, 0)
        self.Sinv = {}

    def new_message(self, cols):
        return torch.zeros((cols, self.n2), dtype=torch.float64)

    def sweep(self, m_in, m_out):
        j0, j1 = self.j0, self.j1
        for j in range(j0, j1):
            Sj = self.Tdiag[j].copy()
            if j == j0 and self.rank > 0:
                Sj += m_in.numpy().T
            if j > j0:
                Sj -= self.Tsub[j - 1] @ self.Sinv[j - 1] @ self.Tsup[j - 1]
            self.Sinv[j] = np.linalg.inv(Sj)
        if self.rank < self.nranks - 1:
            M = self.Tdiag[j1].copy()
            if j1 > j0:
                M -= self.Tsub[j1 - 1] @ self.Sinv[j1 - 1] @ self.Tsup[j1 - 1]
            m_out.copy_(torch.from_numpy(np.ascontiguousarray(M.T)))

    def solve_forward(self, f, m_in, m_out):
        F = f.numpy().reshape(-1, self.N).T.copy()
        self.F = F
        red = {j: (F[self.iidx[j]].copy() if self.j0 <= j < self.j1 else np.zeros((self.n2, F.shape[1])))
               for j in range(self.K)}
        for s in range(self.s0, self.s1):
            xs = self.Ainv[s] @ F[self.sidx[s]]
            for j in (s - 1, s):
                if 0 <= j < self.K:
                    red[j] -= self.A[np.ix_(self.iidx[j], self.sidx[s])] @ xs
        if self.rank > 0:
            red[self.j0] += m_in.numpy().T
        u = {}
        for j in range(self.j0, self.j1):
            r = red[j] - (self.Tsub[j - 1] @ u[j - 1] if j > self.j0 else 0.0)
            u[j] = self.Sinv[j] @ r
        if self.rank < self.nranks - 1:
            out = red[self.j1] - (self.Tsub[self.j1 - 1] @ u[self.j1 - 1] if self.j1 > self.j0 else 0.0)
            m_out.copy_(torch.from_numpy(np.ascontiguousarray(out.T)))
        self.u = u

    def solve_backward(self, m_in, m_out, u_t):
        u = self.u
        if self.rank < self.nranks - 1:
            u[self.j1] = m_in.numpy().T.copy()
        for j in range(self.j1 - 1, self.j0 - 1, -1):
            if j + 1 < self.K:
                u[j] = u[j] - self.Sinv[j] @ (self.Tsup[j] @ u[j + 1])
        if self.rank > 0:
            m_out.copy_(torch.from_numpy(np.ascontiguousarray(u[self.j0].T)))
        U = u_t.numpy().reshape(-1, self.N).T  # view (N x nrhs)
        for s in range(self.s0, self.s1):
            rhs = self.F[self.sidx[s]].copy()
            for j in (s - 1, s):
                if 0 <= j < self.K:
                    rhs -= self.A[np.ix_(self.sidx[s], self.iidx[j])] @ u[j]
            U[self.sidx[s]] = self.Ainv[s] @ rhs
        for j in range(self.j0, self.j1):
            U[self.iidx[j]] = u[j]
