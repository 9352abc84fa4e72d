"""CPU (numpy) backend with the method set of paper_2211_07572_b200.distributed.Shard.

Test infrastructure only: it restates, densely and for small grids, what the
engine's shard entry points compute (engine.cu shard_eliminate_impl /
shard_sweep_impl / shard_solve_local_impl / shard_solve_fwd_impl /
shard_solve_bwd_impl: partitioned elimination with the separator sweep) so that
the multi-process orchestration (distributed.factorize_dist / solve_dist over
gloo) can be checked on CPU against the oracle's unsharded solve.  The interior
chain and its spikes are formed as dense matrices here (the engine sweeps them
block by block).  Block definitions follow stage_one.hpp:284-297 (T blocks),
:415-462 (reduce / recover) and stage_two.hpp:131-188 (sweep)."""
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

    # ---- partitioned stage two ------------------------------------------------
    def eliminate(self):
        n2, j0, j1 = self.n2, self.j0, self.j1
        self.has_left, self.has_right = self.rank > 0, self.rank < self.nranks - 1
        self.ia, self.ib = (j0 + 1 if self.has_left else 0), j1
        ia, ib = self.ia, self.ib
        m = ib - ia
        Z = np.zeros((n2, n2))
        self.a = self.b = self.c = self.d = self.yl = Z
        if m == 0:
            if self.has_left and self.has_right:
                self.b, self.c = -self.Tsup[j0], -self.Tsub[j0]
            return
        AI = np.zeros((m * n2, m * n2))
        for k, j in enumerate(range(ia, ib)):
            AI[k * n2:(k + 1) * n2, k * n2:(k + 1) * n2] = self.Tdiag[j]
            if j + 1 < ib:
                AI[k * n2:(k + 1) * n2, (k + 1) * n2:(k + 2) * n2] = self.Tsup[j]
                AI[(k + 1) * n2:(k + 2) * n2, k * n2:(k + 1) * n2] = self.Tsub[j]
        self.AI = AI
        if self.has_left:
            EL = np.zeros((m * n2, n2))
            EL[:n2] = self.Tsub[j0]
            YL = np.linalg.solve(AI, EL)
            self.a = self.Tsup[j0] @ YL[:n2]
            if self.has_right:
                self.yl = YL[-n2:]
                self.c = self.Tsub[ib - 1] @ self.yl
        if self.has_right:
            ER = np.zeros((m * n2, n2))
            ER[-n2:] = self.Tsup[ib - 1]
            YR = np.linalg.solve(AI, ER)
            self.d = self.Tsub[ib - 1] @ YR[-n2:]
            if self.has_left:
                self.b = self.Tsup[j0] @ YR[:n2]

    def sweep(self, m_in, m_out):
        j0, j1 = self.j0, self.j1
        if self.has_left:
            self.Shat = self.Tdiag[j0] - self.a + m_in.numpy().T
            if self.has_right:
                self.xhat = np.linalg.solve(self.Shat, self.b)
        if self.has_right:
            M = self.Tdiag[j1] - self.d
            if self.has_left:
                M = M - self.c @ self.xhat
            m_out.copy_(torch.from_numpy(np.ascontiguousarray(M.T)))

    def solve_local(self, f):
        F = f.numpy().reshape(-1, self.N).T.copy()
        self.F = F
        red = {j: (F[self.iidx[j]].copy() if self.j0 <= j < self.j1 else np.zeros((self.n2, F.shape[1])))
               for j in range(self.K)}
        for s in range(self.s0, self.s1):
            xs = self.Ainv[s] @ F[self.sidx[s]]
            for j in (s - 1, s):
                if 0 <= j < self.K:
                    red[j] -= self.A[np.ix_(self.iidx[j], self.sidx[s])] @ xs
        self.red = red
        ia, ib, n2 = self.ia, self.ib, self.n2
        if ib > ia:
            z = np.linalg.solve(self.AI, np.vstack([red[j] for j in range(ia, ib)]))
            self.z = {j: z[(j - ia) * n2:(j - ia + 1) * n2] for j in range(ia, ib)}

    def solve_forward(self, m_in, m_out):
        j0, j1, ia, ib = self.j0, self.j1, self.ia, self.ib
        interior = ib > ia
        if self.has_left:
            rhs = self.red[j0] + m_in.numpy().T
            if interior:
                rhs = rhs - self.Tsup[j0] @ self.z[ia]
            self.v = np.linalg.solve(self.Shat, rhs)
        if self.has_right:
            q = self.red[j1].copy()
            if interior:
                t = self.z[ib - 1] - (self.yl @ self.v if self.has_left else 0.0)
                q = q - self.Tsub[ib - 1] @ t
            elif self.has_left:
                q = q - self.Tsub[j0] @ self.v
            m_out.copy_(torch.from_numpy(np.ascontiguousarray(q.T)))

    def solve_backward(self, m_in, m_out, u_t):
        j0, j1, ia, ib, n2 = self.j0, self.j1, self.ia, self.ib, self.n2
        u = {}
        if self.has_right:
            u[j1] = m_in.numpy().T.copy()
        if self.has_left:
            u[j0] = self.v + (self.xhat @ u[j1] if self.has_right else 0.0)
            m_out.copy_(torch.from_numpy(np.ascontiguousarray(u[j0].T)))
        if ib > ia:
            rhs = np.vstack([self.red[j] for j in range(ia, ib)])
            if self.has_left:
                rhs[:n2] -= self.Tsub[j0] @ u[j0]
            if self.has_right:
                rhs[-n2:] -= self.Tsup[ib - 1] @ u[j1]
            uI = np.linalg.solve(self.AI, rhs)
            for j in range(ia, ib):
                u[j] = uI[(j - ia) * n2:(j - ia + 1) * n2]
        U = u_t.numpy().reshape(-1, self.N).T  # view (N x nrhs)
        for s in range(self.s0, self.s1):
            rhs = self.F[self.sidx[s]].copy()
            for j in (s - 1, s):
                if 0 <= j < self.K:
                    rhs -= self.A[np.ix_(self.sidx[s], self.iidx[j])] @ u[j]
            U[self.sidx[s]] = self.Ainv[s] @ rhs
        for j in range(self.j0, self.j1):
            U[self.iidx[j]] = u[j]
