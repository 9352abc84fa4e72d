"""Multi-GPU SlabLU: strip-sharded factorization and solve.

The reference has no multi-GPU path; this is the engine's.  Stage one of
SlabLU is independent per strip, so rank r of G owns the contiguous global
strips [s_begin, s_end) and runs their band LU and Schur sweeps alone.  The
block-tridiagonal stage two (stage_two.hpp:131-188) is eliminated in a
partitioned (SPIKE-style) way: for r > 0 the first interface the rank owns is
its separator, the others form its interior chain, which every rank eliminates
on its own; the G - 1 separators then form a small block-tridiagonal system
swept in rank order with ONE message per rank boundary and phase:

  factorize  eliminate (local)  ;  r-1 -> r : M (n2 x n2)   the separator sweep
  solve      solve_local (local);  r-1 -> r : q (n2 x nrhs) separator forward
                                   r+1 -> r : u of the next separator (n2 x nrhs)

Messages are device tensors moved with torch.distributed send/recv (NCCL over
NVLink between processes; gloo through host staging), or plain device copies
between logical shards of one process (``factorize_logical`` /
``solve_logical``), which is how the single-GPU tests exercise the engine's
shard code.  Any backend with the ``Shard`` method set can be driven by the
same orchestration, which is how the CPU tests (gloo) check the protocol.
"""
import ctypes
from dataclasses import dataclass

from . import _lib
from ._lib import lib
from .slablu import SolverConfig, _check


def shard_ranges(n_strips, n_interfaces, rank, nranks):
    """(s_begin, s_end, j_begin, j_end): mirror of the engine's shard_ranges (engine.cu)."""
    s0 = rank * n_strips // nranks
    s1 = (rank + 1) * n_strips // nranks
    j0 = 0 if rank == 0 else s0 - 1
    j1 = n_interfaces if rank == nranks - 1 else s1 - 1
    return s0, s1, j0, j1


@dataclass
class ShardPlan:
    rank: int
    nranks: int
    s_begin: int
    s_end: int
    j_begin: int
    j_end: int
    n_strips: int
    n_interfaces: int


def shard_plan(n1, n2, b, rank, nranks) -> ShardPlan:
    out = _lib.ShardT()
    _check(lib().slablu_gpu_shard_plan(int(n1), int(n2), int(b), int(rank), int(nranks), ctypes.byref(out)))
    return ShardPlan(out.rank, out.nranks, out.s_begin, out.s_end, out.j_begin, out.j_end, out.n_strips,
                     out.n_interfaces)


def _ptr(t):
    return None if t is None else t.data_ptr()


class Shard:
    """One rank's shard of the factorization on its GPU (C-ABI handle).

    row_ptr/col_idx/values: the full operator's CSR as CUDA tensors of the
    shard's device (every rank reads only its strips and interfaces)."""

    def __init__(self, n1, n2, row_ptr, col_idx, values, config: SolverConfig, rank, nranks):
        import torch
        self.torch = torch
        self.n1, self.n2, self.N = int(n1), int(n2), int(n1) * int(n2)
        self.rank, self.nranks = int(rank), int(nranks)
        self.device = row_ptr.device
        h = ctypes.c_void_p()
        cfg = config._c()
        _check(lib().slablu_gpu_shard_factorize_device(self.n1, self.n2, int(values.numel()), row_ptr.data_ptr(),
                                                        col_idx.data_ptr(), values.data_ptr(), ctypes.byref(cfg),
                                                        self.rank, self.nranks, ctypes.byref(h)))
        self._h = h
        st = _lib.Stats()
        _check(lib().slablu_gpu_stats(self._h, ctypes.byref(st)))
        self.b = int(st.b)
        self.plan = shard_plan(self.n1, self.n2, self.b, self.rank, self.nranks)
        self.stats = st

    def _sync(self):
        # The engine runs on its own stream.  torch.distributed recv/all_reduce and torch
        # kernels (zeros_like, sums) complete on torch's current stream of this device, so
        # every engine call first waits for that stream; the engine's calls return with
        # their outputs complete (include/slablu_gpu.h), so no wait is needed after them.
        if self.device.type == "cuda":
            self.torch.cuda.current_stream(self.device).synchronize()

    def new_message(self, cols):
        """An n2 x cols column-major message buffer (torch shape (cols, n2))."""
        return self.torch.empty((cols, self.n2), dtype=self.torch.float64, device=self.device)

    def eliminate(self):
        """Local elimination of the interior chain and its separator spikes (no communication)."""
        self._sync()
        _check(lib().slablu_gpu_shard_eliminate(self._h))

    def sweep(self, m_in, m_out):
        """Separator sweep step: M_in from rank - 1, M_out to rank + 1 (n2 x n2)."""
        self._sync()
        _check(lib().slablu_gpu_shard_sweep(self._h, _ptr(m_in), _ptr(m_out)))

    def solve_local(self, f):
        """f: (nrhs, N) CUDA tensor (column-major N x nrhs); local reduce + interior solve."""
        nrhs = f.shape[0] if f.dim() == 2 else 1
        self._sync()
        _check(lib().slablu_gpu_shard_solve_local(self._h, f.data_ptr(), self.N, nrhs))

    def solve_forward(self, m_in, m_out):
        """Separator forward step: q from rank - 1, q to rank + 1 (n2 x nrhs)."""
        self._sync()
        _check(lib().slablu_gpu_shard_solve_forward(self._h, _ptr(m_in), _ptr(m_out)))

    def solve_backward(self, m_in, m_out, u):
        """u: (nrhs, N) CUDA tensor; receives this shard's unknowns (others untouched)."""
        self._sync()
        _check(lib().slablu_gpu_shard_solve_backward(self._h, _ptr(m_in), _ptr(m_out), u.data_ptr(), self.N))

    def residual(self, f, u, r):
        """r = f - A u (all rows; f, u, r: (nrhs, N) CUDA tensors)."""
        nrhs = f.shape[0] if f.dim() == 2 else 1
        self._sync()
        _check(lib().slablu_gpu_residual(self._h, f.data_ptr(), self.N, nrhs, u.data_ptr(), self.N, r.data_ptr()))

    def refresh_stats(self):
        st = _lib.Stats()
        _check(lib().slablu_gpu_stats(self._h, ctypes.byref(st)))
        self.stats = st
        return st

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().slablu_gpu_destroy(self._h)
            self._h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TorchExchange:
    """Neighbour messages over torch.distributed (NCCL for CUDA tensors, gloo for CPU).

    staged=True moves CUDA messages through host memory (gloo between processes that share
    one GPU, as the single-GPU multi-process tests do)."""

    def __init__(self, group=None, staged=False):
        import torch.distributed as dist
        self.dist, self.group, self.staged = dist, group, staged
        self.rank = dist.get_rank(group)

    def _send(self, t, peer):
        if self.staged and t.is_cuda:
            t = t.cpu()
        self.dist.send(t, peer, group=self.group)

    def _recv(self, t, peer):
        if self.staged and t.is_cuda:
            h = t.new_empty(t.shape, device="cpu")
            self.dist.recv(h, peer, group=self.group)
            t.copy_(h)
        else:
            self.dist.recv(t, peer, group=self.group)

    def send_next(self, t):
        self._send(t, self.rank + 1)

    def send_prev(self, t):
        self._send(t, self.rank - 1)

    def recv_prev(self, t):
        self._recv(t, self.rank - 1)

    def recv_next(self, t):
        self._recv(t, self.rank + 1)


def factorize_dist(shard, ex):
    """Stage two of a sharded factorization across processes (call after stage one): local
    elimination on every rank at once, then the separator sweep in rank order."""
    last = shard.rank == shard.nranks - 1
    shard.eliminate()
    m_in = None
    if shard.rank > 0:
        m_in = shard.new_message(shard.n2)
        ex.recv_prev(m_in)
    m_out = None if last else shard.new_message(shard.n2)
    shard.sweep(m_in, m_out)
    if not last:
        ex.send_next(m_out)


def solve_dist(shard, f, u, ex):
    """u (nrhs, N), zero-initialised by the caller, receives this rank's unknowns."""
    nrhs = f.shape[0] if f.dim() == 2 else 1
    last = shard.rank == shard.nranks - 1
    shard.solve_local(f)  # every rank at once
    m_in = None
    if shard.rank > 0:
        m_in = shard.new_message(nrhs)
        ex.recv_prev(m_in)
    m_out = None if last else shard.new_message(nrhs)
    shard.solve_forward(m_in, m_out)
    if not last:
        ex.send_next(m_out)
    b_in = None
    if not last:
        b_in = shard.new_message(nrhs)
        ex.recv_next(b_in)
    b_out = shard.new_message(nrhs) if shard.rank > 0 else None
    shard.solve_backward(b_in, b_out, u)
    if shard.rank > 0:
        ex.send_prev(b_out)
    return u


def solve_dist_refined(shard, f, ex, refine=1, group=None):
    """Full solution on every rank: pipelined solve, all-reduce of the disjoint pieces, then
    ``refine`` steps of iterative refinement (every rank forms the whole residual r = f - A u)."""
    import torch
    import torch.distributed as dist
    u = torch.zeros_like(f)
    solve_dist(shard, f, u, ex)
    dist.all_reduce(u, group=group)
    for _ in range(refine):
        r = torch.empty_like(f)
        shard.residual(f, u, r)
        du = torch.zeros_like(f)
        solve_dist(shard, r, du, ex)
        dist.all_reduce(du, group=group)
        u += du
    return u


def factorize_logical(shards):
    """Stage two for G shards held by one process (messages are device copies)."""
    for sh in shards:
        sh.eliminate()
    m = None
    for r, sh in enumerate(shards):
        out = sh.new_message(sh.n2) if r < len(shards) - 1 else None
        sh.sweep(m, out)
        m = out


def solve_logical_refined(shards, f, refine=1):
    """solve_logical + iterative refinement; returns the full solution."""
    import torch
    u = sum(solve_logical(shards, f, [torch.zeros_like(f) for _ in shards]))
    for _ in range(refine):
        r = torch.empty_like(f)
        shards[0].residual(f, u, r)
        u = u + sum(solve_logical(shards, r, [torch.zeros_like(f) for _ in shards]))
    return u


def solve_logical(shards, f, u_parts):
    """Pipelined solve over logical shards; u_parts[r] (zeroed) receives shard r's unknowns."""
    nrhs = f.shape[0] if f.dim() == 2 else 1
    for sh in shards:
        sh.solve_local(f)
    m = None
    for r, sh in enumerate(shards):
        out = sh.new_message(nrhs) if r < len(shards) - 1 else None
        sh.solve_forward(m, out)
        m = out
    m = None
    for r in range(len(shards) - 1, -1, -1):
        sh = shards[r]
        out = sh.new_message(nrhs) if r > 0 else None
        sh.solve_backward(m, out, u_parts[r])
        m = out
    return u_parts
