"""Python mirror of the reference's solver API on top of the C ABI.

Names, argument meaning and error behaviour follow the reference library
(/root/reference/proj/include/slablu/):

    ProblemSpec, poisson_log_problem, helmholtz_problem,
    helmholtz_bump_problem, kappa_from_ppw         problem.hpp:35-48, 153-157, 210-261
    SparseSystem, assemble_fd5                     problem.hpp:52-64, 78-132
    error_report, sample_field                     problem.hpp:160-206
    SolverConfig, CompressionChoice, choose_b      driver.hpp:37-66
    GridStrip, SlabPartition, partition            partition.hpp:27-91
    Factorization, factorize, solve                driver.hpp:72-179
    Error, ConfigError, SingularMatrixError        common.hpp:32-60

Compute runs on the B200 through libslablu_gpu.so; this module only
marshals arguments (numpy for host data, torch CUDA tensors for the
device-resident entry points).
"""
import ctypes
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from ._lib import lib


# ---------------------------------------------------------------------------
# errors (common.hpp:32-60)
class Error(RuntimeError):
    pass


class ConfigError(Error):
    pass


class SingularMatrixError(Error):
    def __init__(self, what, index):
        super().__init__(f"{what} (index {index})")
        self.index = index


class UnsupportedError(Error):
    pass


class CompressionError(Error):
    """common.hpp:55-60: the probe missed the tolerance; carries the residual estimate."""

    def __init__(self, what, residual_estimate):
        super().__init__(what)
        self.residual_estimate = residual_estimate


def _check(st):
    if st.code == 0:
        return
    msg = st.msg.decode(errors="replace")
    if st.code == 2:
        raise ConfigError(msg)
    if st.code == 3:
        raise SingularMatrixError(msg, int(st.index))
    if st.code == 6:
        raise UnsupportedError(msg)
    if st.code == 7:
        raise CompressionError(msg, float(st.residual))
    if st.code == 5:
        raise MemoryError(msg)
    raise Error(msg)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def device_count():
    return lib().slablu_gpu_device_count()


# ---------------------------------------------------------------------------
# problems (problem.hpp)
ScalarField = Callable[[float, float], float]


@dataclass
class ProblemSpec:
    n1: int = 0
    n2: int = 0
    h: float = 0.0
    kappa: float = 0.0
    coefficient_field: ScalarField = field(default=lambda x, y: 1.0)
    dirichlet_data: ScalarField = field(default=lambda x, y: 0.0)
    body_load: ScalarField = field(default=lambda x, y: 0.0)
    canned: Optional[int] = None  # 0 poisson_log, 1 helmholtz, 2 helmholtz_bump (native fast path)


def kappa_from_ppw(ppw, n2):
    if not (ppw > 0.0):
        raise ConfigError("kappa_from_ppw: ppw must be positive")
    if n2 < 2:
        raise ConfigError("kappa_from_ppw: n2 must be at least 2")
    return lib().slablu_gpu_kappa_from_ppw(float(ppw), int(n2))


def bessel_j0(t):
    return lib().slablu_gpu_bessel_j0(float(t))


def true_solution_poisson(x, y):
    r = np.hypot(x + 0.1, y - 0.5)
    if r == 0.0:
        raise Error("true_solution_poisson: evaluated at the source point")
    return float(np.log(r))


def true_solution_helmholtz(x, y, kappa):
    if kappa < 0.0:
        raise Error("true_solution_helmholtz: kappa must be nonnegative")
    return bessel_j0(kappa * np.hypot(x + 0.1, y - 0.5))


def poisson_log_problem(n1, n2):
    return ProblemSpec(n1, n2, 1.0 / (n2 + 1), 0.0, lambda x, y: 1.0,
                       true_solution_poisson, lambda x, y: 0.0, canned=0)


def helmholtz_problem(n1, n2, kappa):
    return ProblemSpec(n1, n2, 1.0 / (n2 + 1), kappa, lambda x, y: 1.0,
                       lambda x, y: true_solution_helmholtz(x, y, kappa), lambda x, y: 0.0, canned=1)


def helmholtz_bump_problem(n1, n2, kappa):
    def coef(x, y):
        h = 1.0 / (n2 + 1)
        cx, cy = 0.5 * (n1 + 1) * h, 0.5
        return 1.0 - 0.9 * np.exp(-64.0 * ((x - cx) ** 2 + (y - cy) ** 2))
    return ProblemSpec(n1, n2, 1.0 / (n2 + 1), kappa, coef,
                       lambda x, y: true_solution_helmholtz(x, y, kappa), lambda x, y: 0.0, canned=2)


@dataclass
class SparseSystem:
    """Assembled A u = f: CSR (Eigen RowMajor compressed form) + rhs."""
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    rhs: np.ndarray
    n1: int
    n2: int
    h: float

    def dim(self):
        return self.n1 * self.n2

    def node_index(self, i, j):
        return i * self.n2 + j

    def node_coords(self):
        i, j = np.divmod(np.arange(self.dim()), self.n2)
        return (i + 1) * self.h, (j + 1) * self.h

    def matvec(self, x):
        """A @ x for x of shape (N,) or (N, nrhs) (host, validation only)."""
        import scipy.sparse as sp
        a = sp.csr_matrix((self.values, self.col_idx, self.row_ptr), shape=(self.dim(), self.dim()))
        x = np.asarray(x, np.float64)
        return np.asarray(a @ x.reshape(self.dim(), -1)).reshape(x.shape)


def assemble_fd5(spec: ProblemSpec) -> SparseSystem:
    """Five-point assembly (problem.hpp:78-132), bit-identical to the reference."""
    n = spec.n1 * spec.n2
    rp = np.zeros(max(n, 0) + 1, np.int32)
    ci = np.zeros(max(5 * n, 1), np.int32)
    v = np.zeros(max(5 * n, 1), np.float64)
    rhs = np.zeros(max(n, 1), np.float64)
    nnz = ctypes.c_int64()
    if spec.canned is not None:
        st = lib().slablu_gpu_assemble_canned(int(spec.canned), int(spec.n1), int(spec.n2), float(spec.kappa),
                                              _p(rp), _p(ci), _p(v), _p(rhs), ctypes.byref(nnz))
    else:
        errs = []

        def wrap(fn):
            def cb(x, y, _u):
                try:
                    return float(fn(x, y))
                except Exception as e:  # surfaced after the call
                    errs.append(e)
                    return float("nan")
            return _lib.FIELD_FN(cb)
        cbs = [wrap(spec.coefficient_field), wrap(spec.dirichlet_data), wrap(spec.body_load)]
        st = lib().slablu_gpu_assemble_fd5(int(spec.n1), int(spec.n2), float(spec.h), float(spec.kappa),
                                           cbs[0], cbs[1], cbs[2], None, _p(rp), _p(ci), _p(v), _p(rhs),
                                           ctypes.byref(nnz))
        if errs:
            raise errs[0]
    _check(st)
    k = nnz.value
    return SparseSystem(rp, ci[:k].copy(), v[:k].copy(), rhs[:n].copy(), int(spec.n1), int(spec.n2), float(spec.h))


def sample_field(system: SparseSystem, fn: ScalarField) -> np.ndarray:
    x, y = system.node_coords()
    return np.array([fn(a, b) for a, b in zip(x, y)], np.float64)


def sample_solution(kind, n1, n2, kappa=0.0):
    out = np.zeros(n1 * n2)
    _check(lib().slablu_gpu_sample_solution(int(kind), int(n1), int(n2), float(kappa), _p(out)))
    return out


def gaussian_matrix(rows, cols, seed):
    """mt19937_64 + normal_distribution (common.hpp:72-79), column major."""
    out = np.empty((cols, rows), np.float64)
    lib().slablu_gpu_gaussian_matrix(int(rows), int(cols), int(seed), _p(out))
    return out.T


@dataclass
class ErrorReport:
    relerr_res: float = 0.0
    relerr_true: float = 0.0
    n_rhs: int = 0
    residual_norm_is_absolute: bool = False
    solution_norm_is_absolute: bool = False


def error_report(system, u_calc, u_true, f=None, device=0) -> ErrorReport:
    """problem.hpp:160-196, computed on the GPU (slablu_gpu_error_report: CSR SpMV residual and
    norms with a fixed-order reduction)."""
    n = system.dim()
    if np.shape(u_calc)[0] != n or np.shape(u_true)[0] != n or (f is not None and np.shape(f)[0] != n):
        raise Error("error_report: vector length must equal system dimension")
    u_calc = np.asfortranarray(np.asarray(u_calc, np.float64).reshape(n, -1))
    u_true = np.asfortranarray(np.asarray(u_true, np.float64).reshape(n, -1))
    f = system.rhs.reshape(n, -1) if f is None else np.asarray(f, np.float64).reshape(n, -1)
    f = np.asfortranarray(f)
    if u_calc.shape != u_true.shape or u_calc.shape[1] != f.shape[1] or u_calc.shape[1] < 1:
        raise Error("error_report: column counts must agree")
    out = np.zeros(4)
    rp = np.ascontiguousarray(system.row_ptr, np.int32)
    ci = np.ascontiguousarray(system.col_idx, np.int32)
    v = np.ascontiguousarray(system.values, np.float64)
    _check(lib().slablu_gpu_error_report(n, _p(rp), _p(ci), _p(v), _p(f), _p(u_calc), _p(u_true), u_calc.shape[1],
                                         int(device), _p(out)))
    return ErrorReport(relerr_res=float(out[0]), relerr_true=float(out[1]), n_rhs=u_calc.shape[1],
                       residual_norm_is_absolute=bool(out[2]), solution_norm_is_absolute=bool(out[3]))


def assemble_canned_device(kind, n1, n2, kappa=0.0, device=0):
    """On-device assembly of a canned problem (problem.hpp:210-261 through assemble_fd5 :78-132):
    returns torch CUDA tensors (row_ptr, col_idx, values, rhs)."""
    import torch
    dev = torch.device("cuda", device)
    n = int(n1) * int(n2)
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ci = torch.empty(5 * n, dtype=torch.int32, device=dev)
    v = torch.empty(5 * n, dtype=torch.float64, device=dev)
    rhs = torch.empty(n, dtype=torch.float64, device=dev)
    nnz = ctypes.c_int64()
    torch.cuda.current_stream(dev).synchronize()
    _check(lib().slablu_gpu_assemble_canned_device(int(kind), int(n1), int(n2), float(kappa), int(device), rp.data_ptr(),
                                                   ci.data_ptr(), v.data_ptr(), rhs.data_ptr(), ctypes.byref(nnz)))
    return rp, ci[:nnz.value], v[:nnz.value], rhs


def sample_solution_device(kind, n1, n2, kappa=0.0, device=0):
    import torch
    out = torch.empty(int(n1) * int(n2), dtype=torch.float64, device=torch.device("cuda", device))
    _check(lib().slablu_gpu_sample_solution_device(int(kind), int(n1), int(n2), float(kappa), int(device),
                                                   out.data_ptr()))
    return out


def error_report_device(n, row_ptr, col_idx, values, f, u, u_true=None, device=0) -> ErrorReport:
    """error_report on device tensors (f, u, u_true: (nrhs, n) or (n,) CUDA float64)."""
    nrhs = u.shape[0] if u.dim() == 2 else 1
    _torch_sync(u)
    out = np.zeros(4)
    _check(lib().slablu_gpu_error_report_device(int(n), row_ptr.data_ptr(), col_idx.data_ptr(), values.data_ptr(),
                                                f.data_ptr(), u.data_ptr(), None if u_true is None else u_true.data_ptr(),
                                                nrhs, int(device), _p(out)))
    return ErrorReport(relerr_res=float(out[0]), relerr_true=float(out[1]), n_rhs=nrhs,
                       residual_norm_is_absolute=bool(out[2]), solution_norm_is_absolute=bool(out[3]))


# ---------------------------------------------------------------------------
# configuration and geometry (driver.hpp:37-66, partition.hpp)
class CompressionChoice(enum.IntEnum):
    automatic = 0
    dense = 1
    hbs = 2


@dataclass
class SolverConfig:
    b: int = 0
    c: float = 0.6
    compression: CompressionChoice = CompressionChoice.automatic
    hbs_tol: float = 1e-11
    hbs_trunc_rel: float = 1e-13
    hbs_leaf_size: int = 64
    seed: int = 0
    threads: int = 1
    device: int = 0
    keep_T: bool = False
    refine: int = 1  # iterative-refinement steps per solve (GPU engine extension)

    def _c(self):
        return _lib.Config(int(self.b), float(self.c), int(self.compression), int(self.seed),
                           int(self.threads), int(self.device), int(bool(self.keep_T)), int(self.refine),
                           float(self.hbs_tol), float(self.hbs_trunc_rel), int(self.hbs_leaf_size))


def choose_b(n1, n2, config: SolverConfig = SolverConfig()):
    out = ctypes.c_int64()
    _check(lib().slablu_gpu_choose_b(int(n1), int(n2), int(config.b), float(config.c), ctypes.byref(out)))
    return out.value


@dataclass
class GridStrip:
    first_col: int
    width: int


@dataclass
class SlabPartition:
    n1: int
    n2: int
    b: int
    interfaces: List[GridStrip]
    interiors: List[GridStrip]

    def interface_count(self):
        return len(self.interfaces)

    def interior_count(self):
        return len(self.interiors)

    def dim(self):
        return self.n1 * self.n2

    def interface_offset(self, j):
        return self.interfaces[j].first_col * self.n2

    def interior_offset(self, i):
        return self.interiors[i].first_col * self.n2

    def interior_size(self, i):
        return self.interiors[i].width * self.n2

    def left_interior(self, j):
        return j

    def right_interior(self, j):
        return j + 1 if j + 1 < self.interior_count() else -1


def partition(n1, n2, b) -> SlabPartition:
    cap = max(int(n1) + 2, 4)
    ints = np.zeros(2 * cap, np.int64)
    ifcs = np.zeros(2 * cap, np.int64)
    ni, nf = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().slablu_gpu_partition(int(n1), int(n2), int(b), ctypes.byref(ni), _p(ints), ctypes.byref(nf),
                                      _p(ifcs), cap))
    return SlabPartition(int(n1), int(n2), int(b),
                         [GridStrip(int(ifcs[2 * k]), int(ifcs[2 * k + 1])) for k in range(nf.value)],
                         [GridStrip(int(ints[2 * k]), int(ints[2 * k + 1])) for k in range(ni.value)])


# ---------------------------------------------------------------------------
# factorize / solve (driver.hpp:72-179)
class Factorization:
    """Immutable two-stage factorization held on the GPU."""

    def __init__(self, handle, config):
        self._h = ctypes.c_void_p(handle)
        st = _lib.Stats()
        _check(lib().slablu_gpu_stats(self._h, ctypes.byref(st)))
        self.n1, self.n2, self.b = int(st.n1), int(st.n2), int(st.b)
        self.config = SolverConfig(**{**config.__dict__, "b": int(st.b),
                                      "compression": CompressionChoice(int(st.compression) or 1)})
        self.t_stage1, self.t_stage2 = float(st.t_stage1), float(st.t_stage2)
        self.storage_stage1, self.storage_stage2 = int(st.storage_stage1), int(st.storage_stage2)
        self.hbs_max_rank = int(st.hbs_max_rank)
        self.stats = st
        self.part = None if st.single_slab else partition(self.n1, self.n2, self.b)

    def single_slab(self):
        return bool(self.stats.single_slab)

    def storage_scalars(self):
        return self.storage_stage1 + self.storage_stage2

    def refresh_stats(self):
        st = _lib.Stats()
        _check(lib().slablu_gpu_stats(self._h, ctypes.byref(st)))
        self.stats = st
        return st

    def save(self, path):
        """Versioned binary file (SLBGPU01) of the whole factorization; see load()."""
        _check(lib().slablu_gpu_save(self._h, str(path).encode()))

    def export_sweep(self, path):
        """Stage two in the reference's SweepFactorization layout (SLBSWP01, stage_two.hpp:200-232)."""
        _check(lib().slablu_gpu_export_sweep(self._h, str(path).encode()))

    def set_refine(self, refine):
        """Iterative-refinement steps of later solves (needs the operator kept: factorize with
        refine > 0 to be able to raise it again)."""
        _check(lib().slablu_gpu_set_refine(self._h, int(refine)))
        self.config.refine = int(refine)

    def T_block(self, which, j):
        n2 = self.n2
        out = np.empty((n2, n2), order="F")
        _check(lib().slablu_gpu_T_block(self._h, {"diag": 0, "super": 1, "sub": 2}[which], int(j), _p(out)))
        return out

    def reduce_rhs(self, f):
        n = self.n1 * self.n2
        f = np.asfortranarray(np.asarray(f, np.float64).reshape(n, -1))
        k = self.stats.interfaces
        out = np.empty((k * self.n2, f.shape[1]), order="F")
        _check(lib().slablu_gpu_reduce_rhs(self._h, _p(f), f.shape[1], _p(out)))
        return out

    def sweep_solve(self, red):
        """Staged sweep solve (stage_two.hpp:170-188): interface values u_ifc (k*n2 x nrhs) from
        the reduced right-hand side."""
        red = np.asfortranarray(np.asarray(red, np.float64).reshape(self.stats.interfaces * self.n2, -1))
        out = np.empty_like(red, order="F")
        _check(lib().slablu_gpu_sweep_solve(self._h, _p(red), red.shape[1], _p(out)))
        return out

    def recover(self, f, u_ifc):
        """Staged recover_interiors (stage_one.hpp:438-462): the full solution (N x nrhs) from f and
        the interface values."""
        n = self.n1 * self.n2
        f = np.asfortranarray(np.asarray(f, np.float64).reshape(n, -1))
        u_ifc = np.asfortranarray(np.asarray(u_ifc, np.float64).reshape(-1, f.shape[1]))
        out = np.empty_like(f, order="F")
        _check(lib().slablu_gpu_recover(self._h, _p(f), _p(u_ifc), f.shape[1], _p(out)))
        return out

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().slablu_gpu_destroy(self._h)
            self._h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def factorize(system: SparseSystem, config: SolverConfig = SolverConfig()) -> Factorization:
    if system.dim() == 0:
        raise ConfigError("factorize: empty system")
    h = ctypes.c_void_p()
    cfg = config._c()
    rp = np.ascontiguousarray(system.row_ptr, np.int32)
    ci = np.ascontiguousarray(system.col_idx, np.int32)
    v = np.ascontiguousarray(system.values, np.float64)
    _check(lib().slablu_gpu_factorize(system.n1, system.n2, _p(rp), _p(ci), _p(v), ctypes.byref(cfg),
                                      ctypes.byref(h)))
    return Factorization(h.value, config)


class BlockTridiagonal:
    """stage_two.hpp:31-121: k diagonal blocks, k-1 sub (row j+1, col j) and super blocks, m x m."""

    def __init__(self, diag, sup, sub):
        self.diag, self.super, self.sub = list(diag), list(sup), list(sub)

    def block_count(self):
        return len(self.diag)

    def block_dim(self):
        return 0 if not self.diag else self.diag[0].shape[0]

    def to_dense(self):
        k, m = self.block_count(), self.block_dim()
        a = np.zeros((k * m, k * m))
        for j in range(k):
            a[j * m:(j + 1) * m, j * m:(j + 1) * m] = self.diag[j]
        for j in range(k - 1):
            a[j * m:(j + 1) * m, (j + 1) * m:(j + 2) * m] = self.super[j]
            a[(j + 1) * m:(j + 2) * m, j * m:(j + 1) * m] = self.sub[j]
        return a


class SweepFactorization:
    """stage_two.hpp:126-232 on the GPU: LU factors of the sweep's S_j (slablu_gpu_sweep_build)."""

    def __init__(self, t: BlockTridiagonal, device=0):
        k = t.block_count()
        if k == 0:
            raise ConfigError("BlockTridiagonal: no blocks")
        m = t.block_dim()
        if len(t.super) != k - 1 or len(t.sub) != k - 1:
            raise ConfigError("BlockTridiagonal: off-diagonal count must be k - 1")
        for blk in t.diag + t.super + t.sub:
            if np.shape(blk) != (m, m):
                raise ConfigError("BlockTridiagonal: inconsistent block dimensions")
        blocks = np.concatenate([np.asfortranarray(b, np.float64).ravel(order="F") for b in t.diag + t.super + t.sub])
        h = ctypes.c_void_p()
        _check(lib().slablu_gpu_sweep_build(int(m), int(k), _p(blocks), int(device), ctypes.byref(h)))
        self._h = h
        self.k, self.m = k, m
        st = _lib.Stats()
        _check(lib().slablu_gpu_stats(self._h, ctypes.byref(st)))
        self.stats = st

    def storage_scalars(self):
        return int(self.stats.storage_stage2)

    def solve(self, f):
        f = np.asfortranarray(np.asarray(f, np.float64).reshape(self.k * self.m, -1))
        out = np.empty_like(f, order="F")
        _check(lib().slablu_gpu_sweep_solve(self._h, _p(f), f.shape[1], _p(out)))
        return out

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().slablu_gpu_destroy(self._h)
            self._h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load(path, device=0, config: Optional[SolverConfig] = None) -> Factorization:
    """A factorization saved by Factorization.save (another process, same or another GPU)."""
    h = ctypes.c_void_p()
    _check(lib().slablu_gpu_load(str(path).encode(), int(device), ctypes.byref(h)))
    st = _lib.Stats()
    _check(lib().slablu_gpu_stats(h, ctypes.byref(st)))
    cfg = config or SolverConfig(b=int(st.b), device=int(device))
    return Factorization(h.value, cfg)


def import_sweep(path, device=0) -> "SweepFactorization":
    """SweepFactorization::deserialize (SLBSWP01) onto the GPU; solve with .solve(f)."""
    h = ctypes.c_void_p()
    _check(lib().slablu_gpu_import_sweep(str(path).encode(), int(device), ctypes.byref(h)))
    obj = SweepFactorization.__new__(SweepFactorization)
    obj._h = h
    st = _lib.Stats()
    _check(lib().slablu_gpu_stats(h, ctypes.byref(st)))
    obj.stats, obj.k, obj.m = st, int(st.interfaces), int(st.n2)
    return obj


def sweep_build(t: BlockTridiagonal, device=0) -> SweepFactorization:
    """stage_two.hpp:241-243."""
    return SweepFactorization(t, device)


def _torch_sync(t):
    """The engine runs on its own stream: work queued on torch's current stream that produces
    an input (copies, kernels, NCCL receives) must be complete before the engine reads it."""
    import torch
    if t.is_cuda:
        torch.cuda.current_stream(t.device).synchronize()


def factorize_device(n1, n2, row_ptr, col_idx, values, config: SolverConfig = SolverConfig()) -> Factorization:
    """CSR already resident on the GPU (torch CUDA tensors int32/int32/float64)."""
    _torch_sync(values)
    h = ctypes.c_void_p()
    cfg = config._c()
    _check(lib().slablu_gpu_factorize_device(int(n1), int(n2), int(values.numel()), row_ptr.data_ptr(),
                                             col_idx.data_ptr(), values.data_ptr(), ctypes.byref(cfg),
                                             ctypes.byref(h)))
    return Factorization(h.value, config)


def solve(fact: Factorization, f) -> np.ndarray:
    """u = A^{-1} f for host f of shape (N,) or (N, nrhs); returns (N, nrhs)."""
    n = fact.n1 * fact.n2
    f = np.asarray(f, np.float64)
    if f.shape[0] != n:
        raise Error("solve: rhs length must equal the grid size")
    f2 = np.asfortranarray(f.reshape(n, -1))
    u = np.empty_like(f2, order="F")
    _check(lib().slablu_gpu_solve(fact._h, _p(f2), n, f2.shape[1], _p(u), n))
    return u


def solve_device(fact: Factorization, f, u):
    """Device-resident solve: f, u are torch CUDA float64 tensors of shape (nrhs, N) (column-major N x nrhs)."""
    n = fact.n1 * fact.n2
    nrhs = f.shape[0] if f.dim() == 2 else 1
    _torch_sync(f)
    _check(lib().slablu_gpu_solve_device(fact._h, f.data_ptr(), n, nrhs, u.data_ptr(), n))
    return u


def run_problem(spec: ProblemSpec, config: SolverConfig = SolverConfig()):
    """driver.hpp:268-292: assemble, factorize, solve, error report (GPU times)."""
    import time
    system = assemble_fd5(spec)
    fact = factorize(system, config)
    t0 = time.perf_counter()
    u = solve(fact, system.rhs)
    t_solve = time.perf_counter() - t0
    u_true = (sample_solution(spec.canned, spec.n1, spec.n2, spec.kappa) if spec.canned is not None
              else sample_field(system, spec.dirichlet_data))
    rep = error_report(system, u, u_true)
    return {"N": system.dim(), "n1": spec.n1, "n2": spec.n2, "b": fact.b, "kappa": spec.kappa,
            "T_factor_stage1_s": fact.t_stage1, "T_factor_stage2_s": fact.t_stage2, "T_solve_s": t_solve,
            "M_factor_scalars": fact.storage_scalars(), "relerr_res": rep.relerr_res,
            "relerr_true": rep.relerr_true, "hbs_max_rank": fact.hbs_max_rank, "seed": config.seed}


# ---------------------------------------------------------------------------
# randomized HBS compression of a dense operator (hbs_compress.hpp:186-311)
@dataclass
class CompressOptions:
    tol: float = 1e-10
    trunc_rel: float = 1e-12
    seed: int = 0


@dataclass
class CompressStats:
    products_normal: int = 0
    products_adjoint: int = 0
    rounds: int = 0
    final_rank: int = 0
    residual_estimate: float = 0.0


def _hbs(m, leaf_size, r_start, r_max, adaptive, options, device):
    m = np.asfortranarray(np.asarray(m, dtype=np.float64))
    n = m.shape[0]
    if m.ndim != 2 or m.shape[1] != n:
        raise ConfigError("hbs_compress: square operator required")
    out = np.zeros((n, n), dtype=np.float64, order="F")
    st = _lib.HbsStatsT()
    _check(lib().slablu_gpu_hbs_compress(n, _p(m), int(leaf_size), int(r_start), int(r_max), int(adaptive),
                                          float(options.tol), float(options.trunc_rel), int(options.seed),
                                          int(device), _p(out), ctypes.byref(st)))
    return out, CompressStats(int(st.products_normal), int(st.products_adjoint), int(st.rounds),
                              int(st.final_rank), float(st.residual_estimate))


def hbs_compress(m, leaf_size, rank_bound, options: CompressOptions = CompressOptions(), device=0):
    """hbs_compress (hbs_compress.hpp:211-250) of the dense operator m with the dense sampler
    (test_hbs.cpp:64-68), on the GPU.  Returns (to_dense of the compressed operator, stats)."""
    return _hbs(m, leaf_size, 0, rank_bound, 0, options, device)


def hbs_compress_adaptive(m, leaf_size, r_start, r_max, options: CompressOptions = CompressOptions(), device=0):
    """hbs_compress_adaptive (hbs_compress.hpp:254-311) of the dense operator m, on the GPU."""
    return _hbs(m, leaf_size, r_start, r_max, 1, options, device)
