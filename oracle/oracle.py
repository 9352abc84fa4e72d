"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the CPU oracle.

The oracle (oracle/slablu_oracle.cpp) restates the reference's dense-mode
factorize/solve path on the CPU.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs import this module; the
product package never does.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_slablu.so")
_lib = None

# problem kinds (inc/problem.hpp:210-261)
POISSON_LOG, HELMHOLTZ, HELMHOLTZ_BUMP = 0, 1, 2
# field selectors (oracle/slablu_oracle.cpp Coef / Dir)
COEF_ONE, COEF_BUMP, COEF_LINEAR_X2Y, COEF_NEG_ONE = 0, 1, 2, 3
DIR_ZERO, DIR_POISSON_LOG, DIR_HELMHOLTZ_J0, DIR_X_PLUS_Y = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code, msg, index):
        super().__init__(f"[{code}] {msg}")
        self.code, self.msg, self.index = code, msg, index


class ConfigError(OracleError):
    pass


class SingularMatrixError(OracleError):
    pass


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, D, I, Lg = ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_long
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_last_error_index.restype = Lg
        L.orc_bessel_j0.restype = D
        L.orc_bessel_j0.argtypes = [D]
        L.orc_true_solution_poisson.restype = D
        L.orc_true_solution_poisson.argtypes = [D, D]
        L.orc_true_solution_helmholtz.restype = D
        L.orc_true_solution_helmholtz.argtypes = [D, D, D]
        L.orc_kappa_from_ppw.argtypes = [D, Lg, P]
        L.orc_choose_b.argtypes = [Lg, Lg, Lg, D, P]
        L.orc_partition.argtypes = [Lg, Lg, Lg, P, P, P, P, Lg]
        L.orc_assemble.argtypes = [Lg, Lg, D, D, I, I, D, P]
        L.orc_assemble_canned.argtypes = [I, Lg, Lg, D, P]
        L.orc_system_from_csr.argtypes = [Lg, Lg, D, P, P, P, P, P]
        L.orc_system_free.argtypes = [P]
        L.orc_system_dim.argtypes = [P]
        L.orc_system_dim.restype = Lg
        L.orc_system_nnz.argtypes = [P]
        L.orc_system_nnz.restype = Lg
        L.orc_system_csr.argtypes = [P, P, P, P, P]
        L.orc_sample_dirichlet.argtypes = [I, Lg, Lg, D, P]
        L.orc_spmv.argtypes = [P, P, Lg, P]
        L.orc_factorize.argtypes = [P, Lg, D, I, Lg, I, P]
        L.orc_fact_free.argtypes = [P]
        L.orc_fact_stats.argtypes = [P, P, P]
        L.orc_fact_T_block.argtypes = [P, I, Lg, P]
        L.orc_solve.argtypes = [P, P, Lg, P]
        L.orc_reduce_rhs.argtypes = [P, P, Lg, P]
        L.orc_time_slab_sample.argtypes = [P, Lg, Lg, Lg, P, P]
        L.orc_time_sweep_step.argtypes = [Lg, P]
        L.orc_gaussian_matrix.argtypes = [Lg, Lg, ctypes.c_uint64, P]
        L.orc_slab_factor.argtypes = [P, Lg, Lg, P]
        L.orc_slab_free.argtypes = [P]
        L.orc_slab_info.argtypes = [P, P]
        L.orc_slab_contrib.argtypes = [P, P, Lg, P, P]
        L.orc_slab_T_columns.argtypes = [P, I, P, Lg, P, P]
        L.orc_slab_recover.argtypes = [P, P, P, Lg, P]
        L.orc_set_blas_threads.argtypes = [I]
        L.orc_get_blas_threads.restype = I
        _lib = L
    return _lib


def _check(code):
    if code == 0:
        return
    L = lib()
    msg = L.orc_last_error().decode()
    idx = L.orc_last_error_index()
    cls = {2: ConfigError, 3: SingularMatrixError}.get(code, OracleError)
    raise cls(code, msg, idx)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_blas_threads(t):
    lib().orc_set_blas_threads(int(t))


def bessel_j0(t):
    return lib().orc_bessel_j0(float(t))


def true_solution_poisson(x, y):
    return lib().orc_true_solution_poisson(float(x), float(y))


def true_solution_helmholtz(x, y, k):
    return lib().orc_true_solution_helmholtz(float(x), float(y), float(k))


def kappa_from_ppw(ppw, n2):
    out = ctypes.c_double()
    _check(lib().orc_kappa_from_ppw(float(ppw), int(n2), ctypes.byref(out)))
    return out.value


def choose_b(n1, n2, b=0, c=0.6):
    out = ctypes.c_long()
    _check(lib().orc_choose_b(int(n1), int(n2), int(b), float(c), ctypes.byref(out)))
    return out.value


def partition(n1, n2, b):
    cap = n1 + 2
    ic = np.zeros(2 * cap, np.int64)
    fc = np.zeros(2 * cap, np.int64)
    ni, nf = ctypes.c_long(), ctypes.c_long()
    _check(lib().orc_partition(int(n1), int(n2), int(b), ctypes.byref(ni), _ptr(ic), ctypes.byref(nf), _ptr(fc), cap))
    return ic[: 2 * ni.value].reshape(-1, 2), fc[: 2 * nf.value].reshape(-1, 2)


def gaussian_matrix(rows, cols, seed):
    out = np.empty((cols, rows), np.float64)
    lib().orc_gaussian_matrix(int(rows), int(cols), int(seed), _ptr(out))
    return out.T  # column-major data as an (rows x cols) F-ordered view


class System:
    def __init__(self, handle, n1, n2, h):
        self._h = ctypes.c_void_p(handle)
        self.n1, self.n2, self.h = n1, n2, h
        L = lib()
        n = L.orc_system_dim(self._h)
        nnz = L.orc_system_nnz(self._h)
        self.row_ptr = np.empty(n + 1, np.int32)
        self.col_idx = np.empty(nnz, np.int32)
        self.values = np.empty(nnz, np.float64)
        self.rhs = np.empty(n, np.float64)
        L.orc_system_csr(self._h, _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(self.values), _ptr(self.rhs))

    @property
    def dim(self):
        return self.n1 * self.n2

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            try:
                lib().orc_system_free(self._h)
            except Exception:
                pass
            self._h = None

    def dense(self):
        n = self.dim
        a = np.zeros((n, n))
        for r in range(n):
            for p in range(self.row_ptr[r], self.row_ptr[r + 1]):
                a[r, self.col_idx[p]] = self.values[p]
        return a

    def matvec(self, x):
        x = np.asfortranarray(np.asarray(x, np.float64).reshape(self.dim, -1))
        y = np.empty_like(x, order="F")
        lib().orc_spmv(self._h, _ptr(x), x.shape[1], _ptr(y))
        return y


def assemble(n1, n2, h, kappa=0.0, coef=COEF_ONE, dirichlet=DIR_ZERO, load=0.0):
    hdl = ctypes.c_void_p()
    _check(lib().orc_assemble(int(n1), int(n2), float(h), float(kappa), int(coef), int(dirichlet), float(load), ctypes.byref(hdl)))
    return System(hdl.value, n1, n2, h)


def assemble_canned(kind, n1, n2, kappa=0.0):
    hdl = ctypes.c_void_p()
    _check(lib().orc_assemble_canned(int(kind), int(n1), int(n2), float(kappa), ctypes.byref(hdl)))
    return System(hdl.value, n1, n2, 1.0 / (n2 + 1))


def system_from_csr(n1, n2, h, row_ptr, col_idx, values, rhs):
    hdl = ctypes.c_void_p()
    rp = np.ascontiguousarray(row_ptr, np.int32)
    ci = np.ascontiguousarray(col_idx, np.int32)
    v = np.ascontiguousarray(values, np.float64)
    r = np.ascontiguousarray(rhs, np.float64)
    _check(lib().orc_system_from_csr(int(n1), int(n2), float(h), _ptr(rp), _ptr(ci), _ptr(v), _ptr(r), ctypes.byref(hdl)))
    return System(hdl.value, n1, n2, h)


def sample_dirichlet(kind, n1, n2, kappa=0.0):
    out = np.empty(n1 * n2)
    _check(lib().orc_sample_dirichlet(int(kind), int(n1), int(n2), float(kappa), _ptr(out)))
    return out


class Factorization:
    def __init__(self, handle, system):
        self._h = ctypes.c_void_p(handle)
        self.system = system
        st = np.zeros(6, np.int64)
        tm = np.zeros(2)
        lib().orc_fact_stats(self._h, _ptr(st), _ptr(tm))
        self.b, self.k, self.strips, self.single_slab = int(st[0]), int(st[1]), int(st[2]), bool(st[3])
        self.storage_stage1, self.storage_stage2 = int(st[4]), int(st[5])
        self.t_stage1, self.t_stage2 = float(tm[0]), float(tm[1])

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().orc_fact_free(self._h)
            except Exception:
                pass
            self._h = None

    def solve(self, f):
        n = self.system.dim
        f = np.asfortranarray(np.asarray(f, np.float64).reshape(n, -1))
        u = np.empty_like(f, order="F")
        _check(lib().orc_solve(self._h, _ptr(f), f.shape[1], _ptr(u)))
        return u

    def reduce_rhs(self, f):
        n, n2 = self.system.dim, self.system.n2
        f = np.asfortranarray(np.asarray(f, np.float64).reshape(n, -1))
        out = np.empty((self.k * n2, f.shape[1]), order="F")
        _check(lib().orc_reduce_rhs(self._h, _ptr(f), f.shape[1], _ptr(out)))
        return out

    def T_block(self, which, j):
        """which: 'diag' | 'super' | 'sub' (reduced blocks before stage two)."""
        n2 = self.system.n2
        out = np.empty((n2, n2), order="F")
        _check(lib().orc_fact_T_block(self._h, {"diag": 0, "super": 1, "sub": 2}[which], int(j), _ptr(out)))
        return out


def factorize(system, b=0, c=0.6, threads=1, chunk=0, keep_T=False):
    hdl = ctypes.c_void_p()
    _check(lib().orc_factorize(system._h, int(b), float(c), int(threads), int(chunk), int(keep_T), ctypes.byref(hdl)))
    return Factorization(hdl.value, system)


class Slab:
    """One slab interior factored alone (factor_one_interior, inc/stage_one.hpp:163-238) and
    its per-slab stage-one / solve terms, for staged parity at sizes where the whole oracle
    factorization does not fit (tests only)."""

    def __init__(self, system, b, strip):
        hdl = ctypes.c_void_p()
        _check(lib().orc_slab_factor(system._h, int(b), int(strip), ctypes.byref(hdl)))
        self._h = ctypes.c_void_p(hdl.value)
        self.system = system
        info = np.zeros(4, np.int64)
        lib().orc_slab_info(self._h, _ptr(info))
        self.first_col, self.width, self.left_ifc, self.right_ifc = (int(v) for v in info)

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().orc_slab_free(self._h)
            except Exception:
                pass
            self._h = None

    def contrib(self, f):
        """(to_left A^-1 f_i, to_right A^-1 f_i), each n2 x nrhs (reduce_rhs :423-432)."""
        n, n2 = self.system.dim, self.system.n2
        f = np.asfortranarray(np.asarray(f, np.float64).reshape(n, -1))
        oL = np.empty((n2, f.shape[1]), order="F")
        oR = np.empty((n2, f.shape[1]), order="F")
        _check(lib().orc_slab_contrib(self._h, _ptr(f), f.shape[1], _ptr(oL), _ptr(oR)))
        return oL, oR

    def T_columns(self, side, cols):
        """(to_left, to_right) . A^-1 . from_side[:, cols] (side 'left' | 'right')."""
        n2 = self.system.n2
        c = np.ascontiguousarray(cols, np.int64)
        oL = np.empty((n2, c.size), order="F")
        oR = np.empty((n2, c.size), order="F")
        _check(lib().orc_slab_T_columns(self._h, 0 if side == "left" else 1, _ptr(c), c.size, _ptr(oL), _ptr(oR)))
        return oL, oR

    def recover(self, f, u_ifc):
        """A^-1 (f_i - from_L u_L - from_R u_R) in natural order ((width*n2) x nrhs)."""
        n, n2 = self.system.dim, self.system.n2
        f = np.asfortranarray(np.asarray(f, np.float64).reshape(n, -1))
        u_ifc = np.asfortranarray(np.asarray(u_ifc, np.float64).reshape(-1, f.shape[1]))
        out = np.empty((self.width * n2, f.shape[1]), order="F")
        _check(lib().orc_slab_recover(self._h, _ptr(f), _ptr(u_ifc), f.shape[1], _ptr(out)))
        return out


def time_slab_sample(system, b, strip, nrhs_sample):
    t1, t2 = ctypes.c_double(), ctypes.c_double()
    _check(lib().orc_time_slab_sample(system._h, int(b), int(strip), int(nrhs_sample), ctypes.byref(t1), ctypes.byref(t2)))
    return t1.value, t2.value


def time_sweep_step(m):
    t = ctypes.c_double()
    _check(lib().orc_time_sweep_step(int(m), ctypes.byref(t)))
    return t.value


def error_report(system, u, u_true, f=None):
    """inc/problem.hpp:160-190 (numpy restatement for tests)."""
    u = np.asarray(u).reshape(system.dim, -1)
    u_true = np.asarray(u_true).reshape(system.dim, -1)
    f = system.rhs.reshape(-1, 1) if f is None else np.asarray(f).reshape(system.dim, -1)
    res = np.linalg.norm(system.matvec(u) - f)
    fn = np.linalg.norm(f)
    err = np.linalg.norm(u - u_true)
    un = np.linalg.norm(u_true)
    return (res / fn if fn > 0 else res), (err / un if un > 0 else err)
