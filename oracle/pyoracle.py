"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes driver for the CPU restatement (oracle/build/liboracle.so). Imported only by tests/,
__graft_entry__.smoke(), tools/make_goldens.py and bench.py's CPU legs — never by the
product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")

METHODS = {"ddelm": 0, "ddelm-cs": 1, "ddelm-nn": 2}


class _Config(C.Structure):
    _fields_ = [
        ("problem", C.c_char_p),
        ("s", C.c_int), ("n_grid", C.c_int), ("M", C.c_int),
        ("l", C.c_double),
        ("seed", C.c_ulonglong),
        ("method", C.c_int),
        ("theta", C.c_double),
        ("flux_variant", C.c_int),
        ("change_of_variables", C.c_int),
        ("cg_rel_tol", C.c_double),
        ("cg_max_iter", C.c_int), ("cg_stop_after", C.c_int),
        ("workers", C.c_int), ("cg_workers", C.c_int),
        ("debug_flip_flux_row", C.c_int),
        ("layers_only", C.c_int),
        ("alpha", C.c_double),
        ("forcing_seed", C.c_ulonglong), ("rho_seed", C.c_ulonglong),
    ]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.ddo_create.restype = C.c_void_p
        L.ddo_create.argtypes = [C.POINTER(_Config), C.c_char_p, C.c_int]
        L.ddo_destroy.argtypes = [C.c_void_p]
        L.ddo_solve.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                C.c_char_p, C.c_int]
        for name in ("ddo_info", "ddo_timings", "ddo_residuals", "ddo_mu", "ddo_coeffs",
                     "ddo_ranks", "ddo_layer", "ddo_local", "ddo_kbar", "ddo_field",
                     "ddo_field_of", "ddo_errors", "ddo_apply_cs", "ddo_apply_reduced", "ddo_dense", "ddo_apply_p",
                     "ddo_random_matrix", "ddo_lsfactor", "ddo_cod_pinv", "ddo_set_lapack"):
            getattr(L, name).argtypes = None  # variadic pointer args, set per call
        L.ddo_tanh_record.argtypes = [C.c_int]
        L.ddo_tanh_recorded.argtypes = [C.c_void_p]
        L.ddo_tanh_recorded.restype = C.c_longlong
        L.ddo_tanh_table.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong]
        L.ddo_tanh_misses.restype = C.c_longlong
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class OracleResult:
    iterations: int
    converged: bool
    negative_curvature: bool
    residual_history: np.ndarray
    mu: np.ndarray
    coeffs: np.ndarray          # (N, M)
    ranks: np.ndarray           # (N,)
    ranks_bar: np.ndarray       # (N,) or -1
    qr_ratio: np.ndarray        # (N, 2)
    timings: dict
    n_delta: int
    n_pi: int


class OracleWorkspace:
    """Workspace + solve through the restatement (runner.cpp:126-155 semantics)."""

    def __init__(self, problem="poisson_sinpi", s=2, n_grid=10, M=64, l=8.0, seed=1,
                 flux_variant="mean_edge", trace_basis="change_of_variables", workers=1,
                 cg_workers=1, debug_flip_flux_row=-1, layers_only=False, alpha=32.0, forcing_seed=2,
                 rho_seed=3):
        L = lib()
        self._cfg = _Config(problem.encode(), s, n_grid, M, float(l), seed, 2, 0.999,
                            1 if flux_variant == "mean_edge" else 0,
                            1 if trace_basis == "change_of_variables" else 0,
                            1e-9, 0, 0, workers, cg_workers, debug_flip_flux_row,
                            1 if layers_only else 0, float(alpha), forcing_seed, rho_seed)
        err = C.create_string_buffer(512)
        self.h = L.ddo_create(C.byref(self._cfg), err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.s, self.M = s, M

    def __del__(self):
        if getattr(self, "h", None):
            lib().ddo_destroy(C.c_void_p(self.h))
            self.h = None

    def info(self):
        a = np.zeros(11, dtype=np.int32)
        lib().ddo_info(C.c_void_p(self.h), _p(a))
        return a

    def solve(self, method="ddelm-nn", theta=0.999, rel_tol=1e-9, max_iter=0, stop_after=0):
        err = C.create_string_buffer(512)
        rc = lib().ddo_solve(C.c_void_p(self.h), METHODS[method], C.c_double(theta),
                             C.c_double(rel_tol), max_iter, stop_after, err, 512)
        if rc == 2:
            raise ValueError(err.value.decode())
        if rc != 0:
            raise RuntimeError(err.value.decode())
        return self.result()

    def result(self) -> OracleResult:
        L, h = lib(), C.c_void_p(self.h)
        info = self.info()
        N, nd, npi, nmu, M = (int(x) for x in info[:5])
        res = np.zeros(int(info[9]))
        L.ddo_residuals(h, _p(res))
        mu = np.zeros(nmu)
        L.ddo_mu(h, _p(mu))
        co = np.zeros((N, M))
        L.ddo_coeffs(h, _p(co))
        rk = np.zeros(N, dtype=np.int32)
        rkb = np.zeros(N, dtype=np.int32)
        qr = np.zeros((N, 2))
        L.ddo_ranks(h, _p(rk), _p(rkb), _p(qr))
        t = np.zeros(6)
        L.ddo_timings(h, _p(t))
        tim = dict(zip(["assembly", "factorization", "setup", "cg", "reconstruction", "build"], t))
        return OracleResult(int(info[6]), bool(info[7]), bool(info[8]), res, mu, co, rk, rkb, qr,
                            tim, nd, npi)

    def layer(self, i):
        M = self.M
        w0, w1, b = np.zeros(M), np.zeros(M), np.zeros(M)
        lib().ddo_layer(C.c_void_p(self.h), C.c_int(i), _p(w0), _p(w1), _p(b))
        return w0, w1, b

    def local(self, i):
        rows = int(self.info()[5])
        K = np.zeros((self.M, rows))  # column-major (rows x M) -> read as (M, rows) then .T
        f = np.zeros(rows)
        lib().ddo_local(C.c_void_p(self.h), C.c_int(i), _p(K), _p(f))
        return K.T.copy(), f

    def kbar(self, i):
        rows = int(self.info()[5])
        K = np.zeros((self.M, rows))
        rc = lib().ddo_kbar(C.c_void_p(self.h), C.c_int(i), _p(K))
        if rc:
            raise RuntimeError("Neumann layer not built")
        return K.T.copy()

    def field(self, n=257, coeffs=None):
        u, gx, gy = np.zeros(n * n), np.zeros(n * n), np.zeros(n * n)
        if coeffs is None:
            lib().ddo_field(C.c_void_p(self.h), C.c_int(n), _p(u), _p(gx), _p(gy))
        else:
            c = np.ascontiguousarray(coeffs, dtype=np.float64)
            lib().ddo_field_of(C.c_void_p(self.h), _p(c), C.c_int(n), _p(u), _p(gx), _p(gy))
        return u, gx, gy

    def apply_cs(self, v, theta=0.999):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros_like(v)
        lib().ddo_apply_cs(C.c_void_p(self.h), C.c_double(theta), _p(v), _p(out))
        return out

    def apply_p(self, v, transpose=False):
        """apply_P / apply_PT (solvers.cpp:450-474)."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros_like(v)
        lib().ddo_apply_p(C.c_void_p(self.h), C.c_int(1 if transpose else 0), _p(v), _p(out))
        return out

    def apply_reduced(self, v):
        """reduced_apply (solvers.cpp:262-274) on mu = [mu_Delta; mu_Pi]."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros_like(v)
        lib().ddo_apply_reduced(C.c_void_p(self.h), _p(v), _p(out))
        return out

    def dense(self, method="ddelm-nn", theta=0.999):
        """dense_oracle_solve (solvers.cpp:609-709): (reduced_op, reduced_rhs, mu_full, coeffs)."""
        info = self.info()
        N, nd, npi, nmu, M = (int(x) for x in info[:5])
        dim = nmu if method == "ddelm" else nd
        op, rhs, mu, co = np.zeros(dim * dim), np.zeros(dim), np.zeros(nmu), np.zeros((N, M))
        d = C.c_int()
        rc = lib().ddo_dense(C.c_void_p(self.h), METHODS[method], C.c_double(theta), C.byref(d), _p(op),
                             _p(rhs), _p(mu), _p(co))
        if rc:
            raise ValueError("dense_oracle_solve: system too large for the dense path")
        return op.reshape(dim, dim).T.copy(), rhs, mu, co

    def errors(self, n=257):
        l2, h1 = C.c_double(), C.c_double()
        rc = lib().ddo_errors(C.c_void_p(self.h), C.c_int(n), C.byref(l2), C.byref(h1))
        if rc:
            raise RuntimeError("problem has no exact solution")
        return l2.value, h1.value


def scipy_lapack_path() -> str:
    """SciPy's bundled OpenBLAS/LAPACK (symbols scipy_d*_)."""
    import glob

    import scipy
    libs = glob.glob(os.path.join(os.path.dirname(scipy.__file__), "..", "scipy.libs", "libscipy_openblas*.so"))
    if not libs:
        raise RuntimeError("SciPy's libscipy_openblas not found")
    return os.path.abspath(sorted(libs)[0])


def use_lapack(on: bool = True) -> str | None:
    """Switch the oracle's LsFactor to LAPACK (dgeqrf / dgeqp3 / dtzrzf, lapack.cpp) — the CPU
    baseline mode — or back to the restatement the goldens were made with."""
    path = scipy_lapack_path() if on else None
    if lib().ddo_set_lapack(path.encode() if path else None) != 0:
        raise RuntimeError("ddo_set_lapack failed")
    return path


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """The reference tests' seeded N(0,1) matrix (test_solvers.cpp:14-21), bit-exact."""
    out = np.zeros((cols, rows))
    lib().ddo_random_matrix(C.c_int(rows), C.c_int(cols), C.c_ulonglong(seed), _p(out))
    return out.T.copy()


def lsfactor(K: np.ndarray, tol: float = 1e-10):
    """Oracle LsFactor (solvers.cpp:24-45): (rank, deficient, pinv n x m, Q m x n zero-padded)."""
    K = np.asarray(K, dtype=np.float64)
    m, n = K.shape
    Kf = np.ascontiguousarray(K.T)
    rank, dfc = C.c_int(), C.c_int()
    pinv = np.zeros((m, n))  # column-major n x m
    Q = np.zeros((n, m))     # column-major m x n
    rc = lib().ddo_lsfactor(_p(Kf), C.c_int(m), C.c_int(n), C.c_double(tol), C.byref(rank), C.byref(dfc),
                            _p(pinv), _p(Q))
    if rc != 0:
        raise RuntimeError("ddo_lsfactor failed")
    return rank.value, bool(dfc.value), pinv.T.copy(), Q.T.copy()


def cod_pinv(K: np.ndarray) -> np.ndarray:
    """Eigen COD pseudo-inverse with the default threshold (the reference tests' svd_pinv)."""
    K = np.asarray(K, dtype=np.float64)
    m, n = K.shape
    Kf = np.ascontiguousarray(K.T)
    out = np.zeros((m, n))
    if lib().ddo_cod_pinv(_p(Kf), C.c_int(m), C.c_int(n), _p(out)) != 0:
        raise RuntimeError("ddo_cod_pinv failed")
    return out.T.copy()


def field_rel_l2(u_a: np.ndarray, u_b: np.ndarray, n: int) -> float:
    """Trapezoid-weighted relative L2 of (a - b) against b on the n x n grid
    (runner.cpp:269-281 field_diff, evaluated at n)."""
    w1 = np.full(n, 1.0 / (n - 1))
    w1[0] = w1[-1] = 0.5 / (n - 1)
    w = np.outer(w1, w1).ravel()
    d = u_a - u_b
    den = np.sum(w * u_b * u_b)
    num = np.sum(w * d * d)
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))


# ---- parity decomposition hooks (oracle/model.cpp feature_tanh; tools/parity_decomposition.py)
def tanh_record(on: bool) -> None:
    """Record every feature tanh argument of the next workspace builds (use workers=1)."""
    lib().ddo_tanh_record(1 if on else 0)


def tanh_recorded() -> np.ndarray:
    n = lib().ddo_tanh_recorded(None)
    out = np.empty(n)
    lib().ddo_tanh_recorded(_p(out))
    return out


def tanh_table(z: np.ndarray | None, t: np.ndarray | None = None) -> None:
    """Replace the feature tanh by t[k] at argument z[k] (bitwise key); None restores std::tanh."""
    if z is None:
        lib().ddo_tanh_table(None, None, 0)
        return
    z = np.ascontiguousarray(z, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    lib().ddo_tanh_table(_p(z), _p(t), z.size)


def tanh_misses() -> int:
    return int(lib().ddo_tanh_misses())
