"""B200-native DDELM-NN hot path (arXiv 2503.10032): Python mirror of the reference solver API.

The reference's C++ surface (proj/include/ddelm/solvers.hpp) is

    Workspace(problem, s, n_grid, M, l, seed, SolverOptions)   solvers.hpp:79-80
    ddelm_cs_solve(ws, CgOptions) / ddelm_nn_solve(ws, theta, CgOptions)   solvers.hpp:178-181
    SolveReport{coeffs, mu, mu_delta, mu_pi, iterations, converged, residual_history, ...}

and this module exposes the same names over the C-ABI library libddelm_gpu.so
(include/ddelm_gpu.h). Errors follow the reference: std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError. There is no CPU fallback: without the built library or a
CUDA device every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from .configs import CONFIGS  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libddelm_gpu.so")

PROBLEMS = {"poisson_sinpi": 0, "poisson_sin2pi_exp": 1, "poisson_sin2pi_cos3pi_x2y": 2,
            "poisson_grf": 3, "varcoef_poisson": 4, "biharmonic_sinpi": 5}
METHODS = {"ddelm": 0, "ddelm-cs": 1, "ddelm-nn": 2}

DDELM_OK, DDELM_ERR_INVALID_ARGUMENT, DDELM_ERR_RUNTIME, DDELM_ERR_CUDA, DDELM_ERR_CAPACITY = range(5)

# every symbol declared in include/ddelm_gpu.h
EXPORTS = ("ddelm_gpu_last_error", "ddelm_gpu_version", "ddelm_gpu_create", "ddelm_gpu_build",
           "ddelm_gpu_build_coarse", "ddelm_gpu_build_neumann", "ddelm_gpu_solve",
           "ddelm_gpu_reseed", "ddelm_gpu_destroy", "ddelm_gpu_get_mu", "ddelm_gpu_get_coeffs",
           "ddelm_gpu_get_residuals", "ddelm_gpu_get_ranks", "ddelm_gpu_get_layer",
           "ddelm_gpu_get_local", "ddelm_gpu_apply_operator", "ddelm_gpu_invalidate",
           "ddelm_gpu_stream", "ddelm_gpu_set_profiling", "ddelm_gpu_get_kernel_stats",
           "ddelm_gpu_get_device_span_ms", "ddelm_gpu_get_phase_ms", "ddelm_gpu_get_launch_count",
           "ddelm_gpu_lsq_create", "ddelm_gpu_lsq_generate", "ddelm_gpu_lsq_factor",
           "ddelm_gpu_lsq_get_block", "ddelm_gpu_lsq_ld", "ddelm_gpu_lsq_destroy",
           "ddelm_gpu_nccl_unique_id", "ddelm_gpu_create_sharded", "ddelm_gpu_get_shard",
           "ddelm_gpu_plan_tables", "ddelm_gpu_sample_field", "ddelm_gpu_relative_errors",
           "ddelm_gpu_field_diff", "ddelm_gpu_apply_reduced", "ddelm_gpu_dense_oracle",
           "ddelm_gpu_apply_neumann", "ddelm_gpu_set_cg_blocks", "ddelm_gpu_create_sharded_host",
           "ddelm_gpu_exchange_lists", "ddelm_gpu_cg_driver", "ddelm_gpu_lsfactor_batch",
           "ddelm_gpu_fp64_peak", "ddelm_gpu_tanh")


class _Desc(C.Structure):
    _fields_ = [("problem", C.c_int), ("s", C.c_int), ("n_grid", C.c_int), ("M", C.c_int),
                ("l", C.c_double), ("seed", C.c_uint64), ("flux_variant", C.c_int),
                ("change_of_variables", C.c_int), ("rank_tol", C.c_double), ("device", C.c_int),
                ("debug_flip_flux_row", C.c_int), ("alpha", C.c_double),
                ("forcing_seed", C.c_uint64), ("rho_seed", C.c_uint64)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("negative_curvature", C.c_int),
                ("n_delta", C.c_int), ("n_pi", C.c_int), ("n_mu", C.c_int),
                ("n_subdomains", C.c_int), ("M", C.c_int),
                ("assembly_seconds", C.c_double), ("factorization_seconds", C.c_double),
                ("setup_seconds", C.c_double), ("cg_seconds", C.c_double),
                ("reconstruct_seconds", C.c_double), ("total_seconds", C.c_double)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load the C-ABI library (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `make -C paper_2503_10032_b200/csrc` "
                          "(the DDELM-NN path has no CPU fallback)")
    L = C.CDLL(path)
    L.ddelm_gpu_last_error.restype = C.c_char_p
    L.ddelm_gpu_version.restype = C.c_char_p
    L.ddelm_gpu_create.argtypes = [C.POINTER(_Desc), C.POINTER(C.c_void_p)]
    for fn in ("ddelm_gpu_build", "ddelm_gpu_build_coarse", "ddelm_gpu_build_neumann"):
        getattr(L, fn).argtypes = [C.c_void_p]
    L.ddelm_gpu_solve.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int,
                                  C.POINTER(_Report)]
    L.ddelm_gpu_reseed.argtypes = [C.c_void_p, C.c_uint64]
    L.ddelm_gpu_set_cg_blocks.argtypes = [C.c_void_p, C.c_int]
    L.ddelm_gpu_destroy.argtypes = [C.c_void_p]
    L.ddelm_gpu_get_mu.argtypes = [C.c_void_p, C.c_void_p]
    L.ddelm_gpu_get_coeffs.argtypes = [C.c_void_p, C.c_void_p]
    L.ddelm_gpu_get_residuals.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    L.ddelm_gpu_sample_field.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_relative_errors.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_field_diff.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_get_ranks.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_get_layer.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_get_local.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int)]
    L.ddelm_gpu_apply_operator.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_apply_reduced.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_invalidate.argtypes = [C.c_void_p]
    L.ddelm_gpu_apply_neumann.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_dense_oracle.argtypes = [C.c_void_p, C.c_int, C.c_double, C.POINTER(C.c_int), C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_stream.argtypes = [C.c_void_p]
    L.ddelm_gpu_stream.restype = C.c_void_p
    L.ddelm_gpu_set_profiling.argtypes = [C.c_void_p, C.c_int]
    L.ddelm_gpu_get_kernel_stats.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_double),
                                             C.POINTER(C.c_longlong), C.POINTER(C.c_double),
                                             C.POINTER(C.c_double)]
    L.ddelm_gpu_get_device_span_ms.argtypes = [C.c_void_p]
    L.ddelm_gpu_get_device_span_ms.restype = C.c_double
    L.ddelm_gpu_get_phase_ms.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    L.ddelm_gpu_get_launch_count.argtypes = [C.c_void_p]
    L.ddelm_gpu_get_launch_count.restype = C.c_longlong
    L.ddelm_gpu_lsq_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.ddelm_gpu_lsq_generate.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
    L.ddelm_gpu_lsq_factor.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ddelm_gpu_lsq_get_block.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_lsq_ld.argtypes = [C.c_void_p]
    L.ddelm_gpu_lsq_destroy.argtypes = [C.c_void_p]
    L.ddelm_gpu_nccl_unique_id.argtypes = [C.c_void_p]
    L.ddelm_gpu_create_sharded.argtypes = [C.POINTER(_Desc), C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
    L.ddelm_gpu_get_shard.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.ddelm_gpu_plan_tables.argtypes = [C.POINTER(_Desc), C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]
    L.ddelm_gpu_create_sharded_host.argtypes = [C.POINTER(_Desc), C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]
    L.ddelm_gpu_exchange_lists.argtypes = [C.POINTER(_Desc), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_void_p, C.c_int]
    L.ddelm_gpu_lsfactor_batch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_double,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddelm_gpu_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.ddelm_gpu_tanh.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_longlong]
    L.ddelm_gpu_cg_driver.argtypes = [C.c_void_p]
    L.ddelm_gpu_cg_driver.restype = C.c_char_p
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == DDELM_OK:
        return
    msg = load_library().ddelm_gpu_last_error().decode()
    if rc == DDELM_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(f"[ddelm_gpu rc={rc}] {msg}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class ProblemParams:
    """ProblemParams (problems.hpp:64-68): GRF smoothness and seeds."""
    alpha: float = 32.0
    forcing_seed: int = 2
    rho_seed: int = 3


@dataclass
class ProblemSpec:
    """make_problem (problems.cpp:132-188) — the Poisson-kind problems on the device path."""
    name: str
    params: ProblemParams = field(default_factory=ProblemParams)

    def __post_init__(self):
        if self.name not in PROBLEMS:
            raise ValueError(f"make_problem: unknown problem '{self.name}'")
        if not self.params.alpha > 0:
            raise ValueError("sample_grf: alpha must be positive")


def make_problem(name: str, params: ProblemParams | None = None) -> ProblemSpec:
    return ProblemSpec(name, params or ProblemParams())


@dataclass
class SolverOptions:
    """SolverOptions (solvers.hpp:49-58)."""
    flux_variant: str = "pointwise"      # pointwise | mean_edge
    change_of_variables: bool = False
    rank_tol: float = 1e-10
    workers: int = 1                     # accepted for API parity; the device batches subdomains
    debug_flip_flux_row: int = -1


@dataclass
class CgOptions:
    """CgOptions (solvers.hpp:173-176)."""
    rel_tol: float = 1e-9
    max_iter: int = 0


@dataclass
class SolveReport:
    """SolveReport (solvers.hpp:162-171)."""
    coeffs: np.ndarray
    mu: np.ndarray
    mu_delta: np.ndarray
    mu_pi: np.ndarray
    iterations: int
    converged: bool
    negative_curvature: bool
    residual_history: np.ndarray
    setup_seconds: float = 0.0
    cg_seconds: float = 0.0
    reconstruct_seconds: float = 0.0
    assembly_seconds: float = 0.0
    factorization_seconds: float = 0.0
    total_seconds: float = 0.0
    phase_ms: dict = field(default_factory=dict)
    launches: int = 0


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for a sharded workspace (rank 0 creates it, the caller broadcasts it)."""
    buf = (C.c_ubyte * 128)()
    _check(load_library().ddelm_gpu_nccl_unique_id(buf))
    return bytes(buf)


def _cfg_desc(cfg) -> _Desc:
    return _Desc(PROBLEMS[cfg["problem"]], cfg["s"], cfg["n_grid"], cfg["M"], float(cfg["l"]), cfg["seed"],
                 1 if cfg["flux_variant"] == "mean_edge" else 0,
                 1 if cfg["trace_basis"] == "change_of_variables" else 0, 1e-10, 0, -1,
                 float(cfg.get("alpha", 32.0)), int(cfg.get("forcing_seed", 2)), int(cfg.get("rho_seed", 3)))


# exchange points / tables of the sharded iteration (plan.hpp XPoint / XTable)
XPOINTS = ("op1", "op2", "nn1", "nn2", "op3", "op4")
XTABLES = ("t", "psi", "t3", "o", "x", "tr", "zz", "xc", "opi", "pap")


def device_tanh(x: np.ndarray, device: int = 0) -> np.ndarray:
    """tanh with the feature builder's device tanh (ddelm_gpu_tanh; parity-decomposition hook)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    _check(load_library().ddelm_gpu_tanh(device, _ptr(x), _ptr(y), x.size))
    return y


def fp64_peak(device: int = 0) -> float:
    """Measured FP64 tensor-pipe TFLOP/s of this B200 (DMMA loop; ddelm_gpu_fp64_peak)."""
    t = C.c_double()
    _check(load_library().ddelm_gpu_fp64_peak(device, C.byref(t)))
    return t.value


def exchange_lists(cfg, rank: int, world: int, one_level: bool = False) -> dict:
    """Host-side exchange plan of one rank (no GPU needed): per point, the (table, slot) entries
    it sends / receives and the per-peer counts (plan.cpp build_exchange_plan)."""
    L = load_library()
    d = _cfg_desc(cfg)

    def get(pt, which):
        n = L.ddelm_gpu_exchange_lists(C.byref(d), rank, world, int(one_level), pt, which, None, 0)
        if n < 0:
            _check(-n)
        a = np.zeros(max(n, 1), dtype=np.int32)
        L.ddelm_gpu_exchange_lists(C.byref(d), rank, world, int(one_level), pt, which, _ptr(a), n)
        return a[:n]

    out = {}
    for pt, name in enumerate(XPOINTS):
        out[name] = {"send": get(pt, 0).reshape(-1, 2), "recv": get(pt, 1).reshape(-1, 2),
                     "scnt": get(pt, 2), "rcnt": get(pt, 3), "soff": get(pt, 4)}
    out["max_msg"] = int(get(0, 5)[0])
    return out


@dataclass
class LsFactorBatch:
    """LsFactor (solvers.cpp:24-78) of a batch of matrices, computed on the device."""
    rank: np.ndarray        # (nmat,)
    deficient: np.ndarray   # (nmat,) bool: COD branch
    reff: np.ndarray        # (nmat,) R0 rows kept by the pivoted factorisation
    pinv: np.ndarray        # (nmat, n, m)
    Q: np.ndarray           # (nmat, m, n), columns >= rank zero

    def apply_pinv(self, t, v):
        return self.pinv[t] @ v

    def apply_pinv_transpose(self, t, u):
        return self.pinv[t].T @ u

    def apply_projection(self, t, v):
        q = self.Q[t][:, :self.rank[t]]
        return q @ (q.T @ v)


def lsfactor_batch(K, rank_tol: float = 1e-10, device: int = 0) -> LsFactorBatch:
    """K: (nmat, m, n) or (m, n) float64. Runs the batched QR / COD kernels of the hot path
    (include/ddelm_gpu.h ddelm_gpu_lsfactor_batch)."""
    K = np.asarray(K, dtype=np.float64)
    if K.ndim == 2:
        K = K[None]
    nmat, m, n = K.shape
    Kf = np.ascontiguousarray(np.transpose(K, (0, 2, 1)))  # column-major blocks
    rank = np.zeros(nmat, dtype=np.int32)
    defi = np.zeros(nmat, dtype=np.int32)
    reff = np.zeros(nmat, dtype=np.int32)
    pinv = np.zeros((nmat, m, n))  # column-major n x m == row-major m x n
    Q = np.zeros((nmat, n, m))
    _check(load_library().ddelm_gpu_lsfactor_batch(device, nmat, m, n, _ptr(Kf), float(rank_tol), _ptr(rank),
                                                   _ptr(defi), _ptr(reff), _ptr(pinv), _ptr(Q)))
    return LsFactorBatch(rank=rank, deficient=defi.astype(bool), reff=reff,
                         pinv=np.transpose(pinv, (0, 2, 1)).copy(), Q=np.transpose(Q, (0, 2, 1)).copy())


def plan_tables(cfg, rank: int, world: int) -> dict:
    """Host-side owner-slot tables of one shard (no GPU needed): the sharding logic under test."""
    L = load_library()
    d = _cfg_desc(cfg)
    out = {}
    for which, name in enumerate(["gamma_dst", "flux_dst", "nd_dst", "corner_dst", "cross_dst", "meta"]):
        n = L.ddelm_gpu_plan_tables(C.byref(d), rank, world, which, None, 0)
        if n < 0:
            _check(-n)
        a = np.zeros(max(n, 1), dtype=np.int32)
        L.ddelm_gpu_plan_tables(C.byref(d), rank, world, which, _ptr(a), n)
        out[name] = a[:n]
    keys = ["sub_lo", "n_local", "n_global", "n_delta", "n_pi", "npf", "gmax", "fmax", "dmax", "crmax", "ncq"]
    out.update({k: int(v) for k, v in zip(keys, out.pop("meta"))})
    return out


def shard_range(n_subs: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous strip [lo, hi) of subdomains owned by `rank` (plan.cpp shard_range)."""
    return n_subs * rank // world, n_subs * (rank + 1) // world


class Workspace:
    """Device-resident Workspace (solvers.hpp:78-160) on one B200.

    shard=(rank, world, nccl_id) builds a sharded workspace: this process/GPU owns the strip
    shard_range(s*s, rank, world) of subdomains; interface vectors and the coarse problem are
    replicated and every cross-subdomain sum is an owner-slot table whose foreign slots arrive
    over NCCL send/recv between the CG phases. shard=(rank, world, "host:/shm-name") selects the
    host-staged test backend (several ranks on one GPU)."""

    def __init__(self, problem: ProblemSpec | str, s: int, n_grid: int, M: int, l: float, seed: int,
                 opts: SolverOptions | None = None, device: int = 0, shard: tuple | None = None):
        L = load_library()
        if isinstance(problem, str):
            problem = make_problem(problem)
        opts = opts or SolverOptions()
        if opts.flux_variant not in ("pointwise", "mean_edge"):
            raise ValueError("flux_variant must be pointwise or mean_edge")
        pp = problem.params
        d = _Desc(PROBLEMS[problem.name], s, n_grid, M, float(l), seed,
                  1 if opts.flux_variant == "mean_edge" else 0, 1 if opts.change_of_variables else 0,
                  float(opts.rank_tol), device, int(opts.debug_flip_flux_row), float(pp.alpha),
                  int(pp.forcing_seed), int(pp.rho_seed))
        h = C.c_void_p()
        if shard is None:
            _check(L.ddelm_gpu_create(C.byref(d), C.byref(h)))
        else:
            rank, world, nid = shard
            if isinstance(nid, str) and nid.startswith("host:"):
                # test backend: slot segments host-staged through a shared-memory mailbox
                _check(L.ddelm_gpu_create_sharded_host(C.byref(d), int(rank), int(world),
                                                       nid[5:].encode(), C.byref(h)))
            else:
                idbuf = (C.c_ubyte * 128).from_buffer_copy(nid) if nid is not None else None
                _check(L.ddelm_gpu_create_sharded(C.byref(d), int(rank), int(world), idbuf, C.byref(h)))
        self._h = h
        self.problem, self.s, self.n_grid, self.M, self.l, self.seed = problem, s, n_grid, M, l, seed
        self.opts = opts
        lo, cnt, ng = C.c_int(), C.c_int(), C.c_int()
        _check(L.ddelm_gpu_get_shard(h, C.byref(lo), C.byref(cnt), C.byref(ng)))
        self.sub_lo, self.n_local, self.n_global = lo.value, cnt.value, ng.value
        self.n_subs = cnt.value
        cc = 2 if problem.name == "biharmonic_sinpi" else 1  # trace components (geometry.cpp:155-157)
        self.n_delta = 2 * s * (s - 1) * (n_grid - 2) * cc
        self.n_pi = (s - 1) * (s - 1) * cc

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            load_library().ddelm_gpu_destroy(h)
            self._h = None

    # reference lazily builds layers; these mirror the member functions
    def build(self):
        _check(load_library().ddelm_gpu_build(self._h))

    def assemble_coarse(self):
        _check(load_library().ddelm_gpu_build_coarse(self._h))

    def build_neumann(self):
        _check(load_library().ddelm_gpu_build_neumann(self._h))

    def reseed(self, seed: int):
        _check(load_library().ddelm_gpu_reseed(self._h, seed))
        self.seed = seed

    @property
    def cg_driver(self) -> str:
        """CG driver of the last solve: graph-while, graph-chunked, host-loop or persistent."""
        return load_library().ddelm_gpu_cg_driver(self._h).decode()

    def set_cg_blocks(self, mode: str):
        """'coeff' (default: the reference's grouping, its CG trajectory) or 'compact'
        (precomputed interface-level blocks; include/ddelm_gpu.h ddelm_gpu_set_cg_blocks)."""
        code = {"coeff": 0, "compact": 1}[mode]
        _check(load_library().ddelm_gpu_set_cg_blocks(self._h, code))
        self.cg_blocks = mode

    def ranks(self):
        N = self.n_subs
        rk, rkb = np.zeros(N, np.int32), np.zeros(N, np.int32)
        ratio = np.zeros(2 * N)
        _check(load_library().ddelm_gpu_get_ranks(self._h, _ptr(rk), _ptr(rkb), _ptr(ratio)))
        return rk, rkb, ratio.reshape(N, 2)

    def layer(self, i: int):
        w0, w1, b = np.zeros(self.M), np.zeros(self.M), np.zeros(self.M)
        _check(load_library().ddelm_gpu_get_layer(self._h, i, _ptr(w0), _ptr(w1), _ptr(b)))
        return w0, w1, b

    def local_matrix(self, i: int, which: int = 0) -> np.ndarray:
        """K_i (which=0) or Kbar_i (which=1) as built by the feature kernel (rows x M)."""
        rows = C.c_int()
        _check(load_library().ddelm_gpu_get_local(self._h, i, which, None, C.byref(rows)))
        K = np.zeros((self.M, rows.value))
        _check(load_library().ddelm_gpu_get_local(self._h, i, which, _ptr(K), C.byref(rows)))
        return K.T.copy()

    def local_rhs(self, i: int) -> np.ndarray:
        """f_i (assembly.cpp:21-33) as the device holds it (GRF problems: evaluated on the device)."""
        rows = C.c_int()
        _check(load_library().ddelm_gpu_get_local(self._h, i, 2, None, C.byref(rows)))
        f = np.zeros(rows.value)
        _check(load_library().ddelm_gpu_get_local(self._h, i, 2, _ptr(f), C.byref(rows)))
        return f

    def invalidate(self):
        """Drop built layers, keep the device-resident feature layers."""
        _check(load_library().ddelm_gpu_invalidate(self._h))

    @property
    def stream_handle(self) -> int:
        return int(load_library().ddelm_gpu_stream(self._h) or 0)

    def set_profiling(self, on: bool = True):
        _check(load_library().ddelm_gpu_set_profiling(self._h, 1 if on else 0))

    def kernel_stats(self, family: str) -> dict:
        ms, n, fl, by = C.c_double(), C.c_longlong(), C.c_double(), C.c_double()
        _check(load_library().ddelm_gpu_get_kernel_stats(self._h, family.encode(), C.byref(ms),
                                                         C.byref(n), C.byref(fl), C.byref(by)))
        return {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}

    def device_span_ms(self) -> float:
        return float(load_library().ddelm_gpu_get_device_span_ms(self._h))

    def apply_operator(self, v: np.ndarray, theta: float = 0.999) -> np.ndarray:
        """cs_reduced_apply with the NN weight (theta = 0: coarse operator), on the device."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros_like(v)
        _check(load_library().ddelm_gpu_apply_operator(self._h, float(theta), _ptr(v), _ptr(out)))
        return out

    def sample_field(self, n: int = 257):
        """Field and gradient of the last solve on the n x n grid, flat b*n + a (sample_field,
        metrics.cpp:18-57), evaluated on the device."""
        u, gx, gy = np.zeros(n * n), np.zeros(n * n), np.zeros(n * n)
        _check(load_library().ddelm_gpu_sample_field(self._h, int(n), _ptr(u), _ptr(gx), _ptr(gy)))
        return u, gx, gy

    def relative_errors(self, n: int = 257) -> tuple[float, float]:
        """(L2, H1) relative errors against the exact solution (metrics.cpp:112-128)."""
        l2, h1 = C.c_double(), C.c_double()
        _check(load_library().ddelm_gpu_relative_errors(self._h, int(n), C.byref(l2), C.byref(h1)))
        return l2.value, h1.value

    def field_diff(self, ref_coeffs: np.ndarray, n: int = 257) -> tuple[float, float]:
        """(L2, H1) relative difference against the ELM field of ref_coeffs on the same layers
        (oracle_check's field_diff, runner.cpp:269-281)."""
        c = np.ascontiguousarray(ref_coeffs, dtype=np.float64)
        l2, h1 = C.c_double(), C.c_double()
        _check(load_library().ddelm_gpu_field_diff(self._h, int(n), _ptr(c), C.byref(l2), C.byref(h1)))
        return l2.value, h1.value

    def apply_reduced(self, v: np.ndarray) -> np.ndarray:
        """reduced_apply (solvers.cpp:262-274), the one-level operator on mu = [mu_Delta; mu_Pi]."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros_like(v)
        _check(load_library().ddelm_gpu_apply_reduced(self._h, _ptr(v), _ptr(out)))
        return out

    def apply_P(self, v: np.ndarray) -> np.ndarray:
        """The Neumann map P = Abar Kbar^+ Bbar on n_delta values (Workspace::apply_P,
        solvers.cpp:450-461), through the device NN1 phase."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros_like(v)
        _check(load_library().ddelm_gpu_apply_neumann(self._h, 0, _ptr(v), _ptr(out)))
        return out

    def apply_PT(self, u: np.ndarray) -> np.ndarray:
        """The adjoint P^T (Workspace::apply_PT, solvers.cpp:463-474), through the NN2 phase."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        _check(load_library().ddelm_gpu_apply_neumann(self._h, 1, _ptr(u), _ptr(out)))
        return out

    def _solve(self, method: str, theta: float, cg: CgOptions | None, fetch: bool = True) -> SolveReport:
        """fetch=False leaves mu / coefficients / history on the device (device-resident timing)."""
        cg = cg or CgOptions()
        L = load_library()
        rep = _Report()
        _check(L.ddelm_gpu_solve(self._h, METHODS[method], float(theta), float(cg.rel_tol),
                                 int(cg.max_iter), C.byref(rep)))
        nmu = rep.n_mu
        mu = np.zeros(nmu)
        co = np.zeros((rep.n_subdomains, rep.M))
        hist = np.zeros(max(rep.iterations, 1))
        n = 0
        if fetch:
            _check(L.ddelm_gpu_get_mu(self._h, _ptr(mu)))
            _check(L.ddelm_gpu_get_coeffs(self._h, _ptr(co)))
            n = L.ddelm_gpu_get_residuals(self._h, _ptr(hist), hist.size)
        ms = np.zeros(8)
        L.ddelm_gpu_get_phase_ms(self._h, _ptr(ms), 8)
        names = ["features", "qr", "cod", "coarse", "neumann", "rhs", "cg", "reconstruct"]
        return SolveReport(coeffs=co, mu=mu, mu_delta=mu[:rep.n_delta], mu_pi=mu[rep.n_delta:],
                           iterations=rep.iterations, converged=bool(rep.converged),
                           negative_curvature=bool(rep.negative_curvature),
                           residual_history=hist[:max(n, 0)],
                           setup_seconds=rep.setup_seconds, cg_seconds=rep.cg_seconds,
                           reconstruct_seconds=rep.reconstruct_seconds,
                           assembly_seconds=rep.assembly_seconds,
                           factorization_seconds=rep.factorization_seconds,
                           total_seconds=rep.total_seconds,
                           phase_ms=dict(zip(names, ms.tolist())),
                           launches=int(L.ddelm_gpu_get_launch_count(self._h)))


def ddelm_cs_solve(ws: Workspace, cg: CgOptions | None = None) -> SolveReport:
    """ddelm_cs_solve (solvers.cpp:582-588)."""
    return ws._solve("ddelm-cs", 0.0, cg)


def ddelm_nn_solve(ws: Workspace, theta: float, cg: CgOptions | None = None) -> SolveReport:
    """ddelm_nn_solve (solvers.cpp:590-605): theta in [0, 1]; theta == 0 is exactly CS."""
    if theta < 0.0 or theta > 1.0:
        raise ValueError("ddelm_nn_solve: theta must lie in [0, 1]")
    return ws._solve("ddelm-nn", theta, cg)


def ddelm_solve(ws: Workspace, cg: CgOptions | None = None) -> SolveReport:
    """One-level DDELM (solvers.cpp:493-531): CG on mu = [mu_Delta; mu_Pi] with reduced_apply."""
    return ws._solve("ddelm", 0.0, cg)


@dataclass
class DenseOracle:
    """solvers.hpp DenseOracle: the brute-force dense solve of the same discrete system."""
    reduced_op: np.ndarray   # (dim, dim)
    reduced_rhs: np.ndarray
    mu_reduced: np.ndarray
    mu_full: np.ndarray
    coeffs: np.ndarray       # (n_subs, M)


def dense_oracle_solve(ws: Workspace, method: str = "ddelm-nn", theta: float = 0.999) -> DenseOracle:
    """dense_oracle_solve (solvers.cpp:609-709) on the device: K, B, A (and Kbar, Bbar, Abar for NN)
    assembled densely, every pseudo-inverse through the device QR / COD kernels with Eigen's default
    threshold; the reduced system solved by a device COD. sum(M) + n_mu <= 3000 (ValueError above,
    as the reference). Regenerates the local matrices: the next solve rebuilds the factorisations."""
    nmu = ws.n_delta + ws.n_pi
    dim = nmu if method == "ddelm" else ws.n_delta
    op = np.zeros((dim, dim))
    rhs, mu, co = np.zeros(dim), np.zeros(nmu), np.zeros((ws.n_subs, ws.M))
    d = C.c_int()
    _check(load_library().ddelm_gpu_dense_oracle(ws._h, METHODS[method], float(theta), C.byref(d), _ptr(op),
                                                 _ptr(rhs), _ptr(mu), _ptr(co)))
    op = op.T.copy()  # column-major -> (row, col)
    return DenseOracle(op, rhs, mu[:dim].copy(), mu, co)


@dataclass
class OracleCheckReport:
    """runner.hpp OracleCheckReport."""
    mu_diff: float
    field_diff: float
    op_diff: float
    op_row: int
    op_col: int
    passed: bool


def oracle_check(name_or_cfg, device: int = 0) -> OracleCheckReport:
    """oracle_check (runner.cpp:252-316): the iterative solve to 1e-12 against the dense oracle —
    relative mu difference, field difference on the 65 x 65 grid, and the largest entry of
    (iterative operator - dense reduced operator) over the unit vectors; pass below 1e-6 each."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    method, theta = cfg["method"], float(cfg.get("theta", 0.999))
    ws = workspace_from_config(cfg, device)
    dense = dense_oracle_solve(ws, method, theta)
    tight = CgOptions(rel_tol=1e-12, max_iter=0)
    rep = (ddelm_solve(ws, tight) if method == "ddelm" else ddelm_cs_solve(ws, tight)
           if method == "ddelm-cs" else ddelm_nn_solve(ws, theta, tight))
    mn = np.linalg.norm(dense.mu_full)
    mu_diff = float(np.linalg.norm(rep.mu - dense.mu_full) / (mn if mn > 0 else 1.0))
    field = ws.field_diff(dense.coeffs, 65)[0]
    dim = dense.reduced_op.shape[0]
    op_diff, op_row, op_col = 0.0, -1, -1
    for j in range(dim):
        e = np.zeros(dim)
        e[j] = 1.0
        col = ws.apply_reduced(e) if method == "ddelm" else \
            ws.apply_operator(e, theta if method == "ddelm-nn" else 0.0)
        d = np.abs(col - dense.reduced_op[:, j])
        i = int(np.argmax(d))
        if d[i] > op_diff:
            op_diff, op_row, op_col = float(d[i]), i, j
    return OracleCheckReport(mu_diff, field, op_diff, op_row, op_col,
                             mu_diff < 1e-6 and field < 1e-6 and op_diff < 1e-6)


class LsqBatch:
    """C5 microbenchmark: batched local least squares (QR of [K | B]) + interface Schur block S
    (include/ddelm_gpu.h, ddelm_gpu_lsq_*). Flops per block follow SURVEY.md §8d."""

    def __init__(self, nblocks: int, m: int, n: int, k: int, device: int = 0):
        L = load_library()
        h = C.c_void_p()
        _check(L.ddelm_gpu_lsq_create(nblocks, m, n, k, device, C.byref(h)))
        self._h = h
        self.nblocks, self.m, self.n, self.k = nblocks, m, n, k
        self.ld = int(L.ddelm_gpu_lsq_ld(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            load_library().ddelm_gpu_lsq_destroy(h)
            self._h = None

    def generate(self, seed: int = 1, kind: str = "tanh"):
        _check(load_library().ddelm_gpu_lsq_generate(self._h, seed, {"tanh": 0, "gaussian": 1}[kind]))

    def factor(self) -> tuple[float, float]:
        qr, sc = C.c_double(), C.c_double()
        _check(load_library().ddelm_gpu_lsq_factor(self._h, C.byref(qr), C.byref(sc)))
        return qr.value, sc.value

    def block(self, b: int):
        """(A (ld x (n+k)) column-major as an (n+k, ld) array transposed, tau (n), S (k x k))."""
        A = np.zeros((self.n + self.k, self.ld))
        tau = np.zeros(self.n)
        S = np.zeros((self.k, self.k))
        _check(load_library().ddelm_gpu_lsq_get_block(self._h, b, _ptr(A), _ptr(tau), _ptr(S)))
        return A.T[: self.m].copy(), tau, S

    def flops_per_block(self) -> float:
        m, n, k = self.m, self.n, self.k
        return (2.0 * m * n * n - 2.0 * n ** 3 / 3.0) + (4.0 * m * n * k - 2.0 * n * n * k) + 2.0 * (m - n) * k * k


def workspace_from_config(name_or_cfg, device: int = 0, shard: tuple | None = None) -> Workspace:
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    opts = SolverOptions(flux_variant=cfg["flux_variant"],
                         change_of_variables=cfg["trace_basis"] == "change_of_variables",
                         debug_flip_flux_row=int(cfg.get("debug_flip_flux_row", -1)))
    problem = make_problem(cfg["problem"], ProblemParams(cfg.get("alpha", 32.0), cfg.get("forcing_seed", 2),
                                                         cfg.get("rho_seed", 3)))
    return Workspace(problem, cfg["s"], cfg["n_grid"], cfg["M"], cfg["l"], cfg["seed"], opts, device,
                     shard)


def solve_config(name_or_cfg, device: int = 0, ws: Workspace | None = None,
                 cg_blocks: str | None = None) -> tuple[Workspace, SolveReport]:
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    ws = ws or workspace_from_config(cfg, device)
    if cg_blocks is not None:
        ws.set_cg_blocks(cg_blocks)
    cg = CgOptions(rel_tol=cfg["cg_rel_tol"])
    if cfg["method"] == "ddelm-cs":
        return ws, ddelm_cs_solve(ws, cg)
    if cfg["method"] == "ddelm":
        return ws, ddelm_solve(ws, cg)
    return ws, ddelm_nn_solve(ws, cfg["theta"], cg)
