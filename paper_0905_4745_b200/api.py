"""Python mirror of the reference's public interface for the hot path.

Names, argument meaning and error behaviour follow
``include/minnorm/{solver,lsq,srft,fft,errors}.hpp`` of the reference
(``/root/reference/proj``); every call goes through the C ABI of
``libminnorm_b200.so`` (include/minnorm_b200.h) and runs on the GPU.
Host numpy arrays and CUDA torch tensors are both accepted; complex arrays
use the reference's layout (column-major complex<double>).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L


# ------------------------------------------------------------------ errors --
class ConfigError(ValueError):
    """minnorm::ConfigError (include/minnorm/errors.hpp:10-13)."""


class DimensionError(ValueError):
    """minnorm::DimensionError (include/minnorm/errors.hpp:16-19)."""


class RankDeficiencyError(RuntimeError):
    """minnorm::RankDeficiencyError (include/minnorm/errors.hpp:22-31)."""

    def __init__(self, what: str, deficient_columns: int):
        super().__init__(what)
        self._deficient = int(deficient_columns)

    def deficient_columns(self) -> int:
        return self._deficient


class ParseError(RuntimeError):
    """minnorm::ParseError (include/minnorm/errors.hpp:34-49): 1-based line / column, 0 when unknown."""

    def __init__(self, what: str, line: int = 0, column: int = 0):
        super().__init__(what)
        self._line, self._column = int(line), int(column)

    def line(self) -> int:
        return self._line

    def column(self) -> int:
        return self._column


class UnsupportedError(RuntimeError):
    """A shape this build has no GPU kernel for (e.g. an FFT length with large prime factors)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure."""


def _check(status: int) -> None:
    if status == L.MNB_OK:
        return
    msg = L.last_error()
    if status == L.MNB_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == L.MNB_ERR_CONFIG:
        raise ConfigError(msg)
    if status == L.MNB_ERR_DIMENSION:
        raise DimensionError(msg)
    if status == L.MNB_ERR_RANK_DEFICIENCY:
        raise RankDeficiencyError(msg, L.load().mnb_last_deficient_columns())
    if status == L.MNB_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == L.MNB_ERR_PARSE:
        ln, col = ctypes.c_int64(), ctypes.c_int64()
        L.load().mnb_last_parse_location(ctypes.byref(ln), ctypes.byref(col))
        raise ParseError(msg, ln.value, col.value)
    if status == L.MNB_ERR_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise DeviceError(f"[status {status}] {msg}")


class Sampling(enum.IntEnum):
    """RandomStream::Sampling (include/minnorm/rng.hpp:18)."""
    without_replacement = 0
    with_replacement = 1


# -------------------------------------------------------------- rng seeds --
_GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_seed(seed: int, tag: int) -> int:
    """RandomStream::derive_seed (src/rng.cpp:37-39): seed of substream(tag)."""
    return _mix(_mix((seed + _GOLDEN) & _M64) ^ _mix((tag + 2 * _GOLDEN) & _M64))


# ----------------------------------------------------------- array helpers --
def _is_torch_cuda(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)


def _host_c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x), dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- context --
class Context:
    """One GPU (one rank).  Owns a CUDA stream, the (sharded) problem matrix
    and the workspaces; see mnb_context_* in include/minnorm_b200.h."""

    def __init__(self, device: int = 0, _handle=None):
        self._lib = L.load()
        self._keep = None
        if _handle is None:
            h = ctypes.c_void_p()
            _check(self._lib.mnb_context_create(device, ctypes.byref(h)))
            _handle = h
        self._h = _handle
        self.device = device
        self.rank, self.world_size = 0, 1
        self.is_distributed = False
        self.m = self.n = self.col_begin = self.n_local = 0
        self.dtype = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(L.load().mnb_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def distributed(cls, device: int, rank: int, world_size: int, unique_id: bytes) -> "Context":
        lib = L.load()
        h = ctypes.c_void_p()
        uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(lib.mnb_context_create_distributed(device, rank, world_size, uid, ctypes.byref(h)))
        ctx = cls(device, _handle=h)
        ctx.rank, ctx.world_size = rank, world_size
        ctx.is_distributed = True
        return ctx

    def set_shard(self, A, n_global: Optional[int] = None) -> None:
        """Distributed context: A is this rank's column shard of an m x n_global matrix, the
        columns mnb_shard_columns(n_global, world_size, rank) assigns.  n_global defaults to the
        one of the last set_matrix call; a shard whose width does not match is a DimensionError."""
        n_global = int(n_global or self.n)
        if n_global <= 0:
            raise ValueError("distributed context: pass n_global (the global column count) with the first shard")
        col_begin, count = shard_columns(n_global, self.world_size, self.rank)
        if A.shape[1] != count:
            raise DimensionError(f"rank {self.rank} of {self.world_size}: shard has {A.shape[1]} columns, "
                                 f"mnb_shard_columns({n_global}) assigns {count}")
        self.set_matrix(A, n_global=n_global, col_begin=col_begin)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.mnb_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int) -> None:
        _check(self._lib.mnb_context_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    def set_matrix(self, A, n_global: Optional[int] = None, col_begin: int = 0, deferred: bool = False) -> None:
        """A: this rank's column shard (m x n_local), complex128 or float64.
        numpy arrays are copied to the GPU; CUDA torch tensors are borrowed
        (column-major, i.e. a transposed-contiguous tensor or a (n,m) row-major
        tensor viewed as A^T).  deferred=True (MNB_HOST_ASYNC): a page-locked
        host array is copied by the next solve, overlapped with its sketches;
        the array is kept referenced until that solve returns."""
        if _is_torch_cuda(A):
            import torch
            if A.dtype == torch.complex128:
                dtype = L.MNB_C128
            elif A.dtype == torch.float64:
                dtype = L.MNB_F64
            else:
                raise TypeError("A must be complex128 or float64")
            m, nl = A.shape
            if not (A.stride(0) == 1 and A.stride(1) == m):
                raise ValueError("device A must be column-major (A.T contiguous)")
            # the library works on its own stream: whatever torch queued to produce A (on any of
            # its streams) must be complete before a solve reads the borrowed pointer
            torch.cuda.synchronize(A.device)
            self._keep = A
            ptr, loc = ctypes.c_void_p(A.data_ptr()), L.MNB_DEVICE
        else:
            A = np.asarray(A)
            if A.dtype == np.float64:
                dtype = L.MNB_F64
            else:
                A = A.astype(np.complex128, copy=False)
                dtype = L.MNB_C128
            A = np.asfortranarray(A)
            m, nl = A.shape
            self._keep = A
            ptr, loc = _ptr(A), (L.MNB_HOST_ASYNC if deferred else L.MNB_HOST)
        n_global = nl if n_global is None else n_global
        _check(self._lib.mnb_set_matrix(self._h, dtype, m, n_global, col_begin, nl, ptr, m, loc))
        if loc == L.MNB_HOST:
            self._keep = None  # copied
        self.m, self.n, self.col_begin, self.n_local = m, n_global, col_begin, nl
        self.dtype = dtype

    # ---- the sketch-QR building blocks (csrc/k_cholqr.cu), on host arrays
    def chol_upper(self, G, shift_factor: float = 0.0, rank_rows: float = 0.0):
        """Upper Cholesky R (G = R^H R) of a Hermitian matrix; returns (R, status dict)."""
        G = np.array(G, dtype=np.complex128, order="F")
        m = G.shape[0]
        st = (ctypes.c_double * 7)()
        _check(self._lib.mnb_chol_upper(self._h, _ptr(G), m, shift_factor, rank_rows, st))
        return G, {"info": int(st[0]), "deficient": int(st[1]), "dmin": st[2], "dmax": st[3], "trace": st[4],
                   "shift": st[5], "kernel_ms": st[6]}

    def trtri_upper(self, R):
        """Inverse of an upper-triangular matrix; returns (X, ||X||_F^2)."""
        R = np.array(R, dtype=np.complex128, order="F")
        m = R.shape[0]
        X = np.empty((m, m), dtype=np.complex128, order="F")
        out = (ctypes.c_double * 2)()
        _check(self._lib.mnb_trtri_upper(self._h, _ptr(R), m, _ptr(X), out))
        self.last_kernel_ms = out[1]
        return X, out[0]

    def csne_solve(self, S, b):
        """Step 2's z = Q R^{-H} b (src/solver.cpp:93-96) of the sketch S = Q R; returns (z, status dict)."""
        S = np.array(S, dtype=np.complex128, order="F")
        b = np.ascontiguousarray(b, dtype=np.complex128)
        l, m = S.shape
        z = np.empty(l, dtype=np.complex128)
        st = (ctypes.c_double * 4)()
        _check(self._lib.mnb_csne_solve(self._h, _ptr(S), l, m, _ptr(b), _ptr(z), st))
        return z, {"accepted": bool(st[0]), "corrections": int(st[1]), "residual": st[2], "znorm": st[3]}

    def bench_pcg_pass(self, reps: int = 10) -> float:
        out = ctypes.c_double()
        _check(self._lib.mnb_bench_pcg_pass(self._h, reps, ctypes.byref(out)))
        return out.value


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def shard_columns(n: int, world_size: int, rank: int) -> tuple[int, int]:
    """Column partition of every multi-GPU entry point (mnb_shard_columns)."""
    b, c = ctypes.c_int64(), ctypes.c_int64()
    _check(L.load().mnb_shard_columns(n, world_size, rank, ctypes.byref(b), ctypes.byref(c)))
    return b.value, c.value


def redistribute_plan(m: int, n_global: int, world_size: int, rank: int) -> np.ndarray:
    """The distributed sketch's all-to-all table (mnb_redistribute_plan): one row per peer h,
    [send_row0, send_rows, send_offset, recv_col0, recv_cols, recv_offset] (offsets in elements
    of the pack buffer / of this rank's my_rows x n_global column-major row block)."""
    plan = np.zeros((world_size, 6), np.int64)
    _check(L.load().mnb_redistribute_plan(int(m), int(n_global), int(world_size), int(rank),
                                          plan.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return plan


# ----------------------------------------------------------------- solver --
@dataclass
class SolverConfig:
    """include/minnorm/solver.hpp:26-34"""
    sketch_size: Optional[int] = None
    alpha: float = 4.0
    epsilon: float = 1e-6
    seed: int = 42
    sampling: Sampling = Sampling.without_replacement
    lsq_max_iterations: int = 300
    capture_c: bool = False

    def _c(self) -> L.SolverConfigC:
        c = L.SolverConfigC()
        c.sketch_size = int(self.sketch_size or 0)
        c.alpha, c.epsilon, c.seed = float(self.alpha), float(self.epsilon), int(self.seed) & _M64
        c.sampling, c.capture_c = int(self.sampling), int(bool(self.capture_c))
        c.lsq_max_iterations = int(self.lsq_max_iterations)
        return c


@dataclass
class SolveReport:
    """include/minnorm/solver.hpp:36-46 (+ device timings in `extra`)."""
    x: np.ndarray
    step_seconds: list
    c_norm_ratio: float
    residual_norm: float
    lsq_iterations: int
    lsq_converged: bool
    sketch_size: int
    lsq_tau: float
    c: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)


def _report(rc: L.SolveReportC, x, c) -> SolveReport:
    extra = {k: getattr(rc, k) for k in ("lsq_achieved_excess", "param_seconds", "total_seconds", "qr_path",
                                         "redistribute_seconds", "pcg_seconds", "pcg_pass_ms_sum",
                                         "pcg_pass_launches", "kernel_launches", "world_size")}
    extra["sketch_seconds"] = list(rc.sketch_seconds)
    extra["qr_seconds"] = list(rc.qr_seconds)
    extra["sketch_kernel_ms"] = list(rc.sketch_kernel_ms)
    return SolveReport(x=x, step_seconds=list(rc.step_seconds), c_norm_ratio=rc.c_norm_ratio,
                       residual_norm=rc.residual_norm, lsq_iterations=int(rc.lsq_iterations),
                       lsq_converged=bool(rc.lsq_converged), sketch_size=int(rc.sketch_size), lsq_tau=rc.lsq_tau,
                       c=c, extra=extra)


class ProblemInstance:
    """include/minnorm/solver.hpp:14-24: A (m x n, m < n) and b (m)."""

    def __init__(self, A, b):
        self.A, self.b = A, b

    def m(self) -> int:
        return int(self.A.shape[0])

    def n(self) -> int:
        return int(self.A.shape[1])

    def validate(self) -> None:
        """src/solver.cpp:37-48"""
        m, n = self.m(), self.n()
        if m < 1 or m >= n:
            raise DimensionError(f"problem must be underdetermined: 1 <= m < n, got m={m}, n={n}")
        if len(self.b) != m:
            raise DimensionError(f"right-hand side length {len(self.b)} does not match m={m}")


def solve_randomized(inst: ProblemInstance, cfg: SolverConfig = SolverConfig(), ctx: Optional[Context] = None,
                     x_out=None, c_out=None, n_global: Optional[int] = None) -> SolveReport:
    """solve_randomized (include/minnorm/solver.hpp:55; src/solver.cpp:50-128) on the GPU.

    With a distributed context, `inst.A` is this rank's column shard (Context.set_shard:
    n_global is required with the first shard) and the returned x / c are this rank's entries."""
    ctx = ctx or default_context()
    A = inst.A
    if A is not None:
        if len(inst.b) != A.shape[0]:
            raise DimensionError(f"right-hand side length {len(inst.b)} does not match m={A.shape[0]}")
        if not ctx.is_distributed:
            if A.shape[0] < 1 or A.shape[0] >= A.shape[1]:
                raise DimensionError(f"problem must be underdetermined: 1 <= m < n, got m={A.shape[0]}, "
                                     f"n={A.shape[1]}")
            ctx.set_matrix(A, deferred=True)  # pinned host A: copied in slabs under the sketches
        else:
            ctx.set_shard(A, n_global)
    b = _host_c128(inst.b.cpu().numpy() if _is_torch_cuda(inst.b) else inst.b)
    rc = L.SolveReportC()
    if x_out is not None:  # device tensors (torch), zero-copy
        xp, xl = ctypes.c_void_p(x_out.data_ptr()), L.MNB_DEVICE
        cp = ctypes.c_void_p(c_out.data_ptr()) if c_out is not None else None
        x = x_out
        c = c_out
    else:
        x = np.zeros(ctx.n_local, np.complex128)
        c = np.zeros(ctx.n_local, np.complex128) if cfg.capture_c else None
        xp, xl, cp = _ptr(x), L.MNB_HOST, (_ptr(c) if c is not None else None)
    try:
        _check(ctx._lib.mnb_solve_randomized(ctx._h, _ptr(b), L.MNB_HOST, ctypes.byref(cfg._c()), xp, xl, cp,
                                             ctypes.byref(rc)))
    finally:
        if A is not None and not _is_torch_cuda(A):
            ctx._keep = None  # a deferred host copy is complete once the solve returns
    return _report(rc, x, c)


# -------------------------------------------------------------------- lsq --
@dataclass
class LsqConfig:
    """include/minnorm/lsq.hpp:12-18 (stream = RandomStream(stream_seed))."""
    sketch_size: int = 0
    tau: float = 1e-12
    max_iterations: int = 300
    stream_seed: int = 42
    sampling: Sampling = Sampling.without_replacement


def apply_adjoint_matrix(y, ctx: Optional[Context] = None, with_ax: bool = False):
    """x = A^H y for the context matrix (this rank's columns) -- Step 5 of solve_randomized
    (src/solver.cpp:118-125) -- and, with with_ax, A x (summed over ranks) from the same pass."""
    ctx = ctx or default_context()
    y = _host_c128(y)
    if y.size != ctx.m:
        raise DimensionError(f"y length {y.size} does not match m={ctx.m}")
    x = np.zeros(ctx.n_local, np.complex128)
    ax = np.zeros(ctx.m, np.complex128) if with_ax else None
    _check(ctx._lib.mnb_apply_adjoint_matrix(ctx._h, _ptr(y), L.MNB_HOST, _ptr(x), L.MNB_HOST,
                                             _ptr(ax) if ax is not None else None))
    return (x, ax) if with_ax else x


@dataclass
class ClassicalReport:
    """mnb_classical_report (include/minnorm_b200.h): the path taken and its diagnostics."""
    path: int           # 0 Gram + corrected seminormal equations, 1 Householder QR of A^H
    refinements: int
    residual_norm: float
    seconds: float


def solve_classical(inst: ProblemInstance, ctx: Optional[Context] = None, report: bool = False,
                    n_global: Optional[int] = None):
    """solve_classical (include/minnorm/solver.hpp:59; src/solver.cpp:130-146) on the GPU:
    the minimal-norm x of A x = b by the deterministic O(m^2 n) method (the paper's t0
    baseline).  Returns x (this rank's entries), or (x, ClassicalReport) with report=True.
    Raises like the reference: DimensionError, RankDeficiencyError."""
    ctx = ctx or default_context()
    A = inst.A
    if A is not None:
        if len(inst.b) != A.shape[0]:
            raise DimensionError(f"right-hand side length {len(inst.b)} does not match m={A.shape[0]}")
        if not ctx.is_distributed:
            ctx.set_matrix(A)
        else:
            ctx.set_shard(A, n_global)
    b = _host_c128(inst.b.cpu().numpy() if _is_torch_cuda(inst.b) else inst.b)
    x = np.zeros(ctx.n_local, np.complex128)
    rc = L.ClassicalReportC()
    try:
        _check(ctx._lib.mnb_solve_classical(ctx._h, _ptr(b), L.MNB_HOST, _ptr(x), L.MNB_HOST, ctypes.byref(rc)))
    finally:
        if A is not None and not _is_torch_cuda(A):
            ctx._keep = None
    rep = ClassicalReport(path=int(rc.path), refinements=int(rc.refinements), residual_norm=float(rc.residual_norm),
                          seconds=float(rc.seconds))
    return (x, rep) if report else x


@dataclass
class LsqSolution:
    """include/minnorm/lsq.hpp:20-26"""
    y: np.ndarray
    achieved_excess: float
    iterations: int
    converged: bool
    residual_norms: list


def solve_least_squares(B, c, cfg: LsqConfig, ctx: Optional[Context] = None) -> LsqSolution:
    """solve_least_squares(B, c, cfg) (include/minnorm/lsq.hpp:37; src/lsq.cpp:43-113).

    The GPU boundary streams A = B^H (the solver only ever passes B = A^H,
    src/solver.cpp:112); B is conjugate-transposed on the host here."""
    ctx = ctx or default_context()
    B = np.asarray(B)
    if B.ndim != 2:
        raise ValueError("B must be a matrix")
    n, m = B.shape
    c = _host_c128(c)
    if m < 1 or n <= m:
        raise ValueError("solve_least_squares: B must be tall (n > m >= 1)")
    if c.size != n:
        raise ValueError("solve_least_squares: c length mismatch")
    A = np.asfortranarray(np.conj(B.astype(np.complex128)).T)
    ctx.set_matrix(A)
    cc = L.LsqConfigC()
    cc.sketch_size, cc.tau, cc.max_iterations = int(cfg.sketch_size), float(cfg.tau), int(cfg.max_iterations)
    cc.stream_seed, cc.sampling = int(cfg.stream_seed) & _M64, int(cfg.sampling)
    y = np.zeros(m, np.complex128)
    norms = np.zeros(max(int(cfg.max_iterations), 1) + 2, np.float64)
    sol = L.LsqSolutionC()
    _check(ctx._lib.mnb_solve_least_squares(ctx._h, _ptr(c), L.MNB_HOST, ctypes.byref(cc), _ptr(y),
                                            norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            ctypes.byref(sol)))
    it = int(sol.iterations)
    return LsqSolution(y=y, achieved_excess=sol.achieved_excess, iterations=it, converged=bool(sol.converged),
                       residual_norms=list(norms[:it + 1]))


# ------------------------------------------------------------------- srft --
class SrftOperator:
    """SrftOperator (include/minnorm/srft.hpp:21-59): parameters drawn on the
    host (bit-identical to the reference RandomStream), applied on the GPU."""

    def __init__(self, handle, l: int, n: int, sampling: Sampling):
        self._lib = L.load()
        self._h = handle
        self.l, self.n, self.mode = l, n, Sampling(sampling)

    def __del__(self):
        try:
            if self._h:
                self._lib.mnb_srft_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def field(self, name: str) -> np.ndarray:
        f = L.FIELDS[name]
        if f <= 2:
            out = np.zeros(self.n, np.complex128)
        elif f <= 8:
            out = np.zeros(self.n - 1, np.float64)
        elif f <= 10:
            out = np.zeros(self.n, np.int64)
        else:
            out = np.zeros(self.l, np.int64)
        _check(self._lib.mnb_srft_get_field(self._h, f, _ptr(out)))
        return out

    def __getattr__(self, name):
        if name in L.FIELDS:
            return self.field(name)
        raise AttributeError(name)

    def _vec(self, fn, x, nin, nout, ctx):
        ctx = ctx or default_context()
        x = _host_c128(x)
        if x.size != nin:
            raise ValueError(f"length {x.size}, expected {nin}")
        y = np.zeros(nout, np.complex128)
        _check(fn(ctx._h, self._h, _ptr(x), _ptr(y)))
        return y

    def apply_h(self, x, ctx: Optional[Context] = None) -> np.ndarray:
        return self._vec(self._lib.mnb_srft_apply_h, x, self.n, self.n, ctx)

    def apply(self, x, ctx: Optional[Context] = None) -> np.ndarray:
        return self._vec(self._lib.mnb_srft_apply, x, self.n, self.l, ctx)

    def apply_adjoint(self, v, ctx: Optional[Context] = None) -> np.ndarray:
        return self._vec(self._lib.mnb_srft_apply_adjoint, v, self.l, self.n, ctx)

    def apply_to_columns(self, M, ctx: Optional[Context] = None) -> np.ndarray:
        """T·M (src/srft.cpp:147-153).  M is n x m; the GPU streams A = M^H
        (the context's problem matrix is replaced)."""
        ctx = ctx or default_context()
        M = np.asarray(M)
        if M.shape[0] != self.n:
            raise ValueError("apply_to_columns: matrix must have n rows")
        ctx.set_matrix(np.asfortranarray(np.conj(M.astype(np.complex128)).T))
        return self.sketch(ctx)

    def sketch(self, ctx: Optional[Context] = None) -> np.ndarray:
        """T·A^H of the context matrix: l x m (column j = T conj(A[j, :]))."""
        ctx = ctx or default_context()
        out = np.zeros((self.l, ctx.m), np.complex128, order="F")
        _check(self._lib.mnb_srft_apply_to_columns(ctx._h, self._h, _ptr(out), L.MNB_HOST))
        return out

    def materialize_dense(self, max_n: int = 2048, ctx: Optional[Context] = None) -> np.ndarray:
        """src/srft.cpp:155-166 (T applied to every basis vector)."""
        if self.n > max_n:
            raise ValueError("materialize_dense: n exceeds the allocation cap")
        return self.apply_to_columns(np.eye(self.n, dtype=np.complex128), ctx)


def build_srft(l: int, n: int, stream_seed: int = 42,
               mode: Sampling = Sampling.without_replacement) -> SrftOperator:
    """build_srft(l, n, RandomStream(stream_seed), mode) (src/srft.cpp:95-113)."""
    lib = L.load()
    h = ctypes.c_void_p()
    _check(lib.mnb_srft_build(int(l), int(n), int(stream_seed) & _M64, int(mode), ctypes.byref(h)))
    return SrftOperator(h, int(l), int(n), mode)


def srft_from_fields(l, n, d, sample, theta, theta_tilde, perm, perm_tilde, zeta, zeta_tilde,
                     mode: Sampling = Sampling.without_replacement) -> SrftOperator:
    """An operator with hand-set fields + finalize() (tests/test_support.hpp:110-126)."""
    lib = L.load()
    arrs = [_host_c128(d), np.ascontiguousarray(sample, np.int64), np.ascontiguousarray(theta, np.float64),
            np.ascontiguousarray(theta_tilde, np.float64), np.ascontiguousarray(perm, np.int64),
            np.ascontiguousarray(perm_tilde, np.int64), _host_c128(zeta), _host_c128(zeta_tilde)]
    h = ctypes.c_void_p()
    _check(lib.mnb_srft_from_fields(int(l), int(n), int(mode), *[_ptr(a) for a in arrs], ctypes.byref(h)))
    return SrftOperator(h, int(l), int(n), mode)


# -------------------------------------------------------------------- fft --
def dft(x, ctx: Optional[Context] = None) -> np.ndarray:
    """Unitary DFT (include/minnorm/fft.hpp:12, src/fft.cpp:121-126)."""
    ctx = ctx or default_context()
    y = _host_c128(x).copy()
    if y.size == 0:
        raise ValueError("Fft: length must be positive")
    _check(ctx._lib.mnb_dft(ctx._h, y.size, _ptr(y), 0))
    return y


def idft(x, ctx: Optional[Context] = None) -> np.ndarray:
    """Inverse unitary DFT (src/fft.cpp:128-131)."""
    ctx = ctx or default_context()
    y = _host_c128(x).copy()
    if y.size == 0:
        raise ValueError("Fft: length must be positive")
    _check(ctx._lib.mnb_dft(ctx._h, y.size, _ptr(y), 1))
    return y


# --------------------------------------------------------- matrix market --
def read_matrix_market(path: str) -> np.ndarray:
    """read_matrix_market (include/minnorm/matrix_market.hpp; src/matrix_market.cpp:65-102): a dense
    complex m x n matrix (column-major).  Raises ParseError with the reference's line / column."""
    lib = L.load()
    rows, cols = ctypes.c_int64(), ctypes.c_int64()
    p = str(path).encode()
    _check(lib.mnb_mm_read_dims(p, ctypes.byref(rows), ctypes.byref(cols)))
    out = np.zeros((rows.value, cols.value), np.complex128, order="F")
    _check(lib.mnb_mm_read(p, out.ctypes.data_as(ctypes.c_void_p), rows.value, cols.value))
    return out


def read_vector_market(path: str) -> np.ndarray:
    """read_vector_market (src/matrix_market.cpp:104-111): a one-column file, else DimensionError."""
    A = read_matrix_market(path)
    if A.shape[1] != 1:
        raise DimensionError(f"'{path}' holds a {A.shape[0]}x{A.shape[1]} matrix where a vector was expected")
    return A[:, 0].copy()


def write_matrix_market(path: str, A) -> None:
    """write_matrix_market (src/matrix_market.cpp:113-130): 17 significant digits, so equal values
    round-trip to byte-identical files.  A vector is written as one column."""
    A = np.asarray(A)
    if A.ndim == 1:
        A = A.reshape(-1, 1)
    A = np.asfortranarray(A.astype(np.complex128, copy=False))
    _check(L.load().mnb_mm_write(str(path).encode(), A.ctypes.data_as(ctypes.c_void_p), A.shape[0], A.shape[1]))


@dataclass
class GeneratedInstance:
    """include/minnorm/bench.hpp: A = U diag(sigma) V^H, b = A p_true."""
    A: np.ndarray
    b: np.ndarray
    p_true: np.ndarray
    kappa: float


def generate_instance(m: int, n: int, kappa: float, stream_seed: int) -> GeneratedInstance:
    """generate_instance(m, n, kappa, RandomStream(stream_seed)) (src/bench.cpp:46-74), host side."""
    A = np.zeros((m, n), np.complex128, order="F")
    b = np.zeros(m, np.complex128)
    p = np.zeros(n, np.complex128)
    _check(L.load().mnb_generate_instance(int(m), int(n), float(kappa), int(stream_seed) & _M64, _ptr(A), _ptr(b),
                                          _ptr(p)))
    return GeneratedInstance(A=A, b=b, p_true=p, kappa=float(kappa))
