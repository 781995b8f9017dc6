"""oracle/minnorm_oracle.py -- TEST INFRASTRUCTURE ONLY (the CPU checker).

Solver-level restatement of the reference's randomized minimal-norm solve
(``/root/reference/proj``) on top of ``oracle/_build/liboracle.so`` (the C++
restatement of rng/fft/srft in ``oracle/minnorm_oracle.cpp``) and
numpy/scipy LAPACK for the dense QR / triangular solves that the reference
delegates to Eigen3 (``Eigen::HouseholderQR``: src/solver.cpp:86,
src/lsq.cpp:58; LAPACK ``zgeqrf`` uses the same Householder convention,
R_jj = -sign(Re x_0)·||x||).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module,
and only as the checker / CPU baseline -- never as the thing measured or
shipped.  The product lives in ``paper_0905_4745_b200/`` and never imports
anything from ``oracle/``.

B = A^H is never materialised (the reference copies it at
src/solver.cpp:76); every product with B goes through A directly.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_REF_PATH = os.path.join(_HERE, "_ref", "libminnorm_ref.so")
EPS = np.finfo(np.float64).eps

_lib = None
_ref = None


def build(force: bool = False) -> None:
    """Compile the oracle (and the verbatim reference pieces when the
    reference tree is present).  Test infrastructure."""
    targets = ["all"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    if force or not os.path.exists(_LIB_PATH) or ("ref" in targets and not os.path.exists(_REF_PATH)):
        subprocess.check_call(["make", "-s", "-C", _HERE] + targets)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, u64, ci, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        L.or_last_error.restype = ctypes.c_char_p
        L.or_derive_seed.restype = u64
        L.or_derive_seed.argtypes = [u64, u64]
        L.or_rng_u64.argtypes = [u64, i64, dp]
        L.or_rng_draw.argtypes = [u64, ci, i64, dp]
        L.or_rng_below.argtypes = [u64, u64, i64, dp]
        L.or_rng_permutation.argtypes = [u64, i64, dp]
        L.or_rng_sample.argtypes = [u64, i64, i64, ci, dp]
        L.or_cmul.argtypes = [dp, dp, dp, i64, ci]
        L.or_rotation_chain.argtypes = [dp, dp, dp, i64, ci]
        L.or_fft_stage.argtypes = [dp, dp, i64, i64, ci]
        L.or_fft.argtypes = [dp, i64, ci]
        L.or_srft_build.restype = vp
        L.or_srft_build.argtypes = [i64, i64, u64, ci]
        L.or_srft_from_fields.restype = vp
        L.or_srft_from_fields.argtypes = [i64, i64, ci] + [dp] * 8
        L.or_srft_free.argtypes = [vp]
        L.or_srft_field.argtypes = [vp, ci, dp]
        L.or_srft_apply_h.argtypes = [vp, dp, dp]
        L.or_srft_apply.argtypes = [vp, dp, dp]
        L.or_srft_apply_adjoint.argtypes = [vp, dp, dp]
        L.or_srft_sketch_rows.argtypes = [vp, dp, ci, i64, i64, i64, dp, ci]
        L.or_gemv_AH.argtypes = [dp, ci, i64, i64, i64, dp, dp, ci]
        L.or_gemv_A.argtypes = [dp, ci, i64, i64, i64, dp, dp, ci]
        _lib = L
    return _lib


def ref_lib():
    """The reference's own rng/kernels compiled verbatim (None if not built)."""
    global _ref
    if _ref is None and os.path.exists(_REF_PATH):
        R = ctypes.CDLL(_REF_PATH)
        u64, i64, ci, dp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        R.ref_derive_seed.restype = u64
        R.ref_derive_seed.argtypes = [u64, u64]
        R.ref_rng_u64.argtypes = [u64, i64, dp]
        R.ref_rng_draw.argtypes = [u64, ci, i64, dp]
        R.ref_rng_permutation.argtypes = [u64, i64, dp]
        R.ref_rng_sample.argtypes = [u64, i64, i64, ci, dp]
        R.ref_kernels_select.argtypes = [ctypes.c_char_p]
        R.ref_cmul.argtypes = [dp, dp, dp, i64, ci]
        R.ref_rotation_chain.argtypes = [dp, dp, dp, i64, ci]
        R.ref_fft_stage.argtypes = [dp, dp, i64, i64, ci]
        _ref = R
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.complex128)


# ------------------------------------------------------------------ rng -----
def derive_seed(seed: int, tag: int) -> int:
    """src/rng.cpp:37-39"""
    return int(lib().or_derive_seed(seed, tag))


def rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    lib().or_rng_u64(seed, count, _p(out))
    return out


def rng_draw(seed: int, kind: str, count: int) -> np.ndarray:
    k = {"u01": 0, "angle": 1, "unit_circle": 2, "sign": 3, "complex_gaussian": 4}[kind]
    out = np.zeros(count * (2 if k in (2, 4) else 1), np.float64)
    lib().or_rng_draw(seed, k, count, _p(out))
    return out.view(np.complex128) if k in (2, 4) else out


def rng_permutation(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.int64)
    lib().or_rng_permutation(seed, n, _p(out))
    return out


def rng_sample(seed: int, l: int, n: int, without: bool = True) -> np.ndarray:
    out = np.zeros(max(l, 0), np.int64)
    if lib().or_rng_sample(seed, l, n, int(without), _p(out)) != 0:
        raise ValueError(lib().or_last_error().decode())
    return out


# ------------------------------------------------------------------ fft -----
def dft(x) -> np.ndarray:
    """src/fft.cpp:90-97 (+ :121-126)."""
    y = _c128(x).copy()
    if y.size == 0:
        raise ValueError("Fft: length must be positive")
    lib().or_fft(_p(y), y.size, 0)
    return y


def idft(x) -> np.ndarray:
    """src/fft.cpp:99-110 (+ :128-131)."""
    y = _c128(x).copy()
    lib().or_fft(_p(y), y.size, 1)
    return y


# ----------------------------------------------------------------- srft -----
FIELDS = {"d": 0, "zeta": 1, "zeta_tilde": 2, "theta": 3, "theta_tilde": 4, "cos_theta": 5,
          "sin_theta": 6, "cos_theta_tilde": 7, "sin_theta_tilde": 8, "perm": 9,
          "perm_tilde": 10, "sample": 11}


class Srft:
    """SrftOperator (include/minnorm/srft.hpp:21-59) restated; built by
    build_srft (src/srft.cpp:95-113)."""

    def __init__(self, handle, l: int, n: int, without: bool):
        self._h = ctypes.c_void_p(handle)
        self.l, self.n, self.without = l, n, without

    @classmethod
    def build(cls, l: int, n: int, stream_seed: int, without: bool = True) -> "Srft":
        h = lib().or_srft_build(l, n, stream_seed, int(without))
        if not h:
            raise ValueError(lib().or_last_error().decode())
        return cls(h, l, n, without)

    @classmethod
    def from_fields(cls, l, n, d, sample, theta, theta_tilde, perm, perm_tilde, zeta, zeta_tilde,
                    without=True) -> "Srft":
        a = [_c128(d), np.ascontiguousarray(sample, np.int64), np.ascontiguousarray(theta, np.float64),
             np.ascontiguousarray(theta_tilde, np.float64), np.ascontiguousarray(perm, np.int64),
             np.ascontiguousarray(perm_tilde, np.int64), _c128(zeta), _c128(zeta_tilde)]
        h = lib().or_srft_from_fields(l, n, int(without), *[_p(v) for v in a])
        return cls(h, l, n, without)

    def __del__(self):
        try:
            if self._h:
                lib().or_srft_free(self._h)
        except Exception:
            pass

    def field(self, name: str) -> np.ndarray:
        f = FIELDS[name]
        if f <= 2:
            out = np.zeros(self.n, np.complex128)
        elif f <= 8:
            out = np.zeros(self.n - 1, np.float64)
        elif f <= 10:
            out = np.zeros(self.n, np.int64)
        else:
            out = np.zeros(self.l, np.int64)
        lib().or_srft_field(self._h, f, _p(out))
        return out

    def apply_h(self, x) -> np.ndarray:
        x = _c128(x)
        out = np.zeros(self.n, np.complex128)
        lib().or_srft_apply_h(self._h, _p(x), _p(out))
        return out

    def apply(self, x) -> np.ndarray:
        x = _c128(x)
        out = np.zeros(self.l, np.complex128)
        lib().or_srft_apply(self._h, _p(x), _p(out))
        return out

    def apply_adjoint(self, v) -> np.ndarray:
        v = _c128(v)
        out = np.zeros(self.n, np.complex128)
        lib().or_srft_apply_adjoint(self._h, _p(v), _p(out))
        return out

    def sketch(self, A: np.ndarray, row0: int = 0, nrows: int | None = None, threads: int | None = None):
        """T·A^H restricted to rows [row0,row0+nrows) of A (src/srft.cpp:147-153 on
        B = A^H, src/solver.cpp:76,81).  Returns l×nrows (column j = T·conj(A[row0+j,:]))."""
        A = _fortran(A)
        m, n = A.shape
        assert n == self.n
        nrows = m - row0 if nrows is None else nrows
        out = np.zeros((self.l, nrows), np.complex128, order="F")
        lib().or_srft_sketch_rows(self._h, _p(A), int(A.dtype == np.float64), m, row0, nrows, _p(out),
                                  threads or os.cpu_count() or 1)
        return out


def _fortran(A: np.ndarray) -> np.ndarray:
    if A.dtype not in (np.complex128, np.float64):
        A = A.astype(np.complex128)
    return np.asfortranarray(A)


# ---------------------------------------------------------- A products ------
def AH_v(A: np.ndarray, v: np.ndarray) -> np.ndarray:
    """B·v with B = A^H (n-vector), without forming B."""
    v = _c128(v)
    if A.dtype == np.float64:
        return (v.real @ A) + 1j * (v.imag @ A)
    return np.conj(np.conj(v) @ A)


def A_r(A: np.ndarray, r: np.ndarray) -> np.ndarray:
    """B^H·r = A·r (m-vector)."""
    r = _c128(r)
    if A.dtype == np.float64:
        return (A @ r.real) + 1j * (A @ r.imag)
    return A @ r


# ------------------------------------------------------------------ lsq -----
def deficient_count(R: np.ndarray, rows: int) -> int:
    """src/lsq.cpp:18-27 and src/solver.cpp:25-33."""
    dg = np.abs(np.diag(R))
    thr = float(rows) * EPS * (dg.max() if dg.size else 0.0)
    return int(np.sum((dg < thr) | (np.diag(R) == 0)))


def max_multiplicity(sample: np.ndarray) -> int:
    """src/lsq.cpp:31-39."""
    if sample.size == 0:
        return 1
    _, counts = np.unique(sample, return_counts=True)
    return int(max(1, counts.max()))


class RankDeficiencyError(RuntimeError):
    def __init__(self, what, deficient_columns):
        super().__init__(what)
        self.deficient_columns = deficient_columns


class ConfigError(ValueError):
    pass


class DimensionError(ValueError):
    pass


@dataclass
class LsqSolution:
    y: np.ndarray
    achieved_excess: float = 0.0
    iterations: int = 0
    converged: bool = False
    residual_norms: list = field(default_factory=list)
    R: np.ndarray | None = None


def solve_least_squares(A: np.ndarray, c: np.ndarray, sketch_size: int, tau: float,
                        max_iterations: int = 300, stream_seed: int = 42, without: bool = True,
                        threads: int | None = None, E: np.ndarray | None = None) -> LsqSolution:
    """src/lsq.cpp:43-113 with B = A^H (n×m).  `E` may pass a precomputed sketch."""
    m, n = A.shape
    c = _c128(c)
    if m < 1 or n <= m:
        raise ValueError("solve_least_squares: B must be tall (n > m >= 1)")
    if c.size != n:
        raise ValueError("solve_least_squares: c length mismatch")
    if sketch_size <= m or sketch_size > n:
        raise ValueError("solve_least_squares: sketch size must lie in (m, n]")
    if not tau > 0.0:
        raise ValueError("solve_least_squares: tau must be positive")
    if max_iterations < 1:
        raise ValueError("solve_least_squares: max_iterations must be at least 1")
    op = Srft.build(sketch_size, n, stream_seed, without)
    if E is None:
        E = op.sketch(A, threads=threads)                                 # lsq.cpp:55-56
    R = sla.qr(E, mode="r", overwrite_a=False, check_finite=False)[0][:m, :m]   # lsq.cpp:58-59
    bad = deficient_count(R, n)                                           # lsq.cpp:60-63
    if bad > 0:
        raise RankDeficiencyError(
            f"solve_least_squares: sketch QR found {bad} numerically dependent columns", bad)
    dup = float(max_multiplicity(op.field("sample")))                     # lsq.cpp:70

    def apply_m(u):                                                      # lsq.cpp:71
        return AH_v(A, sla.solve_triangular(R, u, lower=False, check_finite=False))

    def apply_m_adj(r):                                                  # lsq.cpp:72-74
        return sla.solve_triangular(R, A_r(A, r), trans="C", lower=False, check_finite=False)

    sol = LsqSolution(y=np.zeros(m, np.complex128), R=R)
    u = np.zeros(m, np.complex128)                                        # lsq.cpp:77-86
    r = c.copy()
    g = apply_m_adj(r)
    d = g.copy()
    gg = float(np.vdot(g, g).real)
    floor2 = 1e-28 * float(np.vdot(c, c).real)
    rr = float(np.vdot(r, r).real)
    excess = dup * gg
    sol.residual_norms.append(np.sqrt(rr))
    sol.converged = excess <= tau * max(rr - excess, 0.0) or rr <= floor2
    while not sol.converged and sol.iterations < max_iterations and gg > 0.0:   # lsq.cpp:88-107
        q = apply_m(d)
        qq = float(np.vdot(q, q).real)
        if qq == 0.0:
            break
        step = gg / qq
        u += step * d
        r -= step * q
        rr = float(np.vdot(r, r).real)
        sol.iterations += 1
        sol.residual_norms.append(np.sqrt(rr))
        g = apply_m_adj(r)
        gg_next = float(np.vdot(g, g).real)
        excess = dup * gg_next
        if excess <= tau * max(rr - excess, 0.0) or rr <= floor2:
            sol.converged = True
            break
        d = g + (gg_next / gg) * d
        gg = gg_next
    sol.y = sla.solve_triangular(R, u, lower=False, check_finite=False)    # lsq.cpp:109
    min_est = max(rr - excess, 0.0)
    sol.achieved_excess = excess / min_est if min_est > 0.0 else 0.0
    return sol


def least_squares_qr(A: np.ndarray, c: np.ndarray) -> np.ndarray:
    """src/lsq.cpp:115-128 on B = A^H (pivoted QR)."""
    B = np.conj(A).T
    n, m = B.shape
    Q, R, P = sla.qr(B, mode="economic", pivoting=True)
    bad = deficient_count(R, n)
    if bad > 0:
        raise RankDeficiencyError(f"least_squares_qr: {bad} numerically dependent columns", bad)
    z = sla.solve_triangular(R, np.conj(Q).T @ _c128(c), lower=False)
    y = np.zeros(m, np.complex128)
    y[P] = z
    return y


# --------------------------------------------------------------- solver -----
@dataclass
class SolveReport:
    """include/minnorm/solver.hpp:36-46"""
    x: np.ndarray
    step_seconds: list = field(default_factory=lambda: [0.0] * 5)
    c_norm_ratio: float = 0.0
    residual_norm: float = 0.0
    lsq_iterations: int = 0
    lsq_converged: bool = True
    sketch_size: int = 0
    lsq_tau: float = 0.0
    c: np.ndarray | None = None
    S: np.ndarray | None = None
    E_R: np.ndarray | None = None


def validate(A: np.ndarray, b: np.ndarray) -> None:
    """src/solver.cpp:37-48"""
    m, n = A.shape
    if m < 1 or m >= n:
        raise DimensionError(f"problem must be underdetermined: 1 <= m < n, got m={m}, n={n}")
    if b.size != m:
        raise DimensionError(f"right-hand side length {b.size} does not match m={m}")
    if not (np.all(np.isfinite(A)) and np.all(np.isfinite(b))):
        raise DimensionError("matrix and right-hand side entries must be finite")


def solve_randomized(A: np.ndarray, b: np.ndarray, sketch_size: int | None = None, alpha: float = 4.0,
                     epsilon: float = 1e-6, seed: int = 42, without: bool = True,
                     lsq_max_iterations: int = 300, capture_c: bool = False,
                     threads: int | None = None, keep: bool = False) -> SolveReport:
    """src/solver.cpp:50-128 (tags 11/12 at :19)."""
    A = _fortran(A)
    b = _c128(b)
    validate(A, b)
    m, n = A.shape
    if not (0.0 < epsilon < 1.0):
        raise ConfigError("epsilon must lie in (0, 1)")
    if not alpha > 1.0:
        raise ConfigError("alpha must exceed 1")
    l = 4 * m if sketch_size is None else int(sketch_size)
    if l <= m or l >= n:
        raise ConfigError(f"sketch size l={l} must satisfy m < l < n (m={m}, n={n})")
    rep = SolveReport(x=np.zeros(n, np.complex128), sketch_size=l,
                      lsq_tau=epsilon * epsilon * float(l) / (alpha * float(n)))
    if not np.any(b != 0):
        if capture_c:
            rep.c = np.zeros(n, np.complex128)
        return rep
    root_seed = seed
    # Step 1: S = T A*
    t0 = time.perf_counter()
    T = Srft.build(l, n, derive_seed(root_seed, 11), without)
    S = T.sketch(A, threads=threads)
    rep.step_seconds[0] = time.perf_counter() - t0
    # Step 2: z = Q [R^{-H} b; 0]
    t0 = time.perf_counter()
    Q, R = sla.qr(S, mode="economic", check_finite=False)
    bad = deficient_count(R, l)
    if bad > 0:
        raise RankDeficiencyError(f"sketch S = T A* lost rank ({bad} dependent columns); "
                                  "the problem matrix is rank deficient", bad)
    v = sla.solve_triangular(R, b, trans="C", lower=False, check_finite=False)
    z = Q @ v
    rep.step_seconds[1] = time.perf_counter() - t0
    # Step 3: c = T* z
    t0 = time.perf_counter()
    c = T.apply_adjoint(z)
    rep.step_seconds[2] = time.perf_counter() - t0
    # Step 4
    t0 = time.perf_counter()
    ls = solve_least_squares(A, c, l, rep.lsq_tau, lsq_max_iterations, derive_seed(root_seed, 12),
                             without, threads=threads)
    rep.lsq_iterations, rep.lsq_converged = ls.iterations, ls.converged
    rep.step_seconds[3] = time.perf_counter() - t0
    # Step 5
    t0 = time.perf_counter()
    rep.x = AH_v(A, ls.y)
    rep.step_seconds[4] = time.perf_counter() - t0
    rep.residual_norm = float(np.linalg.norm(A_r(A, rep.x) - b))
    xn = float(np.linalg.norm(rep.x))
    rep.c_norm_ratio = float(np.linalg.norm(c)) * np.sqrt(l / (alpha * n)) / xn if xn > 0 else 0.0
    if capture_c:
        rep.c = c
    if keep:
        rep.S, rep.E_R = S, ls.R
    return rep


def solve_classical(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    """src/solver.cpp:130-146: pivoted Householder QR of A*, x = Q (R*)^{-1} P* b."""
    A = _fortran(A)
    b = _c128(b)
    validate(A, b)
    m, n = A.shape
    if not np.any(b != 0):
        return np.zeros(n, np.complex128)
    Q, R, P = sla.qr(np.conj(A).T, mode="economic", pivoting=True)
    bad = deficient_count(R, n)
    if bad > 0:
        raise RankDeficiencyError(f"pivoted QR found rank deficiency ({bad} dependent columns)", bad)
    w = sla.solve_triangular(R, b[P], trans="C", lower=False)
    return Q @ w


def exact_minnorm(A: np.ndarray, b: np.ndarray, iters: int = 8, chunk: int = 1 << 13, G: np.ndarray | None = None):
    """The minimal-norm solution p = A^H (A A^H)^{-1} b of the float64 problem, to far below the
    float64 conditioning floor u*kappa: iterative refinement of A A^H y = b in y-space with the
    residual b - A (A^H y) and p = A^H y formed in x87 extended precision (u = 5.4e-20), the
    corrections solved with the float64 Cholesky factor of G = A A^H.  Each step contracts the
    error by ~u*kappa^2, so this converges for kappa up to ~1e7 (c1, c2, c4, the c5 analog); the
    extended-precision products make the result accurate to ~u_ext*kappa*sqrt(m).  Returns
    (p, history of relative residuals).  Not a restatement of the reference: the reference's
    own exact-p checks are the pivoted QR (solve_classical) and the SVD (solve_svd); this one
    exists to decide WHICH of two float64 solvers is closer to p at the floor.  `G` may pass a
    precomputed float64 A A^H (the full-size campaign forms it on the GPU)."""
    A = _fortran(A)
    m, n = A.shape
    real = A.dtype == np.float64
    ext = np.longdouble if real else np.clongdouble
    bl = _c128(b).astype(np.clongdouble)
    if G is None:
        G = (A @ A.T).astype(np.complex128) if real else A @ np.conj(A).T
    cf = sla.cho_factor(G, lower=False, check_finite=False)

    def chunk_products(c0, y):
        Ac = A[:, c0:c0 + chunk].astype(ext)  # column-major: y^H A_c runs along contiguous columns
        Ar = np.ascontiguousarray(Ac)          # row-major copy for A_c t
        if real:
            t = (y.real.astype(np.longdouble) @ Ac) + 1j * (y.imag.astype(np.longdouble) @ Ac)
            s = (Ar @ t.real) + 1j * (Ar @ t.imag)
        else:
            t = np.conj(np.conj(y) @ Ac)
            s = Ar @ t
        return c0, t, s

    def products(y):  # (A^H y, A A^H y) in extended precision, column chunks on host threads
        from concurrent.futures import ThreadPoolExecutor
        p = np.zeros(n, np.clongdouble)
        s = np.zeros(m, np.clongdouble)
        with ThreadPoolExecutor(max(1, os.cpu_count() or 1)) as ex:
            for c0, t, sc in ex.map(lambda c: chunk_products(c, y), range(0, n, chunk)):
                p[c0:c0 + chunk] = t
                s += sc  # fixed (chunk) order
        return p, s

    y = np.zeros(m, np.clongdouble)
    hist = []
    bn = float(np.linalg.norm(_c128(b)))
    r = bl
    for it in range(iters):
        rd = r.astype(np.complex128)
        hist.append(float(np.linalg.norm(rd)) / bn)
        if it >= 3 and hist[-1] > 0.1 * hist[-2] and hist[-2] > 0.1 * hist[-3]:
            break  # two steps at the floor of the extended-precision residual
        y = y + sla.cho_solve(cf, rd, check_finite=False).astype(np.clongdouble)
        p, s = products(y)
        r = bl - s
    hist.append(float(np.linalg.norm(r.astype(np.complex128))) / bn)
    return p.astype(np.complex128), hist


# ------------------------------------------------------- instance generator --
@dataclass
class GeneratedInstance:
    """include/minnorm/bench.hpp (GeneratedInstance): A = U diag(sigma) V^H, b = A p_true."""
    A: np.ndarray
    b: np.ndarray
    p_true: np.ndarray
    kappa: float


def _gaussian_matrix(stream_seed: int, rows: int, cols: int) -> np.ndarray:
    """src/bench.cpp:18-23: complex_gaussian() draws in column-major order."""
    return rng_draw(stream_seed, "complex_gaussian", rows * cols).reshape(cols, rows).T.copy()


def _orthonormalize_columns(X: np.ndarray) -> np.ndarray:
    """src/bench.cpp:26-37: modified Gram-Schmidt, two projection sweeps per column."""
    X = X.copy()
    for j in range(X.shape[1]):
        v = X[:, j].copy()
        for _ in range(2):
            for i in range(j):
                v -= np.vdot(X[:, i], v) * X[:, i]
        nv = np.linalg.norm(v)
        if not nv > 0.0:
            raise RuntimeError("orthonormalize_columns: degenerate Gaussian draw")
        X[:, j] = v / nv
    return X


def generate_instance(m: int, n: int, kappa: float, stream_seed: int) -> GeneratedInstance:
    """src/bench.cpp:46-74 (tags 21/22/23 at :16): sigma_j = kappa^{-j/(m-1)}, p_true = V w with
    w_j = sign/sqrt(m), b = A p_true.  `stream_seed` is the seed of the RandomStream passed in."""
    if m < 2:
        raise ValueError("generate_instance: m must be at least 2")
    if m >= n:
        raise ValueError("generate_instance: need m < n")
    if not kappa >= 1.0:
        raise ValueError("generate_instance: kappa must be >= 1")
    U = _orthonormalize_columns(_gaussian_matrix(derive_seed(stream_seed, 21), m, m))
    V = _orthonormalize_columns(_gaussian_matrix(derive_seed(stream_seed, 22), n, m))
    sigma = np.array([kappa ** (-float(j) / float(m - 1)) for j in range(m)])
    A = np.asfortranarray((U * sigma) @ np.conj(V).T)
    w = rng_draw(derive_seed(stream_seed, 23), "sign", m) * (1.0 / np.sqrt(float(m)))
    p = V @ w.astype(np.complex128)
    return GeneratedInstance(A=A, b=A @ p, p_true=p, kappa=kappa)


def normalized_error(x: np.ndarray, p_true: np.ndarray, kappa: float) -> float:
    """src/bench.cpp:76-80"""
    pn = float(np.linalg.norm(p_true))
    if not pn > 0.0:
        raise ValueError("normalized_error: p_true must be nonzero")
    return float(np.linalg.norm(x - p_true)) / (kappa * pn)


def bench_epsilon(kappa: float, m: int, l: int, alpha: float = 4.0) -> float:
    """src/bench.cpp:82-84"""
    return 1e-14 * kappa * np.sqrt(alpha * m / l)


def solve_svd(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    """src/solver.cpp:148-156 (desk-scale caps m<=64, n<=1024)."""
    A = _fortran(A)
    b = _c128(b)
    validate(A, b)
    if A.shape[0] > 64 or A.shape[1] > 1024:
        raise ValueError("solve_svd: desk-scale reference only (m <= 64, n <= 1024)")
    U, s, Vh = np.linalg.svd(A.astype(np.complex128), full_matrices=False)
    return np.conj(Vh).T @ ((np.conj(U).T @ b) / s)
