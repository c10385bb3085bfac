"""CPU oracle for the BILU numeric phase -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_1908_10169_b200``) never imports it and shares no code with it.

The arithmetic lives in ``bilu_oracle.c`` (plain C, fp64 scalar loops, no BLAS);
this module only builds it with gcc and marshals arguments (ctypes).  Each C
function cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bilu_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "bilu_oracle.h"))
    ):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-D_POSIX_C_SOURCE=199309L", "-shared", "-fPIC",
             "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class _Factor(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("nblk", ctypes.c_int32),
        ("bstart", ctypes.POINTER(ctypes.c_int32)),
        ("Lp", ctypes.POINTER(ctypes.c_int64)), ("Li", ctypes.POINTER(ctypes.c_int32)),
        ("Lvp", ctypes.POINTER(ctypes.c_int64)), ("Lv", ctypes.POINTER(ctypes.c_double)),
        ("Up", ctypes.POINTER(ctypes.c_int64)), ("Ui", ctypes.POINTER(ctypes.c_int32)),
        ("Uvp", ctypes.POINTER(ctypes.c_int64)), ("Uv", ctypes.POINTER(ctypes.c_double)),
        ("Dp", ctypes.POINTER(ctypes.c_int64)), ("Dv", ctypes.POINTER(ctypes.c_double)),
        ("flops", ctypes.c_double), ("t_factor_s", ctypes.c_double),
        ("n_merges", ctypes.c_int32), ("breakdown_block", ctypes.c_int32),
        ("n_decisions", ctypes.c_int64), ("n_near", ctypes.c_int64),
        ("min_margin", ctypes.c_double), ("n_perturbed", ctypes.c_int64),
        ("n_override_applied", ctypes.c_int64),
    ]


class _Perturb(ctypes.Structure):
    _fields_ = [("perturb", ctypes.c_int32), ("tau", ctypes.c_double), ("rho", ctypes.c_double),
                ("cond_max", ctypes.c_double)]


class _Override(ctypes.Structure):
    _fields_ = [("blk", ctypes.c_int32), ("side", ctypes.c_int32),
                ("idx", ctypes.c_int32), ("keep", ctypes.c_int32)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.orc_bilu_factor.restype = ctypes.c_int
        lib.orc_bilu_factor.argtypes = [
            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int32, ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(_Factor),
        ]
        lib.orc_bilu_factor_seg.restype = ctypes.c_int
        lib.orc_bilu_factor_seg.argtypes = [
            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int32, ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.POINTER(_Factor),
        ]
        lib.orc_bilu_factor_pt.restype = ctypes.c_int
        lib.orc_bilu_factor_pt.argtypes = [
            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int32, ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.POINTER(_Perturb),
            ctypes.POINTER(_Factor),
        ]
        lib.orc_ilu1_blocks.restype = ctypes.c_int32
        lib.orc_ilu1_blocks.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_double, ctypes.c_int32, ctypes.c_void_p]
        lib.orc_ilu1_set.restype = ctypes.c_int32
        lib.orc_ilu1_set.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        lib.orc_cosine_blocks.restype = ctypes.c_int32
        lib.orc_cosine_blocks.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                          ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        lib.orc_mwm.restype = ctypes.c_int
        lib.orc_mwm.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.orc_bilu_apply.restype = ctypes.c_int
        lib.orc_bilu_apply.argtypes = [ctypes.POINTER(_Factor), ctypes.c_void_p, ctypes.c_void_p]
        lib.orc_aggregate_test.restype = ctypes.c_int
        lib.orc_aggregate_test.argtypes = [ctypes.c_int64] * 11
        lib.orc_free.restype = None
        lib.orc_free.argtypes = [ctypes.POINTER(_Factor)]
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    pass


@dataclass
class OracleFactor:
    """Final (post-aggregation) factors in the permuted ordering.

    Per final block K (rows/cols [bstart[K], bstart[K+1])):
      L rows  Li[Lp[K]:Lp[K+1]]  panel Lv[Lvp[K]:Lvp[K+1]] (m x b row-major)
      Ũ cols  Ui[Up[K]:Up[K+1]]  panel Uv[Uvp[K]:Uvp[K+1]] (b x c column-major)
      D_K     Dv[Dp[K]:Dp[K+1]]  (b x b column-major), D_K = P_K^{-1}
    """
    n: int
    bstart: np.ndarray
    Lp: np.ndarray
    Li: np.ndarray
    Lvp: np.ndarray
    Lv: np.ndarray
    Up: np.ndarray
    Ui: np.ndarray
    Uvp: np.ndarray
    Uv: np.ndarray
    Dp: np.ndarray
    Dv: np.ndarray
    flops: float = 0.0
    t_factor_s: float = 0.0
    n_merges: int = 0
    n_decisions: int = 0
    n_near: int = 0
    min_margin: float = float("inf")
    n_perturbed: int = 0
    n_override_applied: int = 0
    _keep: object = field(default=None, repr=False)

    @property
    def nblk(self) -> int:
        return len(self.bstart) - 1

    def block(self, K: int):
        s, e = int(self.bstart[K]), int(self.bstart[K + 1])
        b = e - s
        rows = self.Li[self.Lp[K]:self.Lp[K + 1]]
        L = self.Lv[self.Lvp[K]:self.Lvp[K + 1]].reshape(len(rows), b)
        cols = self.Ui[self.Up[K]:self.Up[K + 1]]
        Ut = self.Uv[self.Uvp[K]:self.Uvp[K + 1]].reshape(len(cols), b).T
        D = self.Dv[self.Dp[K]:self.Dp[K + 1]].reshape(b, b).T
        return s, e, rows, L, cols, Ut, D


def _np(ptr, count, dtype):
    if count == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)


def factor(indptr, indices, data, block_sizes, tau, aggregate=True, max_block=128,
           overrides=None, near_rel=1e-8, seg=None, perturb=None) -> OracleFactor:
    """Run the oracle on an already-permuted CSR matrix (Ã).  seg: optional aggregation
    segment per initial block (merges only inside a segment, R18).  perturb:
    None (off) or (tau_p, rho, cond_max) for the Sec. 3.6 perturbation (R19)."""
    lib = _load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    data = np.ascontiguousarray(data, dtype=np.float64)
    bsz = np.ascontiguousarray(block_sizes, dtype=np.int32)
    n = len(indptr) - 1
    ov = None
    nov = 0
    if overrides:
        arr = (_Override * len(overrides))()
        for i, (blk, side, idx, keep) in enumerate(overrides):
            arr[i] = _Override(int(blk), int(side), int(idx), int(keep))
        ov = ctypes.cast(arr, ctypes.c_void_p)
        nov = len(overrides)
    f = _Factor()
    if perturb is not None:
        pt = _Perturb(1, float(perturb[0]), float(perturb[1]), float(perturb[2]))
        sg = None if seg is None else np.ascontiguousarray(seg, dtype=np.int32)
        rc = lib.orc_bilu_factor_pt(
            n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data,
            len(bsz), bsz.ctypes.data, float(tau), int(bool(aggregate)), int(max_block),
            ov, nov, float(near_rel), None if sg is None else sg.ctypes.data, ctypes.byref(pt), ctypes.byref(f))
    elif seg is None:
        rc = lib.orc_bilu_factor(
            n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data,
            len(bsz), bsz.ctypes.data, float(tau), int(bool(aggregate)), int(max_block),
            ov, nov, float(near_rel), ctypes.byref(f))
    else:
        sg = np.ascontiguousarray(seg, dtype=np.int32)
        if len(sg) != len(bsz):
            raise OracleError("seg must have one entry per initial block")
        rc = lib.orc_bilu_factor_seg(
            n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data,
            len(bsz), bsz.ctypes.data, float(tau), int(bool(aggregate)), int(max_block),
            ov, nov, float(near_rel), sg.ctypes.data, ctypes.byref(f))
    if rc != 0:
        bb = f.breakdown_block
        lib.orc_free(ctypes.byref(f))
        raise OracleError({1: "bad argument", 2: "breakdown in block %d" % bb,
                           3: "out of memory",
                           5: "override refused: it names a decision farther than 1e-6 relative from tau "
                              "(only near-threshold decisions may be replayed, DESIGN.md R15)"}.get(rc, "error %d" % rc))
    nb = f.nblk
    bstart = _np(f.bstart, nb + 1, np.int64)
    Lp = _np(f.Lp, nb + 1, np.int64)
    Lvp = _np(f.Lvp, nb + 1, np.int64)
    Up = _np(f.Up, nb + 1, np.int64)
    Uvp = _np(f.Uvp, nb + 1, np.int64)
    Dp = _np(f.Dp, nb + 1, np.int64)
    out = OracleFactor(
        n=f.n, bstart=bstart, Lp=Lp, Li=_np(f.Li, int(Lp[-1]), np.int64), Lvp=Lvp,
        Lv=_np(f.Lv, int(Lvp[-1]), np.float64), Up=Up, Ui=_np(f.Ui, int(Up[-1]), np.int64),
        Uvp=Uvp, Uv=_np(f.Uv, int(Uvp[-1]), np.float64), Dp=Dp,
        Dv=_np(f.Dv, int(Dp[-1]), np.float64), flops=f.flops, t_factor_s=f.t_factor_s,
        n_merges=f.n_merges, n_decisions=f.n_decisions, n_near=f.n_near,
        min_margin=f.min_margin, n_perturbed=f.n_perturbed, n_override_applied=f.n_override_applied)
    lib.orc_free(ctypes.byref(f))
    return out


def _as_struct(fac: OracleFactor):
    """Re-expose an OracleFactor to C (for orc_bilu_apply)."""
    keep = {
        "bstart": np.ascontiguousarray(fac.bstart, dtype=np.int32),
        "Lp": np.ascontiguousarray(fac.Lp, dtype=np.int64),
        "Li": np.ascontiguousarray(fac.Li, dtype=np.int32),
        "Lvp": np.ascontiguousarray(fac.Lvp, dtype=np.int64),
        "Lv": np.ascontiguousarray(fac.Lv, dtype=np.float64),
        "Up": np.ascontiguousarray(fac.Up, dtype=np.int64),
        "Ui": np.ascontiguousarray(fac.Ui, dtype=np.int32),
        "Uvp": np.ascontiguousarray(fac.Uvp, dtype=np.int64),
        "Uv": np.ascontiguousarray(fac.Uv, dtype=np.float64),
        "Dp": np.ascontiguousarray(fac.Dp, dtype=np.int64),
        "Dv": np.ascontiguousarray(fac.Dv, dtype=np.float64),
    }
    f = _Factor()
    f.n = fac.n
    f.nblk = fac.nblk
    for k, arr in keep.items():
        ctype = {np.int32: ctypes.c_int32, np.int64: ctypes.c_int64,
                 np.float64: ctypes.c_double}[arr.dtype.type]
        setattr(f, k, arr.ctypes.data_as(ctypes.POINTER(ctype)))
    return f, keep


def apply(fac: OracleFactor, x: np.ndarray) -> np.ndarray:
    """y = (L P U)^{-1} x in the permuted ordering."""
    lib = _load()
    f, keep = _as_struct(fac)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(fac.n, dtype=np.float64)
    rc = lib.orc_bilu_apply(ctypes.byref(f), x.ctypes.data, y.ctypes.data)
    if rc != 0:
        raise OracleError("apply failed")
    del keep
    return y


def aggregate_test(p, q, r, s, t, r2, s2, t2, u, v, max_block=128) -> bool:
    return bool(_load().orc_aggregate_test(p, q, r, s, t, r2, s2, t2, u, v, max_block))


def permute_csr(indptr, indices, data, perm):
    """Ã = A(perm, perm) as sorted CSR (plain scipy; the oracle side of the input
    permutation -- the CUDA path does its own inside bilu_analyze)."""
    import scipy.sparse as sp
    n = len(indptr) - 1
    A = sp.csr_matrix((data, indices, indptr), shape=(n, n))
    if perm is not None:
        perm = np.asarray(perm)
        A = A[perm][:, perm]
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float64)


def ilu1_blocks(indptr, indices, data, tau, max_size=8) -> np.ndarray:
    """ILU(1,tau) initial block sizes of Sec. 3.4 (R20) of an already-permuted CSR matrix."""
    lib = _load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    data = np.ascontiguousarray(data, dtype=np.float64)
    n = len(indptr) - 1
    out = np.zeros(n, dtype=np.int32)
    nb = lib.orc_ilu1_blocks(n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, float(tau),
                             int(max_size), out.ctypes.data)
    if nb < 0:
        raise OracleError("bad argument")
    return out[:nb].copy()


def ilu1_set(indptr, indices, data, tau, k, lower=True) -> np.ndarray:
    """Estimated pattern I~_k (lower) or J~_k of Sec. 3.4, ascending."""
    lib = _load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    data = np.ascontiguousarray(data, dtype=np.float64)
    n = len(indptr) - 1
    out = np.zeros(n, dtype=np.int32)
    m = lib.orc_ilu1_set(n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, float(tau), int(k),
                         1 if lower else 0, out.ctypes.data)
    if m < 0:
        raise OracleError("bad argument")
    return out[:m].copy()


def cosine_blocks(indptr, indices, tau=0.8, max_size=128):
    """Cosine-based blocking of Sec. 3.2 (R21): (q new->old, group sizes)."""
    lib = _load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    n = len(indptr) - 1
    q = np.zeros(n, dtype=np.int32)
    sizes = np.zeros(n, dtype=np.int32)
    nb = lib.orc_cosine_blocks(n, indptr.ctypes.data, indices.ctypes.data, float(tau), int(max_size),
                               q.ctypes.data, sizes.ctypes.data)
    if nb < 0:
        raise OracleError("bad argument")
    return q, sizes[:nb].copy()


def mwm(indptr, indices, data):
    """Maximum product transversal + scalings of Sec. 3.1 (R22): (sigma, dl, dr) with
    sigma[i] the column matched to row i; |dl_i a_ij dr_j| <= 1, = 1 on the matching."""
    lib = _load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    data = np.ascontiguousarray(data, dtype=np.float64)
    n = len(indptr) - 1
    sigma = np.zeros(n, dtype=np.int32)
    dl = np.zeros(n)
    dr = np.zeros(n)
    rc = lib.orc_mwm(n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, sigma.ctypes.data,
                     dl.ctypes.data, dr.ctypes.data)
    if rc == -2:
        raise OracleError("structurally singular: no perfect matching")
    if rc != 0:
        raise OracleError("bad argument")
    return sigma, dl, dr
