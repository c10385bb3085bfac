"""Thin ctypes binding of libbilu.so (include/bilu.h): argument marshalling only.

Every step of the numeric phase runs in the library's sm_100a kernels; there is
no CPU fallback -- if the library or a CUDA device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BILU_LIB", os.path.join(_HERE, "libbilu.so"))

STATUS = {0: "BILU_OK", 1: "BILU_ERR_ARG", 2: "BILU_ERR_BREAKDOWN", 3: "BILU_ERR_OOM",
          4: "BILU_ERR_CUDA", 5: "BILU_ERR_NCCL", 6: "BILU_ERR_STATE", 7: "BILU_ERR_NOT_BUILT"}

# every symbol include/bilu.h declares
ABI_SYMBOLS = ["bilu_options_default", "bilu_analyze", "bilu_set_values", "bilu_factor",
               "bilu_apply", "bilu_export", "bilu_factor_view_free", "bilu_destroy",
               "bilu_status_string", "bilu_last_error", "bilu_kernel_launches", "bilu_diag_dgemm", "bilu_diag_tsgemm",
               "bilu_dist_setup", "bilu_factor_local", "bilu_interface_pack", "bilu_interface_unpack",
               "bilu_factor_separators", "bilu_gmres", "bilu_ilu1_blocks",
               "bilu_cosine_blocks", "bilu_dist_separator_rows", "bilu_apply_dist_begin", "bilu_apply_dist_end",
               "bilu_mwm"]


class BiluError(RuntimeError):
    def __init__(self, status, msg, breakdown_block=-1):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status
        self.breakdown_block = breakdown_block


class Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("max_block", ctypes.c_int32),
                ("aggregate", ctypes.c_int32), ("n_ctas", ctypes.c_int32),
                ("near_rel", ctypes.c_double), ("arena_hint", ctypes.c_int64),
                ("stream", ctypes.c_void_p), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_comm", ctypes.c_void_p), ("perturb", ctypes.c_int32), ("perturb_tau", ctypes.c_double),
                ("perturb_rho", ctypes.c_double), ("cond_max", ctypes.c_double),
                ("zone_bytes", ctypes.c_int64)]


class FactorStats(ctypes.Structure):
    _fields_ = [("flops", ctypes.c_double), ("bytes_min", ctypes.c_double),
                ("t_factor_ms", ctypes.c_double), ("t_merge_ms", ctypes.c_double),
                ("nnz_L", ctypes.c_int64), ("nnz_U", ctypes.c_int64), ("nnz_D", ctypes.c_int64),
                ("n_blocks_init", ctypes.c_int32), ("n_blocks_final", ctypes.c_int32),
                ("n_merges", ctypes.c_int32), ("breakdown_block", ctypes.c_int32),
                ("n_retries", ctypes.c_int32), ("n_kernel_launches", ctypes.c_int32),
                ("n_decisions", ctypes.c_int64), ("n_near", ctypes.c_int64),
                ("min_margin", ctypes.c_double), ("n_perturbed", ctypes.c_int64),
                ("zone_blocks", ctypes.c_int32), ("zone_unknowns", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SolveStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("restarts", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("rel_residual", ctypes.c_double), ("t_solve_ms", ctypes.c_double),
                ("n_kernel_launches", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class FactorView(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("n_blocks", ctypes.c_int32),
                ("bstart", ctypes.POINTER(ctypes.c_int32)),
                ("Lp", ctypes.POINTER(ctypes.c_int64)), ("Li", ctypes.POINTER(ctypes.c_int32)),
                ("Lvp", ctypes.POINTER(ctypes.c_int64)), ("Lv", ctypes.POINTER(ctypes.c_double)),
                ("Up", ctypes.POINTER(ctypes.c_int64)), ("Ui", ctypes.POINTER(ctypes.c_int32)),
                ("Uvp", ctypes.POINTER(ctypes.c_int64)), ("Uv", ctypes.POINTER(ctypes.c_double)),
                ("Dp", ctypes.POINTER(ctypes.c_int64)), ("Dv", ctypes.POINTER(ctypes.c_double)),
                ("n_near", ctypes.c_int64),
                ("near_blk", ctypes.POINTER(ctypes.c_int32)), ("near_side", ctypes.POINTER(ctypes.c_int32)),
                ("near_idx", ctypes.POINTER(ctypes.c_int32)), ("near_keep", ctypes.POINTER(ctypes.c_int32)),
                ("near_margin", ctypes.POINTER(ctypes.c_double))]


_lib = None


def load_library():
    """Load libbilu.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libbilu.so not built (run __graft_entry__.build() or "
                          "python paper_1908_10169_b200/build.py)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    lib.bilu_options_default.argtypes = [ctypes.POINTER(Options)]
    lib.bilu_options_default.restype = None
    lib.bilu_analyze.argtypes = [ctypes.c_int32, P, P, P, P, P, ctypes.c_int32,
                                 ctypes.POINTER(Options), ctypes.POINTER(P)]
    lib.bilu_analyze.restype = ctypes.c_int
    lib.bilu_set_values.argtypes = [P, P, ctypes.c_int32]
    lib.bilu_set_values.restype = ctypes.c_int
    lib.bilu_factor.argtypes = [P, ctypes.c_double, ctypes.POINTER(FactorStats)]
    lib.bilu_factor.restype = ctypes.c_int
    lib.bilu_apply.argtypes = [P, P, P, P]
    lib.bilu_apply.restype = ctypes.c_int
    lib.bilu_export.argtypes = [P, ctypes.POINTER(FactorView)]
    lib.bilu_export.restype = ctypes.c_int
    lib.bilu_factor_view_free.argtypes = [ctypes.POINTER(FactorView)]
    lib.bilu_factor_view_free.restype = None
    lib.bilu_destroy.argtypes = [P]
    lib.bilu_destroy.restype = None
    lib.bilu_status_string.argtypes = [ctypes.c_int]
    lib.bilu_status_string.restype = ctypes.c_char_p
    lib.bilu_last_error.argtypes = [P]
    lib.bilu_last_error.restype = ctypes.c_char_p
    lib.bilu_kernel_launches.argtypes = [P]
    lib.bilu_kernel_launches.restype = ctypes.c_int64
    I64, D = ctypes.c_int64, ctypes.c_double
    lib.bilu_diag_dgemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, D, P, I64, I64, P, I64, I64, D, P,
                                    I64, I64, ctypes.c_int, I64, I64, I64, P]
    lib.bilu_diag_dgemm.restype = ctypes.c_int
    lib.bilu_diag_tsgemm.argtypes = lib.bilu_diag_dgemm.argtypes
    lib.bilu_diag_tsgemm.restype = ctypes.c_int
    lib.bilu_dist_setup.argtypes = [P, P, ctypes.c_int32]
    lib.bilu_dist_setup.restype = ctypes.c_int
    lib.bilu_factor_local.argtypes = [P, ctypes.c_double, ctypes.POINTER(FactorStats)]
    lib.bilu_factor_local.restype = ctypes.c_int
    lib.bilu_interface_pack.argtypes = [P, P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
    lib.bilu_interface_pack.restype = ctypes.c_int
    lib.bilu_interface_unpack.argtypes = [P, P, ctypes.c_int64]
    lib.bilu_interface_unpack.restype = ctypes.c_int
    lib.bilu_gmres.argtypes = [P, P, P, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(SolveStats)]
    lib.bilu_gmres.restype = ctypes.c_int
    lib.bilu_factor_separators.argtypes = [P, ctypes.POINTER(FactorStats)]
    lib.bilu_factor_separators.restype = ctypes.c_int
    lib.bilu_ilu1_blocks.argtypes = [ctypes.c_int32, P, P, P, P, D, ctypes.c_int32, ctypes.c_int32, P, P, P, P]
    lib.bilu_ilu1_blocks.restype = ctypes.c_int
    lib.bilu_cosine_blocks.argtypes = [ctypes.c_int32, P, P, D, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P]
    lib.bilu_cosine_blocks.restype = ctypes.c_int
    lib.bilu_mwm.argtypes = [ctypes.c_int32, P, P, P, ctypes.c_int32, P, P, P, P, P]
    lib.bilu_mwm.restype = ctypes.c_int
    lib.bilu_dist_separator_rows.argtypes = [P, ctypes.POINTER(ctypes.c_int64)]
    lib.bilu_dist_separator_rows.restype = ctypes.c_int
    lib.bilu_apply_dist_begin.argtypes = [P, P, P, P]
    lib.bilu_apply_dist_begin.restype = ctypes.c_int
    lib.bilu_apply_dist_end.argtypes = [P, P, P, ctypes.c_int32, P]
    lib.bilu_apply_dist_end.restype = ctypes.c_int
    _lib = lib
    return lib


def default_options(**kw) -> Options:
    lib = load_library()
    o = Options()
    lib.bilu_options_default(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


@dataclass
class Factor:
    """Host copy of the final factors (same layout as oracle.OracleFactor)."""
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
    near: np.ndarray  # rows (blk, side, idx, keep)
    near_margin: np.ndarray

    @property
    def nblk(self):
        return len(self.bstart) - 1

    def block(self, K):
        s, e = int(self.bstart[K]), int(self.bstart[K + 1])
        b = e - s
        rows = self.Li[self.Lp[K]:self.Lp[K + 1]]
        L = self.Lv[self.Lvp[K]:self.Lvp[K + 1]].reshape(len(rows), b)
        cols = self.Ui[self.Up[K]:self.Up[K + 1]]
        Ut = self.Uv[self.Uvp[K]:self.Uvp[K + 1]].reshape(len(cols), b).T
        D = self.Dv[self.Dp[K]:self.Dp[K + 1]].reshape(b, b).T
        return s, e, rows, L, cols, Ut, D


class BILU:
    """bilu_analyze / bilu_set_values / bilu_factor / bilu_apply / bilu_export."""

    def __init__(self, indptr, indices, data, block_sizes, perm=None, **opts):
        self.lib = load_library()
        self._keep = {}
        self.indptr = _arr(indptr, np.int64)
        self.indices = _arr(indices, np.int32)
        self.n = len(self.indptr) - 1
        self.nnz = int(self.indptr[-1])
        bs = _arr(block_sizes, np.int32)
        pm = None if perm is None else _arr(perm, np.int32)
        vals = None if data is None else _arr(data, np.float64)
        self.opt = default_options(**opts)
        h = ctypes.c_void_p()
        rc = self.lib.bilu_analyze(
            self.n, self.indptr.ctypes.data, self.indices.ctypes.data,
            None if vals is None else vals.ctypes.data,
            None if pm is None else pm.ctypes.data, bs.ctypes.data, len(bs),
            ctypes.byref(self.opt), ctypes.byref(h))
        if rc != 0:
            raise BiluError(rc, self.lib.bilu_last_error(None).decode())
        self.h = h
        self.stats = None

    def _check(self, rc, bb=-1):
        if rc != 0:
            raise BiluError(rc, self.lib.bilu_last_error(self.h).decode(), bb)

    def set_values(self, data=None, device_ptr=None):
        if device_ptr is not None:
            self._check(self.lib.bilu_set_values(self.h, ctypes.c_void_p(device_ptr), 1))
        else:
            vals = _arr(data, np.float64)
            self._keep["vals"] = vals
            self._check(self.lib.bilu_set_values(self.h, vals.ctypes.data, 0))

    def factor(self, tau) -> dict:
        st = FactorStats()
        rc = self.lib.bilu_factor(self.h, float(tau), ctypes.byref(st))
        self._check(rc, st.breakdown_block)
        self.stats = st.as_dict()
        return self.stats

    # ---- multi-GPU phases (include/bilu.h "multi-GPU factorization")
    def dist_setup(self, owner, rank: int):
        ow = np.ascontiguousarray(owner, dtype=np.int32)
        self._check(self.lib.bilu_dist_setup(self.h, ow.ctypes.data, int(rank)))

    def factor_local(self, tau) -> dict:
        st = FactorStats()
        rc = self.lib.bilu_factor_local(self.h, float(tau), ctypes.byref(st))
        self._check(rc, st.breakdown_block)
        return st.as_dict()

    def interface_pack(self, device=None):
        """This rank's packed interface panels as a CUDA uint8 tensor (torch owns the memory)."""
        import torch
        nb = ctypes.c_int64()
        self._check(self.lib.bilu_interface_pack(self.h, None, 0, ctypes.byref(nb)))
        buf = torch.empty(max(int(nb.value), 16), dtype=torch.uint8,
                          device=device if device is not None else "cuda:%d" % self.opt.device)
        self._check(self.lib.bilu_interface_pack(self.h, ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                                 ctypes.byref(nb)))
        return buf[:int(nb.value)]

    def interface_unpack(self, buf):
        """Append another rank's packed interface panels (CUDA uint8 tensor on this device)."""
        self._check(self.lib.bilu_interface_unpack(self.h, ctypes.c_void_p(buf.data_ptr()), int(buf.numel())))

    def factor_separators(self) -> dict:
        st = FactorStats()
        rc = self.lib.bilu_factor_separators(self.h, ctypes.byref(st))
        self._check(rc, st.breakdown_block)
        self.stats = st.as_dict()
        return self.stats

    def apply_dist_begin(self, x):
        """bilu_apply_dist_begin: forward sweep over this rank's subtrees; returns this rank's
        separator-row contributions (CUDA float64 tensor) to be summed over the ranks."""
        import torch
        m = ctypes.c_int64(0)
        self._check(self.lib.bilu_dist_separator_rows(self.h, ctypes.byref(m)))
        x = x.contiguous()
        contrib = torch.empty(max(m.value, 1), dtype=torch.float64, device=x.device)[: m.value]
        self._check(self.lib.bilu_apply_dist_begin(self.h, ctypes.c_void_p(x.data_ptr()),
                                                   ctypes.c_void_p(contrib.data_ptr()), None))
        return contrib

    def apply_dist_end(self, contrib_sum, write_separators: bool):
        """bilu_apply_dist_end: separator sweeps and the backward sweep; returns this rank's
        share of y (own subtree rows, separator rows if write_separators, 0 elsewhere)."""
        import torch
        contrib_sum = contrib_sum.contiguous()
        y = torch.empty(self.n, dtype=torch.float64, device=contrib_sum.device)
        self._check(self.lib.bilu_apply_dist_end(self.h, ctypes.c_void_p(contrib_sum.data_ptr()),
                                                 ctypes.c_void_p(y.data_ptr()), int(bool(write_separators)), None))
        return y

    def gmres(self, b, restart=30, tol=1e-8, max_restarts=100):
        """Solve A x = b on the device (bilu_gmres); b a CUDA float64 tensor in A's ordering.
        Returns (x tensor, stats dict)."""
        import torch
        b = b.contiguous()
        x = torch.empty_like(b)
        st = SolveStats()
        self._check(self.lib.bilu_gmres(self.h, ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                        int(restart), float(tol), int(max_restarts), ctypes.byref(st)))
        return x, st.as_dict()

    def apply(self, x_ptr: int, y_ptr: int, stream: int = 0):
        """y = M^{-1} x on DEVICE pointers (original ordering)."""
        self._check(self.lib.bilu_apply(self.h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                        ctypes.c_void_p(stream) if stream else None))

    def apply_tensor(self, x):
        """Convenience: torch CUDA tensor in, torch CUDA tensor out."""
        import torch
        x = x.contiguous()
        y = torch.empty_like(x)
        self.apply(x.data_ptr(), y.data_ptr())
        return y

    def export(self) -> Factor:
        v = FactorView()
        self._check(self.lib.bilu_export(self.h, ctypes.byref(v)))

        def cp(ptr, cnt, dt):
            if cnt == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(ptr, shape=(cnt,)).astype(dt, copy=True)
        nb = v.n_blocks
        Lp = cp(v.Lp, nb + 1, np.int64)
        Lvp = cp(v.Lvp, nb + 1, np.int64)
        Up = cp(v.Up, nb + 1, np.int64)
        Uvp = cp(v.Uvp, nb + 1, np.int64)
        Dp = cp(v.Dp, nb + 1, np.int64)
        nn = v.n_near
        near = np.stack([cp(v.near_blk, nn, np.int64), cp(v.near_side, nn, np.int64),
                         cp(v.near_idx, nn, np.int64), cp(v.near_keep, nn, np.int64)], axis=1) \
            if nn else np.zeros((0, 4), dtype=np.int64)
        out = Factor(n=v.n, bstart=cp(v.bstart, nb + 1, np.int64), Lp=Lp,
                     Li=cp(v.Li, int(Lp[-1]), np.int64), Lvp=Lvp, Lv=cp(v.Lv, int(Lvp[-1]), np.float64),
                     Up=Up, Ui=cp(v.Ui, int(Up[-1]), np.int64), Uvp=Uvp,
                     Uv=cp(v.Uv, int(Uvp[-1]), np.float64), Dp=Dp, Dv=cp(v.Dv, int(Dp[-1]), np.float64),
                     near=near, near_margin=cp(v.near_margin, nn, np.float64))
        self.lib.bilu_factor_view_free(ctypes.byref(v))
        return out

    def kernel_launches(self) -> int:
        return int(self.lib.bilu_kernel_launches(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.bilu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def diag_dgemm(A, B, C, alpha=1.0, beta=0.0, stream=0, tall_skinny=False):
    """C[b] = alpha A[b] B[b] + beta C[b] with the library's DMMA CTA GEMM (one CTA per
    batch entry).  A, B, C: CUDA float64 tensors of shape (batch, M, K), (batch, K, N),
    (batch, M, N), any strides.  Diagnostics only (tests, microbenchmarks)."""
    lib = load_library()
    bt, M, K = A.shape
    N = B.shape[2]
    fn = lib.bilu_diag_tsgemm if tall_skinny else lib.bilu_diag_dgemm
    rc = fn(M, N, K, alpha, A.data_ptr(), A.stride(1), A.stride(2), B.data_ptr(), B.stride(1),
                             B.stride(2), beta, C.data_ptr(), C.stride(1), C.stride(2), bt, A.stride(0),
                             B.stride(0), C.stride(0), ctypes.c_void_p(stream))
    if rc != 0:
        raise BiluError(rc, "bilu_diag_dgemm failed")


def ilu1_blocks(indptr, indices, data, tau, max_size=8, perm=None, device=0, stream=0):
    """bilu_ilu1_blocks: the ILU(1,tau) initial block partition of Sec. 3.4,
    computed on the device for Ã = A(perm, perm).  Returns (block_sizes int32 array, kernels launched)."""
    lib = load_library()
    ip = _arr(indptr, np.int64)
    ix = _arr(indices, np.int32)
    dv = _arr(data, np.float64)
    n = len(ip) - 1
    pm = None if perm is None else _arr(perm, np.int32)
    out = np.zeros(max(n, 1), dtype=np.int32)
    nb = ctypes.c_int32(0)
    nl = ctypes.c_int32(0)
    rc = lib.bilu_ilu1_blocks(n, ip.ctypes.data, ix.ctypes.data, dv.ctypes.data,
                              None if pm is None else pm.ctypes.data, float(tau), int(max_size), int(device),
                              ctypes.c_void_p(stream), out.ctypes.data, ctypes.byref(nb), ctypes.byref(nl))
    if rc != 0:
        raise BiluError(rc, lib.bilu_last_error(None).decode())
    return out[: nb.value].copy(), nl.value


def mwm(indptr, indices, data, device=0, stream=0):
    """bilu_mwm: maximum product transversal + scalings of Sec. 3.1 on the device.
    Returns (sigma int32 array: column matched to each row, dl, dr, kernels launched)."""
    lib = load_library()
    ip = _arr(indptr, np.int64)
    ix = _arr(indices, np.int32)
    dv = _arr(data, np.float64)
    n = len(ip) - 1
    sigma = np.zeros(max(n, 1), dtype=np.int32)
    dl = np.zeros(max(n, 1))
    dr = np.zeros(max(n, 1))
    nl = ctypes.c_int32(0)
    rc = lib.bilu_mwm(n, ip.ctypes.data, ix.ctypes.data, dv.ctypes.data, int(device), ctypes.c_void_p(stream),
                      sigma.ctypes.data, dl.ctypes.data, dr.ctypes.data, ctypes.byref(nl))
    if rc != 0:
        raise BiluError(rc, lib.bilu_last_error(None).decode())
    return sigma[:n].copy(), dl[:n].copy(), dr[:n].copy(), nl.value


def cosine_blocks(indptr, indices, tau=0.8, max_size=128, device=0, stream=0):
    """bilu_cosine_blocks: cosine-based blocking of Sec. 3.2 on the device.
    Returns (q new->old int32 array, block sizes int32 array, kernels launched)."""
    lib = load_library()
    ip = _arr(indptr, np.int64)
    ix = _arr(indices, np.int32)
    n = len(ip) - 1
    q = np.zeros(max(n, 1), dtype=np.int32)
    out = np.zeros(max(n, 1), dtype=np.int32)
    nb = ctypes.c_int32(0)
    nl = ctypes.c_int32(0)
    rc = lib.bilu_cosine_blocks(n, ip.ctypes.data, ix.ctypes.data, float(tau), int(max_size), int(device),
                                ctypes.c_void_p(stream), q.ctypes.data, out.ctypes.data, ctypes.byref(nb),
                                ctypes.byref(nl))
    if rc != 0:
        raise BiluError(rc, lib.bilu_last_error(None).decode())
    return q[:n].copy(), out[: nb.value].copy(), nl.value
