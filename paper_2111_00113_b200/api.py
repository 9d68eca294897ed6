"""Python API over the C-ABI (same names as include/sks.h without the ``sks_`` prefix).

Marshalling only: arrays may be torch tensors (CUDA or CPU) or numpy arrays; their
pointers are passed straight to libsks, which detects host vs device memory.  Output
arrays live where the main input lives (device in -> device out, host in -> host out).
"""
import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

try:
    import torch
except Exception:  # pragma: no cover - torch is part of the image
    torch = None


class SksError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{L.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _is_torch(a):
    return torch is not None and isinstance(a, torch.Tensor)


def _prep(a, dtype=np.float64):
    """-> (object kept alive, pointer) for a contiguous array of `dtype`."""
    if a is None:
        return None, None
    if _is_torch(a):
        tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int8: torch.int8}[dtype]
        t = a.detach()
        if t.dtype != tdt:
            t = t.to(tdt)
        t = t.contiguous()
        return t, t.data_ptr()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr, arr.ctypes.data


def _check_out(out, n):
    """`out` receives n float64 values through its raw pointer: it must be a contiguous float64
    array of exactly n elements (torch tensor on any device, or numpy)."""
    if _is_torch(out):
        ok = out.dtype == torch.float64 and out.is_contiguous() and out.numel() == n and out.dim() == 1
    elif isinstance(out, np.ndarray):
        ok = out.dtype == np.float64 and out.flags["C_CONTIGUOUS"] and out.size == n and out.ndim == 1
    else:
        ok = False
    if not ok:
        raise ValueError(f"out must be a contiguous 1-D float64 array of length {n}")


def _empty_like_place(ref, shape, dtype=np.float64):
    if _is_torch(ref):
        tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int8: torch.int8}[dtype]
        pin = ref.device.type == "cpu"
        t = torch.empty(shape, dtype=tdt, device=ref.device, pin_memory=pin and torch.cuda.is_available())
        return t, t.data_ptr()
    arr = np.empty(shape, dtype=dtype)
    return arr, arr.ctypes.data


@dataclass
class StencilOperator:
    """-Lap(u) + beta (d/dx + d/dy [+ d/dz]) u on an m^dim Dirichlet grid (reading O18)."""
    dim: int
    m: int
    beta: float
    row_begin: int = 0
    row_end: int = None

    @property
    def n_global(self):
        return self.m ** self.dim

    def struct(self):
        rb = self.row_begin
        re = self.n_global if self.row_end is None else self.row_end
        kind = L.SKS_OP_STENCIL2D if self.dim == 2 else L.SKS_OP_STENCIL3D
        return L.Operator(kind, 0, self.m, float(self.beta), self.n_global, rb, re, None, None, None, 0), ()


@dataclass
class CsrOperator:
    """Rows [row_begin, row_end) of a general sparse A; col_idx are GLOBAL int32 indices."""
    row_ptr: object
    col_idx: object
    val: object
    n_global: int
    row_begin: int = 0
    row_end: int = None

    def struct(self):
        rp, prp = _prep(self.row_ptr, np.int32)
        ci, pci = _prep(self.col_idx, np.int32)
        va, pva = _prep(self.val, np.float64)
        re = self.n_global if self.row_end is None else self.row_end
        nnz = int(rp[-1])
        return L.Operator(L.SKS_OP_CSR, 0, 0, 0.0, self.n_global, self.row_begin, re, prp, pci, pva, nnz), (rp, ci, va)


def partition(kind: str, m: int, n_global: int, nranks: int, rank: int):
    lib = L.load()
    k = {"stencil2d": L.SKS_OP_STENCIL2D, "stencil3d": L.SKS_OP_STENCIL3D, "csr": L.SKS_OP_CSR}[kind]
    lo, hi = C.c_int64(), C.c_int64()
    st = lib.sks_partition(k, m, n_global, nranks, rank, C.byref(lo), C.byref(hi))
    if st != 0:
        raise SksError(st, "sks_partition")
    return lo.value, hi.value


def get_unique_id() -> bytes:
    lib = L.load()
    buf = (C.c_ubyte * 128)()
    st = lib.sks_get_unique_id(buf)
    if st != 0:
        raise SksError(st, lib.sks_last_error(None).decode())
    return bytes(buf)


class LoopbackGroup:
    """sks_loopback: `nranks` contexts of ONE process (one thread per rank, one device) exchanging through
    device-to-device copies instead of NCCL (include/sks.h).  Destroy every Context before the group."""

    def __init__(self, nranks: int):
        self.lib = L.load()
        self.h = C.c_void_p()
        st = self.lib.sks_loopback_create(nranks, C.byref(self.h))
        if st != 0:
            raise SksError(st, "sks_loopback_create")
        self.nranks = nranks

    def close(self):
        if self.h:
            self.lib.sks_loopback_destroy(self.h)
            self.h = C.c_void_p()


class Context:
    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, nccl_id: bytes = None,
                 loopback: LoopbackGroup = None):
        self.lib = L.load()
        self.h = C.c_void_p()
        idp = None
        if nccl_id is not None:
            self._id = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            idp = C.addressof(self._id)
        if loopback is not None:
            nranks = loopback.nranks
            st = self.lib.sks_create_loopback(C.byref(self.h), device, rank, loopback.h)
        else:
            st = self.lib.sks_create(C.byref(self.h), device, rank, nranks, idp)
        if st != 0:
            raise SksError(st, self.lib.sks_last_error(None).decode())
        self.device, self.rank, self.nranks = device, rank, nranks

    def close(self):
        if self.h:
            self.lib.sks_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st, what, allow=()):
        if st != 0 and st not in allow:
            raise SksError(st, f"{what}: {self.lib.sks_last_error(self.h).decode()}")
        return st

    def set_stream(self, stream=None):
        """Run the main work on `stream` (torch.cuda.Stream, raw handle, or None)."""
        h = None
        if stream is not None:
            h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._check(self.lib.sks_set_stream(self.h, h), "sks_set_stream")

    # ---------------------------------------------------------------- sGMRES
    def sgmres_solve(self, A, f, x0=None, *, d, k, s, zeta=8, seed=0, tol=1e-8, max_cycles=50,
                     early_exit_factor=0.25, cond_tol=1e14, sketch_batch=0, hist_cap=None, time_steps=False, time_stride=1,
                     basis="arnoldi", cheb=None, adaptive_restart=False, out=None, sketch="sparse", whiten=False):
        op, keep = A.struct()
        fa, pf = _prep(f)
        n = fa.shape[0]
        zero_x0 = x0 is None
        if out is not None:
            # the solution is written into `out` (a pinned host `out` keeps the library's copy at full
            # DMA speed); x0 (if given and not `out` itself) is copied into it first.  The library writes
            # n doubles through the raw pointer, so `out` must be exactly that.
            _check_out(out, n)
            x = out
            if x0 is not None and x0 is not out:
                if _is_torch(x):
                    x.copy_(x0 if _is_torch(x0) else torch.from_numpy(np.asarray(x0, dtype=np.float64)))
                else:
                    x[...] = x0.cpu().numpy() if _is_torch(x0) else x0
        elif x0 is None:  # x0 = 0 is not copied to the device (SKS_OPT_ZERO_X0)
            x = torch.empty_like(fa) if _is_torch(fa) else np.empty(n)
        else:
            x = (x0.detach().clone().to(torch.float64).contiguous() if _is_torch(x0)
                 else np.array(x0, dtype=np.float64, copy=True))
        px = x.data_ptr() if _is_torch(x) else x.ctypes.data
        cap = hist_cap or (d * max_cycles + 8)
        hist = np.zeros(cap)
        hist_true = np.zeros(max_cycles + 2)
        cc, cdx, cdy = cheb if cheb is not None else (0.0, 0.0, 0.0)
        opts = L.SgmresOpts(d, k, s, zeta, seed, tol, max_cycles, sketch_batch, early_exit_factor, cond_tol,
                            (L.SKS_OPT_TIME_STEPS if time_steps else 0)
                            | (L.SKS_OPT_ADAPTIVE_RESTART if adaptive_restart else 0)
                            | (L.SKS_OPT_WHITEN if whiten else 0)
                            | (L.SKS_OPT_ZERO_X0 if zero_x0 else 0), time_stride, L.BASES[basis],
                            L.SKETCHES[sketch],
                            cc, cdx, cdy)
        info = L.SgmresInfo()
        st = self.lib.sks_sgmres_solve(self.h, C.byref(op), pf, px, C.byref(opts), C.byref(info),
                                       hist.ctypes.data, cap, hist_true.ctypes.data, len(hist_true))
        self._check(st, "sks_sgmres_solve", allow=(L.SKS_ENOTCONV,))
        inf = {k_: getattr(info, k_) for k_, _ in info._fields_}
        nh = min(cap, inf["columns"])
        return SgmresResult(x=x, hist=hist[:nh], hist_true=hist_true[:inf["cycles"]], info=inf,
                            converged=(st == 0))

    # ---------------------------------------------------------------- sRR
    def srr_eigs(self, A, v0, *, d, k, s, nev, zeta=8, seed=0, cond_tol=1e14, want_vectors=False,
                 basis="arnoldi", cheb=None, sketch="sparse", stabilize="off", block=0):
        """stabilize: "off", "if_ill" (kappa(T) > cond_tol, Alg. 2) or "always": truncated-SVD
        pencil of Sec. "Stabilization", keeping sigma_i >= sigma_1 / cond_tol.
        basis="block_chebyshev": v0 is the n x b start block Omega (numpy/torch, b = block columns), the
        basis is the block Chebyshev recurrence of depth d / b."""
        op, keep = A.struct()
        if basis == "block_chebyshev":
            # n x b start block -> column-major (each column contiguous): pass its transpose, C-contiguous
            if _is_torch(v0):
                vt = v0.detach().to(torch.float64)
                vt = vt.reshape(-1, 1) if vt.dim() == 1 else vt
                block = vt.shape[1]
                va = vt.t().contiguous()
                pv = va.data_ptr()
                n = vt.shape[0]
            else:
                vt = np.asarray(v0, dtype=np.float64)
                vt = vt.reshape(-1, 1) if vt.ndim == 1 else vt
                block = vt.shape[1]
                va = np.ascontiguousarray(vt.T)
                pv = va.ctypes.data
                n = vt.shape[0]
        else:
            va, pv = _prep(v0)
            n = va.shape[0]
        cap = nev + 1
        th_re, th_im, rt, re = (np.zeros(cap) for _ in range(4))
        Xr = Xi = None
        pxr = pxi = None
        if want_vectors:
            Xr, pxr = _empty_like_place(va, (cap, n))
            Xi, pxi = _empty_like_place(va, (cap, n))
        cc, cdx, cdy = cheb if cheb is not None else (0.0, 0.0, 0.0)
        opts = L.SrrOpts(d, k, s, zeta, seed, cond_tol, L.BASES[basis], L.SKETCHES[sketch],
                         L.STABILIZE[stabilize], int(block), cc, cdx, cdy)
        info = L.SrrInfo()
        st = self.lib.sks_srr_eigs(self.h, C.byref(op), pv, C.byref(opts), nev, cap, th_re.ctypes.data,
                                   th_im.ctypes.data, rt.ctypes.data, re.ctypes.data, pxr, pxi, C.byref(info))
        self._check(st, "sks_srr_eigs")
        inf = {k_: getattr(info, k_) for k_, _ in info._fields_}
        m = inf["nev_out"]
        out = dict(theta=th_re[:m] + 1j * th_im[:m], res_true=rt[:m], res_est=re[:m], info=inf)
        if want_vectors:
            out["X"] = (Xr[:m], Xi[:m])
        return out

    # ---------------------------------------------------------------- parity entry points
    def sketch_apply(self, M, *, s, zeta, seed, cycle=0, n_global=None, row_begin=0):
        Ma, pm = _prep(M)
        if Ma.ndim == 1:
            Ma = Ma.reshape(-1, 1) if not _is_torch(Ma) else Ma.reshape(-1, 1)
        n, c = Ma.shape
        # column-major n x c: pass the transpose-contiguous copy
        Mt = Ma.t().contiguous() if _is_torch(Ma) else np.ascontiguousarray(Ma.T)
        pm = Mt.data_ptr() if _is_torch(Mt) else Mt.ctypes.data
        ng = row_begin + n if n_global is None else n_global
        SM, psm = _empty_like_place(Ma, (c, s))
        st = self.lib.sks_sketch_apply(self.h, ng, row_begin, row_begin + n, s, zeta, seed, cycle, pm, n, c, psm)
        self._check(st, "sks_sketch_apply")
        return SM.t() if _is_torch(SM) else SM.T

    def srft_apply(self, M, *, s, seed, cycle=0):
        """S M for the SRFT sketch (include/sks.h sks_srft_apply, reading O32)."""
        Ma, _ = _prep(M)
        if Ma.ndim == 1:
            Ma = Ma.reshape(-1, 1)
        n, c = Ma.shape
        Mt = Ma.t().contiguous() if _is_torch(Ma) else np.ascontiguousarray(Ma.T)
        pm = Mt.data_ptr() if _is_torch(Mt) else Mt.ctypes.data
        SM, psm = _empty_like_place(Ma, (c, s))
        self._check(self.lib.sks_srft_apply(self.h, n, s, seed, cycle, pm, c, psm), "sks_srft_apply")
        return SM.t() if _is_torch(SM) else SM.T

    def sketch_table(self, row_begin, count, *, s, zeta, seed, cycle=0):
        q = np.zeros(count * zeta, dtype=np.int32)
        sg = np.zeros(count * zeta, dtype=np.int8)
        st = self.lib.sks_sketch_table(self.h, row_begin, count, s, zeta, seed, cycle, q.ctypes.data,
                                       sg.ctypes.data)
        self._check(st, "sks_sketch_table")
        return q.reshape(count, zeta), sg.reshape(count, zeta)

    def apply_operator(self, A, x):
        op, keep = A.struct()
        xa, px = _prep(x)
        y, py = _empty_like_place(xa, xa.shape)
        self._check(self.lib.sks_apply_operator(self.h, C.byref(op), px, py), "sks_apply_operator")
        return y

    def basis(self, A, r0, *, k, ncols):
        op, keep = A.struct()
        ra, pr = _prep(r0)
        n = ra.shape[0]
        B, pb = _empty_like_place(ra, (ncols, n))      # column-major n x ncols
        H = np.zeros((ncols - 1, ncols)) if ncols >= 2 else None
        st = self.lib.sks_basis(self.h, C.byref(op), pr, k, ncols, pb, H.ctypes.data if H is not None else None)
        self._check(st, "sks_basis")
        Bm = B.t() if _is_torch(B) else B.T
        return Bm, (H.T if H is not None else None)


@dataclass
class SgmresResult:
    x: object
    hist: np.ndarray
    hist_true: np.ndarray
    info: dict
    converged: bool
