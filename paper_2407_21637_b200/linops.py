"""Drop-in HODLR matvec on B200 (the north-star path).

``matvec(H, x, working)`` has the signature and error behaviour of the
reference's spec'd operator ``linops.matvec`` (/root/reference/SPEC.md:334-342,
Algorithm 3 HODLR_MATVEC):

* ``H``: a HODLR matrix -- the reference's ``hodlrmp.hodlr.HodlrMatrix`` or this
  package's ``model.HodlrMatrix`` (anything with ``n``, ``depth``,
  ``working_format``, ``offdiag_blocks()`` and ``leaves()``, hodlr.py:95-135);
* ``x``: length-n real vector (or n x s block of right-hand sides);
* ``working``: the working precision (default ``H.working_format``): fp64 and
  fp32 run the throughput kernels; bf16 / fp16 / q52 (the paper's simulated
  low working precisions) run the strict-order kernels,
  bit-identical to the reference's ``Arithmetic(working)``; custom formats
  raise ``NotImplementedError``;
* length mismatch -> ``ValueError``; overflow propagates as inf.

The matrix is packed once per ``H`` into the device layout (cached weakly by
identity; ``HodlrMatrix`` is ``eq=False`` so it hashes by identity) and every
call runs the hand-written sm_100a kernels through the C ABI.  ``x`` is rounded
to the working format on entry (RNE, as ``round_matrix`` would).  There is no
CPU path: without the CUDA extension or a GPU the call raises.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _lib
from .formats import FP32, FP64, format_code

__all__ = ["matvec", "HodlrOperator", "descriptor", "operator_for"]

_WORKING_DTYPE = {4: np.float64, 3: np.float32}
_NARROW = (0, 1, 2)  # q52, bf16, fp16 working: binary64 carriers, strict-order kernels


def _f64(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.float64:
        a = a.astype(np.float64)
    if any(s % 8 for s in a.strides):
        a = np.ascontiguousarray(a)
    return a


class _Descriptor:
    """ctypes ``hodlr_desc`` for H plus the numpy arrays it points into."""

    def __init__(self, H):
        n, depth = int(H.n), int(H.depth)
        self.keep = []
        leaves = list(H.leaves())
        if len(leaves) != 2 ** depth:
            raise ValueError(f"expected {2 ** depth} leaves, got {len(leaves)}")
        bounds = np.array([rng[0] for _, rng, _ in leaves] + [n], dtype=np.int64)
        lptrs = (_lib.c_dp * len(leaves))()
        lds = np.empty(len(leaves), dtype=np.int64)
        for i, (_, (a, b), D) in enumerate(leaves):
            D = _f64(D)
            if D.shape != (b - a, b - a):
                raise ValueError(f"leaf {i} has shape {D.shape}, expected {(b - a, b - a)}")
            if D.strides[1] != 8:
                D = np.ascontiguousarray(D)
            self.keep.append(D)
            lptrs[i] = D.ctypes.data_as(_lib.c_dp)
            lds[i] = D.strides[0] // 8 if D.shape[0] > 1 else D.shape[1]
        facs = []
        for _, _, _, _, up, lo in H.offdiag_blocks():
            for f in (up, lo):
                U, V = _f64(f.U), _f64(f.V)
                self.keep += [U, V]
                r = U.shape[1]
                fi = _lib.FactorIn(
                    format_code(f.fmt), r, U.shape[0], V.shape[0],
                    U.ctypes.data_as(_lib.c_dp), U.strides[0] // 8, U.strides[1] // 8,
                    V.ctypes.data_as(_lib.c_dp), V.strides[0] // 8, V.strides[1] // 8)
                facs.append(fi)
        nf = 2 * (2 ** depth - 1)
        if len(facs) != nf:
            raise ValueError(f"expected {nf} off-diagonal factors, got {len(facs)}")
        farr = (_lib.FactorIn * max(nf, 1))(*facs)
        self.keep += [bounds, lds, lptrs, farr]
        self.desc = _lib.Desc(n, depth, format_code(H.working_format),
                              bounds.ctypes.data_as(ctypes.POINTER(_lib.c_i64)), lptrs,
                              lds.ctypes.data_as(ctypes.POINTER(_lib.c_i64)), farr, 0)


class _EncodedDescriptor:
    """``hodlr_desc`` with payload_encoded = 1 over the narrow arrays of a
    container v2 (``model.EncodedHodlr``): nothing is widened on the host."""

    def __init__(self, E):
        from .model import ENCODED_DTYPE

        n, depth = int(E.n), int(E.depth)
        self.keep = []
        rngs = E.tree.ranges[depth]
        bounds = np.array([a for a, _ in rngs] + [n], dtype=np.int64)
        wdt = np.dtype(ENCODED_DTYPE[E.working_format.name])
        lptrs = (_lib.c_dp * len(rngs))()
        lds = np.empty(len(rngs), dtype=np.int64)
        for i, ((a, b), D) in enumerate(zip(rngs, E.leaf_blocks)):
            if D.dtype != wdt or D.shape != (b - a, b - a):
                raise ValueError(f"leaf {i}: expected {(b - a, b - a)} {wdt}, got {D.shape} {D.dtype}")
            D = np.ascontiguousarray(D)
            self.keep.append(D)
            lptrs[i] = ctypes.cast(D.ctypes.data, _lib.c_dp)
            lds[i] = D.shape[1]
        facs = []
        for k in range(1, depth + 1):
            fmt = E.plan.chosen[k - 1]
            dt = np.dtype(ENCODED_DTYPE[fmt.name])
            for pair in E.blocks[k - 1]:
                for U, V in pair:
                    if U.dtype != dt or V.dtype != dt or U.ndim != 2 or V.ndim != 2 or U.shape[1] != V.shape[1]:
                        raise ValueError(f"level {k}: bad encoded factor ({U.dtype} {U.shape}, {V.dtype} {V.shape})")
                    self.keep += [U, V]
                    it = dt.itemsize
                    facs.append(_lib.FactorIn(
                        format_code(fmt), U.shape[1], U.shape[0], V.shape[0],
                        ctypes.cast(U.ctypes.data, _lib.c_dp), U.strides[0] // it, U.strides[1] // it,
                        ctypes.cast(V.ctypes.data, _lib.c_dp), V.strides[0] // it, V.strides[1] // it))
        farr = (_lib.FactorIn * max(len(facs), 1))(*facs)
        self.keep += [bounds, lds, lptrs, farr]
        self.desc = _lib.Desc(n, depth, format_code(E.working_format),
                              bounds.ctypes.data_as(ctypes.POINTER(_lib.c_i64)), lptrs,
                              lds.ctypes.data_as(ctypes.POINTER(_lib.c_i64)), farr, 1)


def descriptor(H) -> _Descriptor:
    return _Descriptor(H)


def _torch():
    import torch  # plumbing only: device memory and streams

    return torch


def _working_code(H, working) -> int:
    # (format_code raises NotImplementedError for custom formats)
    return format_code(working if working is not None else H.working_format)


class HodlrOperator:
    """Packed, device-resident HODLR matrix (one C-ABI handle)."""

    def __init__(self, H, device: int | None = None, rank: int = 0, nranks: int = 1):
        L = _lib.lib()
        if device is None:
            torch = _torch()
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = int(device)
        self.working_format = H.working_format
        self.n = int(H.n)
        self.depth = int(H.depth)
        self.rank, self.nranks = int(rank), int(nranks)
        d = _EncodedDescriptor(H) if getattr(H, "encoded", False) else _Descriptor(H)
        h = _lib.c_vp()
        if nranks == 1:
            st = L.hodlr_create(ctypes.byref(d.desc), self.device, ctypes.byref(h))
        else:
            st = L.hodlr_create_sharded(ctypes.byref(d.desc), self.device,
                                        _lib.Shard(rank, nranks), ctypes.byref(h))
        _lib.check(st, "hodlr_create")
        self._h = h
        self._lock = threading.Lock()
        info = _lib.Info()
        _lib.check(L.hodlr_info(h, ctypes.byref(info)), "hodlr_info")
        self.n_local = int(info.n_local)
        self.row0 = int(info.row0)
        self.matrix_bytes = int(info.matrix_bytes)
        self.device_bytes = int(info.device_bytes)
        self.launches_per_matvec = int(info.launches_per_matvec)
        self._finalizer = weakref.finalize(self, L.hodlr_destroy, h)

    @classmethod
    def from_container(cls, path, device: int | None = None, rank: int = 0, nranks: int = 1):
        """Device operator straight from a stored matrix (container v1 or v2,
        hodlr.py:297-363): a v2 file's narrow payloads go to the packer as they
        are, without a binary64 copy on the host."""
        from .model import load_encoded, load_hodlr

        E = load_encoded(path)
        return cls(E if E.encoded else load_hodlr(path), device, rank, nranks)

    def path(self, s: int = 1, working=None) -> tuple[str, int]:
        """(kernel path, launches per matvec) for s right-hand sides:
        "fused_sv" (one persistent kernel), "mrhs" (tensor-core multi-RHS
        kernels) or "generic"."""
        p, n = _lib.c_i32(), _lib.c_i32()
        _lib.check(_lib.lib().hodlr_matvec_path(self._h, _working_code(self, working), int(s),
                                                ctypes.byref(p), ctypes.byref(n)), "hodlr_matvec_path")
        return _lib.PATH_NAMES[p.value], int(n.value)

    # ---------------------------------------------------------------- device
    def matvec(self, x, working=None, out=None, stream=None):
        """b = H x for a CUDA tensor x ((n,) or (n, s)), returns a CUDA tensor of
        the working dtype (float64 carrying working-format values for bf16 /
        fp16 / q52 working).  Stream-ordered on ``stream`` (default: current)."""
        torch = _torch()
        code = _working_code(self, working)
        dt = torch.float32 if code == 3 else torch.float64
        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            raise TypeError("HodlrOperator.matvec expects a CUDA tensor; use matvec_host for host arrays")
        if x.device.index != self.device:
            raise ValueError(f"tensor on cuda:{x.device.index}, operator on cuda:{self.device}")
        vec = x.dim() == 1
        X = x.reshape(-1, 1) if vec else x
        if X.dim() != 2 or X.shape[0] != self.n_local:
            raise ValueError(f"length mismatch: x has {x.shape[0]} rows, operator has {self.n_local}")
        if X.dtype != dt:
            X = X.to(dt)  # single RNE rounding fp64 -> fp32 (cvt.rn.f32.f64)
        if X.stride(1) != 1:
            X = X.contiguous()
        s = X.shape[1]
        B = out if out is not None else torch.empty((self.n_local, s), dtype=dt, device=X.device)
        if out is not None and (B.shape != (self.n_local, s) or B.dtype != dt or B.stride(1) != 1):
            raise ValueError("out has the wrong shape / dtype / layout")
        st = stream if stream is not None else torch.cuda.current_stream(X.device)
        with self._lock:
            _lib.check(_lib.lib().hodlr_matvec(
                self._h, code, X.data_ptr(), X.stride(0), B.data_ptr(), B.stride(0), s, None, 0,
                st.cuda_stream), "hodlr_matvec")
        return B[:, 0] if (vec and out is None) else B

    def matvec_strict(self, x, working=None, stream=None):
        """b = H x with the reference's arithmetic model in ``working``: every
        product and partial sum rounded, strict left-to-right contractions
        (arithmetic.py:14-67) -- bit-identical to ``Arithmetic(working)``.
        x: CUDA float64 tensor; returns float64 carrying working-format values."""
        torch = _torch()
        code = _working_code(self, working)
        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            raise TypeError("HodlrOperator.matvec_strict expects a CUDA tensor")
        vec = x.dim() == 1
        X = x.reshape(-1, 1) if vec else x
        if X.dim() != 2 or X.shape[0] != self.n_local:
            raise ValueError(f"length mismatch: x has {x.shape[0]} rows, operator has {self.n_local}")
        X = X.to(torch.float64)
        if X.stride(1) != 1:
            X = X.contiguous()
        s = X.shape[1]
        B = torch.empty((self.n_local, s), dtype=torch.float64, device=X.device)
        st = stream if stream is not None else torch.cuda.current_stream(X.device)
        with self._lock:
            _lib.check(_lib.lib().hodlr_matvec_strict(
                self._h, code, X.data_ptr(), X.stride(0), B.data_ptr(), B.stride(0), s, None, 0,
                st.cuda_stream), "hodlr_matvec_strict")
        return B[:, 0] if vec else B

    # ---------------------------------------------------------------- host
    def matvec_host(self, x, working=None) -> np.ndarray:
        """End-to-end call with host buffers: binary64 in, binary64 out."""
        code = _working_code(self, working)
        x = np.asarray(x, dtype=np.float64)
        vec = x.ndim == 1
        X = np.ascontiguousarray(x.reshape(-1, 1) if vec else x)
        if X.ndim != 2 or X.shape[0] != self.n_local:
            raise ValueError(f"length mismatch: x has {x.shape[0] if x.ndim else 0} rows, "
                             f"H has {self.n_local}")
        B = np.empty_like(X)
        with self._lock:
            _lib.check(_lib.lib().hodlr_matvec_host(self._h, code, X.ctypes.data, B.ctypes.data,
                                                     X.shape[1], None), "hodlr_matvec_host")
        return B[:, 0] if vec else B

    def matvec_host_ptr(self, x_ptr: int, b_ptr: int, s: int, working=None, stream=None) -> None:
        """Host-pointer variant (pinned buffers), used by the e2e benchmark."""
        code = _working_code(self, working)
        _lib.check(_lib.lib().hodlr_matvec_host(self._h, code, x_ptr, b_ptr, s, stream),
                   "hodlr_matvec_host")

    # ---------------------------------------------------------------- sharded
    def as_working(self, x, working=None):
        """x as a CUDA tensor of the working dtype on this operator's device
        (fp64 -> fp32 is one RNE rounding); raises on a host or foreign-device tensor."""
        torch = _torch()
        code = _working_code(self, working)
        if code in _NARROW:
            raise NotImplementedError("sharded matvec: working precision must be fp64 or fp32")
        dt = torch.float64 if code == 4 else torch.float32
        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            raise TypeError("expected a CUDA tensor")
        if x.device.index != self.device:
            raise ValueError(f"tensor on cuda:{x.device.index}, operator on cuda:{self.device}")
        return x if x.dtype == dt else x.to(dt)

    def _check_shard_io(self, code, *tensors):
        torch = _torch()
        dt = torch.float64 if code == 4 else torch.float32
        for t in tensors:
            if t is None or t.numel() == 0:
                continue
            if not t.is_cuda or t.device.index != self.device or t.dtype != dt:
                raise ValueError(f"shard buffers must be {dt} tensors on cuda:{self.device} "
                                 f"(got {t.dtype} on {t.device})")

    def exchange_count(self, s: int = 1) -> int:
        c = _lib.c_i64()
        _lib.check(_lib.lib().hodlr_shard_exchange_count(self._h, s, ctypes.byref(c)))
        return int(c.value)

    def shard_begin(self, x, send, working=None, stream=None):
        torch = _torch()
        code = _working_code(self, working)
        self._check_shard_io(code, x, send)
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _lib.check(_lib.lib().hodlr_matvec_shard_begin(
            self._h, code, x.data_ptr(), x.stride(0), x.shape[1],
            send.data_ptr() if send is not None and send.numel() else None, None, 0,
            st.cuda_stream), "hodlr_matvec_shard_begin")

    def shard_local(self, x, out, working=None, stream=None):
        torch = _torch()
        code = _working_code(self, working)
        self._check_shard_io(code, x, out)
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _lib.check(_lib.lib().hodlr_matvec_shard_local(
            self._h, code, x.data_ptr(), x.stride(0), out.data_ptr(), out.stride(0), x.shape[1],
            None, 0, st.cuda_stream), "hodlr_matvec_shard_local")

    def shard_end(self, x, recv, out, working=None, stream=None):
        torch = _torch()
        code = _working_code(self, working)
        self._check_shard_io(code, x, recv, out)
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _lib.check(_lib.lib().hodlr_matvec_shard_end(
            self._h, code, x.data_ptr(), x.stride(0),
            recv.data_ptr() if recv is not None and recv.numel() else None,
            out.data_ptr(), out.stride(0), x.shape[1], None, 0, st.cuda_stream),
            "hodlr_matvec_shard_end")

    # ---------------------------------------------------------------- checks
    def unpack_factor(self, index: int, rows: int, cols: int, rank: int):
        U = np.empty((rows, rank))
        V = np.empty((cols, rank))
        _lib.check(_lib.lib().hodlr_unpack_factor(self._h, index, U.ctypes.data, V.ctypes.data))
        return U, V

    def unpack_leaf(self, i: int, m: int) -> np.ndarray:
        D = np.empty((m, m))
        _lib.check(_lib.lib().hodlr_unpack_leaf(self._h, i, D.ctypes.data))
        return D

    def close(self):
        self._finalizer()


_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_CACHE_LOCK = threading.Lock()


def operator_for(H, device: int | None = None) -> HodlrOperator:
    """The cached device operator of H (packed on first use)."""
    with _CACHE_LOCK:
        op = _CACHE.get(H)
        if op is None or (device is not None and op.device != device):
            op = HodlrOperator(H, device)
            _CACHE[H] = op
        return op


def matvec(H, x, working=None):
    """Drop-in for the reference's ``linops.matvec(H, x, working)``.

    Host input (numpy / sequence) -> binary64 numpy result of the same shape;
    CUDA tensor input -> CUDA tensor result in the working dtype.
    """
    _working_code(H, working)  # NotImplementedError before any packing
    try:
        import torch

        if isinstance(x, torch.Tensor) and x.is_cuda:
            return operator_for(H, x.device.index).matvec(x, working)
    except ImportError:  # pragma: no cover - torch is in the image
        pass
    xa = np.asarray(x, dtype=np.float64)
    if xa.ndim == 0 or xa.shape[0] != H.n:
        raise ValueError(f"length mismatch: x has {xa.shape[0] if xa.ndim else 0} entries, H is {H.n}")
    return operator_for(H).matvec_host(xa, working)
