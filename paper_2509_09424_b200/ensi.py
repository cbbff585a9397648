"""Thin ctypes binding of libensi.so (include/ensi.h).  Argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this module converts torch
device tensors to (pointer, count, level) views and numpy host arrays to pointers.  There is no CPU
fallback: if libensi.so is missing or no CUDA device is present the calls raise.

Names follow the C ABI: ``ensi_ctx_create`` -> :class:`Context`, ``ensi_load_keys`` ->
:meth:`Context.load_keys`, ``ensi_pcmm_ternary`` -> :meth:`Context.pcmm_ternary`,
``ensi_decrypt_debug`` -> :meth:`Context.decrypt_debug`, etc.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libensi.so")

ENSI_OK, ENSI_EINVAL, ENSI_EDIM, ENSI_ENOTTERNARY, ENSI_ELEVEL, ENSI_ENOKEY, ENSI_ENOMEM, ENSI_ECUDA = range(8)
ERR_NAMES = {0: "ENSI_OK", 1: "ENSI_EINVAL", 2: "ENSI_EDIM", 3: "ENSI_ENOTTERNARY", 4: "ENSI_ELEVEL",
             5: "ENSI_ENOKEY", 6: "ENSI_ENOMEM", 7: "ENSI_ECUDA"}
MEM_HOST, MEM_DEVICE = 0, 1
KERNEL_DEFAULT, KERNEL_CUDA_CORE, KERNEL_TCGEN05, KERNEL_TCGEN05_1CTA, KERNEL_TCGEN05_PAIR = 0, 1, 2, 3, 4

# every symbol include/ensi.h declares (checked by tests/test_abi.py)
EXPORTS = ["ensi_abi_version", "ensi_ctx_create", "ensi_ctx_destroy", "ensi_last_error", "ensi_ctx_moduli",
           "ensi_load_keys", "ensi_weights_pack", "ensi_weights_destroy", "ensi_pcmm_ternary_packed",
           "ensi_pcmm_ternary", "ensi_pcmm_ternary_host", "ensi_ntt", "ensi_rotate_hoisted", "ensi_rotate_batch",
           "ensi_rescale", "ensi_decrypt_debug", "ensi_launch_count", "ensi_last_compact_plan", "ensi_pcmm_kernel", "ensi_load_relin_key",
           "ensi_mul_plain", "ensi_mul_relin", "ensi_ccmm", "ensi_wire_bytes", "ensi_pcmm_ternary_host_wire",
           "ensi_wire_pack", "ensi_wire_unpack", "ensi_pcmm_ternary_compact", "ensi_pcmm_ternary_compact_gather",
           "ensi_ipc_get_handle", "ensi_ipc_open", "ensi_ipc_close", "ensi_peer_signal", "ensi_peer_wait"]


class EnsiError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("log_n", C.c_uint32), ("num_q", C.c_uint32), ("num_p", C.c_uint32), ("dnum", C.c_uint32),
                ("q", C.c_void_p), ("p", C.c_void_p), ("log2_scale", C.c_double)]


class CtView(C.Structure):
    _fields_ = [("data", C.c_void_p), ("count", C.c_uint32), ("level", C.c_uint32), ("log2_scale", C.c_double)]


class CompactView(C.Structure):
    _fields_ = [("data", C.c_void_p), ("count", C.c_uint32), ("level", C.c_uint32), ("log2_scale", C.c_double)]


class Keys(C.Structure):
    _fields_ = [("sk_ntt", C.c_void_p), ("n_rot", C.c_uint32), ("galois", C.c_void_p), ("rot_keys", C.c_void_p),
                ("rot_keys_mem", C.c_uint32)]


class IpcHandle(C.Structure):
    _fields_ = [("handle", C.c_uint8 * 64), ("offset", C.c_uint64)]


class PcmmOpts(C.Structure):
    _fields_ = [("layout", C.c_uint32), ("block_s", C.c_uint32), ("baby", C.c_uint32), ("rescale_out", C.c_uint32),
                ("kernel", C.c_uint32), ("moddown_lazy", C.c_uint32), ("cluster_pairs", C.c_uint32)]


_LIB = None


class CcmmOpts(C.Structure):
    _fields_ = [("form", C.c_uint32), ("block_s", C.c_uint32), ("d", C.c_uint32), ("m", C.c_uint32),
                ("col0", C.c_uint32), ("cols", C.c_uint32)]


def lib():
    """Load libensi.so (raises if it has not been built -- there is no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.ensi_abi_version.restype = u32
        L.ensi_ctx_create.argtypes = [C.POINTER(Params), C.c_int, C.POINTER(vp)]
        L.ensi_ctx_destroy.argtypes = [vp]
        L.ensi_ctx_destroy.restype = None
        L.ensi_last_error.argtypes = [vp]
        L.ensi_last_error.restype = C.c_char_p
        L.ensi_ctx_moduli.argtypes = [vp, vp, vp]
        L.ensi_load_keys.argtypes = [vp, C.POINTER(Keys)]
        L.ensi_weights_pack.argtypes = [vp, vp, u32, u32, u32, C.POINTER(vp)]
        L.ensi_weights_destroy.argtypes = [vp]
        L.ensi_weights_destroy.restype = None
        L.ensi_pcmm_ternary_packed.argtypes = [vp, C.POINTER(CtView), vp, C.POINTER(CtView), C.POINTER(PcmmOpts), vp]
        L.ensi_pcmm_ternary.argtypes = [vp, C.POINTER(CtView), vp, u32, u32, u32, C.POINTER(CtView),
                                        C.POINTER(PcmmOpts), vp]
        L.ensi_pcmm_ternary_host.argtypes = [vp, vp, u32, C.c_double, vp, vp, u32, vp]
        L.ensi_ntt.argtypes = [vp, vp, u32, vp, u32, C.c_int, vp]
        L.ensi_rotate_hoisted.argtypes = [vp, C.POINTER(CtView), u32, vp, C.POINTER(CtView), vp]
        L.ensi_rotate_batch.argtypes = [vp, C.POINTER(CtView), u32, vp, C.POINTER(CtView), vp]
        L.ensi_rescale.argtypes = [vp, C.POINTER(CtView), C.POINTER(CtView), vp]
        L.ensi_decrypt_debug.argtypes = [vp, C.POINTER(CtView), u32, vp, vp]
        L.ensi_launch_count.argtypes = [vp]
        L.ensi_load_relin_key.argtypes = [vp, vp, u32]
        L.ensi_wire_bytes.restype = C.c_uint64
        L.ensi_wire_bytes.argtypes = [vp, u32]
        L.ensi_pcmm_ternary_host_wire.argtypes = [vp, vp, u32, C.c_double, vp, vp, u32, vp]
        L.ensi_wire_pack.argtypes = [vp, C.POINTER(CtView), vp, vp]
        L.ensi_wire_unpack.argtypes = [vp, vp, C.POINTER(CtView), vp]
        L.ensi_pcmm_ternary_compact.argtypes = [vp, C.POINTER(CompactView), vp, C.POINTER(CompactView),
                                                C.POINTER(PcmmOpts), vp]
        L.ensi_pcmm_ternary_compact_gather.argtypes = [vp, C.POINTER(CompactView), vp, C.POINTER(vp), u32, u32, u32,
                                                       C.POINTER(PcmmOpts), vp]
        L.ensi_ipc_get_handle.argtypes = [vp, vp, C.POINTER(IpcHandle)]
        L.ensi_ipc_open.argtypes = [vp, C.POINTER(IpcHandle), C.POINTER(vp)]
        L.ensi_ipc_close.argtypes = [vp, vp]
        L.ensi_peer_signal.argtypes = [vp, C.POINTER(vp), u32, u32, u32, vp]
        L.ensi_peer_wait.argtypes = [vp, vp, u32, u32, vp]
        L.ensi_mul_plain.argtypes = [vp, C.POINTER(CtView), vp, C.c_double, C.POINTER(CtView), vp]
        L.ensi_mul_relin.argtypes = [vp, C.POINTER(CtView), C.POINTER(CtView), C.POINTER(CtView), vp]
        L.ensi_ccmm.argtypes = [vp, C.POINTER(CtView), C.POINTER(CtView), vp, C.POINTER(CtView),
                                C.POINTER(CcmmOpts), vp]
        L.ensi_launch_count.restype = u64
        L.ensi_pcmm_kernel.argtypes = [vp, u32, u32]
        L.ensi_last_compact_plan.argtypes = [vp, C.POINTER(u32), C.POINTER(u32)]
        L.ensi_pcmm_kernel.restype = u32
        _LIB = L
    return _LIB


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _np_ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class Weights:
    """Packed ternary weights (row a2), a model constant."""

    def __init__(self, ctx: "Context", W: np.ndarray):
        W = np.ascontiguousarray(W, dtype=np.int8)
        self.d, self.m = W.shape
        self.ctx = ctx
        h = C.c_void_p()
        rc = lib().ensi_weights_pack(ctx.h, _np_ptr(W), self.d, self.m, self.m, C.byref(h))
        ctx._check(rc)
        self.h = h
        self.nnz = int(np.count_nonzero(W))

    def close(self):
        if self.h:
            lib().ensi_weights_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """ensi_ctx_create(...) on one CUDA device."""

    def __init__(self, log_n: int, num_q: int, num_p: int, dnum: int, device: int = 0, q=None, p=None,
                 log2_scale: float = 40.0):
        self._qa = np.ascontiguousarray(q, np.uint64) if q is not None else None
        self._pa = np.ascontiguousarray(p, np.uint64) if p is not None else None
        prm = Params(log_n, num_q, num_p, dnum,
                     self._qa.ctypes.data if self._qa is not None else None,
                     self._pa.ctypes.data if self._pa is not None else None, log2_scale)
        h = C.c_void_p()
        rc = lib().ensi_ctx_create(C.byref(prm), device, C.byref(h))
        if rc != 0:
            raise EnsiError(rc, "ensi_ctx_create failed")
        self.h = h
        self.log_n, self.n, self.L, self.A, self.dnum, self.device = log_n, 1 << log_n, num_q, num_p, dnum, device
        self.log2_scale = log2_scale
        mods = np.zeros(num_q + num_p, np.uint64)
        psi = np.zeros(num_q + num_p, np.uint64)
        self._check(lib().ensi_ctx_moduli(self.h, _np_ptr(mods), _np_ptr(psi)))
        self.moduli = [int(v) for v in mods]
        self.psi = [int(v) for v in psi]
        self.q = self.moduli[:num_q]
        self.p = self.moduli[num_q:]
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            lib().ensi_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != 0:
            msg = lib().ensi_last_error(self.h)
            raise EnsiError(rc, msg.decode() if msg else "")

    def kernel_name(self, requested: int, level: int) -> str:
        k = int(lib().ensi_pcmm_kernel(self.h, level, requested))
        return {1: "cuda-core", 2: "tcgen05", 3: "tcgen05-1cta", 4: "tcgen05-pair-nomc"}.get(k, "unavailable")

    def launch_count(self) -> int:
        return int(lib().ensi_launch_count(self.h))

    def last_compact_plan(self) -> tuple:
        """(CTA pairs per multicast cluster, clusters launched) of the most recent compact accumulate."""
        c, k = C.c_uint32(), C.c_uint32()
        self._check(lib().ensi_last_compact_plan(self.h, C.byref(c), C.byref(k)))
        return int(c.value), int(k.value)

    def view(self, t, level: int, log2_scale: float = 40.0) -> CtView:
        """torch 64-bit CUDA tensor [count][2][level][N'] on this context's device -> ensi_ct_view."""
        if not (t.is_cuda and t.is_contiguous() and t.dtype.itemsize == 8):
            raise ValueError("ciphertexts must be a contiguous 64-bit CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"tensor on cuda:{t.device.index}, context on cuda:{self.device}")
        if t.dim() != 4 or t.shape[1] != 2 or t.shape[2] != level or t.shape[3] != self.n:
            raise ValueError(f"expected [count][2][{level}][{self.n}], got {tuple(t.shape)}")
        return CtView(t.data_ptr(), t.shape[0], level, log2_scale)

    # ---- keys
    def load_keys(self, sk_ntt: np.ndarray | None = None, galois=None, rot_keys=None):
        """rot_keys: numpy (host, copied) or torch CUDA tensor (device, referenced in place)."""
        sk = np.ascontiguousarray(sk_ntt, np.uint64) if sk_ntt is not None else None
        ga = np.ascontiguousarray(galois if galois is not None else [], np.uint64)
        mem, kp = MEM_HOST, None
        if rot_keys is not None:
            words = ga.shape[0] * self.dnum * 2 * (self.L + self.A) * self.n
            if (rot_keys.size if isinstance(rot_keys, np.ndarray) else rot_keys.numel()) != words:
                raise ValueError(f"rotation keys must hold n_rot x dnum x 2 x (num_q + num_p) x N' = {words} words")
            if isinstance(rot_keys, np.ndarray):
                rk = np.ascontiguousarray(rot_keys, np.uint64)
                kp = rk.ctypes.data
                self._keep_host = rk
            else:
                if not (rot_keys.is_cuda and rot_keys.is_contiguous() and rot_keys.dtype.itemsize == 8):
                    raise ValueError("device rotation keys must be a contiguous 64-bit CUDA tensor")
                mem, kp = MEM_DEVICE, rot_keys.data_ptr()
                self._keep_dev = rot_keys
        keys = Keys(sk.ctypes.data if sk is not None else None, ga.shape[0],
                    ga.ctypes.data if ga.shape[0] else None, kp, mem)
        self._check(lib().ensi_load_keys(self.h, C.byref(keys)))

    def weights(self, W: np.ndarray) -> Weights:
        return Weights(self, W)

    # ---- PCMM (rows a3, a4, a8)
    def pcmm_ternary(self, x, W, y, level: int, layout: int = 0, block_s: int = 0, baby: int = 0,
                     rescale_out: bool = False, kernel: int = 0, stream=None, log2_scale: float = 40.0,
                     moddown_lazy: bool = False) -> float:
        """y = x (x) W.  W: Weights (prepacked) or host int8 array.  Returns y's log2 scale."""
        xv = self.view(x, level, log2_scale)
        yv = self.view(y, level - 1 if rescale_out else level)
        opts = PcmmOpts(layout, block_s, baby, 1 if rescale_out else 0, kernel, 1 if moddown_lazy else 0)
        if isinstance(W, Weights):
            rc = lib().ensi_pcmm_ternary_packed(self.h, C.byref(xv), W.h, C.byref(yv), C.byref(opts),
                                                _stream_ptr(stream))
        else:
            Wa = np.ascontiguousarray(W, np.int8)
            d, m = Wa.shape
            rc = lib().ensi_pcmm_ternary(self.h, C.byref(xv), _np_ptr(Wa), d, m, m, C.byref(yv), C.byref(opts),
                                         _stream_ptr(stream))
        self._check(rc)
        return yv.log2_scale

    def pcmm_ternary_host(self, x_host: np.ndarray, w: Weights, y_host: np.ndarray, level: int, kernel: int = 0,
                          stream=None, log2_scale: float = 40.0):
        """End-to-end Layout A on host buffers (pinned recommended); enqueued on `stream` (sync before reading)."""
        if not (x_host.dtype.itemsize == 8 and y_host.dtype.itemsize == 8 and x_host.flags.c_contiguous
                and y_host.flags.c_contiguous):
            raise ValueError("host buffers must be C-contiguous 64-bit arrays")
        if x_host.shape[0] != w.d or y_host.shape[0] != w.m:
            raise ValueError("x_host / y_host leading dimensions must be d / m of the weights")
        if x_host.size != w.d * 2 * level * self.n or y_host.size != w.m * 2 * level * self.n:
            raise ValueError("host buffers must hold [count][2][level][N'] words")
        self._check(lib().ensi_pcmm_ternary_host(self.h, _np_ptr(x_host), level, log2_scale, w.h, _np_ptr(y_host),
                                                 kernel, _stream_ptr(stream)))

    # ---- compact device layout (ensi_compact_view)
    def compact_view(self, t, level: int, log2_scale: float = 40.0) -> CompactView:
        """uint8 CUDA tensor [count][ensi_wire_bytes(level)] -> ensi_compact_view."""
        wb = self.wire_bytes(level)
        if not (t.is_cuda and t.is_contiguous() and t.dtype.itemsize == 1):
            raise ValueError("compact ciphertexts must be a contiguous 8-bit CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"tensor on cuda:{t.device.index}, context on cuda:{self.device}")
        if t.dim() != 2 or t.shape[1] != wb:
            raise ValueError(f"expected [count][{wb}] bytes, got {tuple(t.shape)}")
        return CompactView(t.data_ptr(), t.shape[0], level, log2_scale)

    def pcmm_ternary_compact(self, x, w: "Weights", y, level: int, kernel: int = 0, stream=None,
                             log2_scale: float = 40.0, cluster_pairs: int = 0) -> float:
        """y = x (x) W on compact ciphertexts (Layout A); returns y's log2 scale.  cluster_pairs: 0 = launch shape
        chosen per layer, 1..4 = that many CTA pairs per multicast cluster (same words)."""
        xv, yv = self.compact_view(x, level, log2_scale), self.compact_view(y, level)
        opts = PcmmOpts(0, 0, 0, 0, kernel, 0, cluster_pairs)
        self._check(lib().ensi_pcmm_ternary_compact(self.h, C.byref(xv), w.h, C.byref(yv), C.byref(opts),
                                                    _stream_ptr(stream)))
        return yv.log2_scale

    def pcmm_ternary_compact_gather(self, x, w: "Weights", dsts, rows_total: int, row0: int, level: int,
                                    kernel: int = 0, stream=None, log2_scale: float = 40.0, cluster_pairs: int = 0):
        """NEXT #4 fused gather: y_i of this call stored into rows row0 + i of every destination (device pointers or
        contiguous uint8 CUDA tensors of rows_total x wire_bytes -- this GPU's gathered buffer and the peers')."""
        xv = self.compact_view(x, level, log2_scale)
        wb = self.wire_bytes(level)
        ptrs = []
        for dbuf in dsts:
            if hasattr(dbuf, "data_ptr"):
                if not (dbuf.is_cuda and dbuf.is_contiguous() and dbuf.dtype.itemsize == 1 and
                        dbuf.numel() == rows_total * wb):
                    raise ValueError(f"destination must be a contiguous uint8 CUDA tensor of {rows_total} x {wb} bytes")
                ptrs.append(dbuf.data_ptr())
            else:
                ptrs.append(int(dbuf))
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        opts = PcmmOpts(0, 0, 0, 0, kernel, 0, cluster_pairs)
        self._check(lib().ensi_pcmm_ternary_compact_gather(self.h, C.byref(xv), w.h, arr, len(ptrs), rows_total, row0,
                                                           C.byref(opts), _stream_ptr(stream)))

    def ipc_handle(self, t) -> bytes:
        """CUDA IPC handle (72 bytes: allocation handle + offset) of a CUDA tensor's storage, for another process."""
        h = IpcHandle()
        self._check(lib().ensi_ipc_get_handle(self.h, C.c_void_p(t.data_ptr()), C.byref(h)))
        return bytes(C.string_at(C.addressof(h), C.sizeof(h)))

    def ipc_open(self, handle: bytes) -> int:
        h = IpcHandle.from_buffer_copy(handle)
        p = C.c_void_p()
        self._check(lib().ensi_ipc_open(self.h, C.byref(h), C.byref(p)))
        return int(p.value)

    def ipc_close(self, ptr: int):
        self._check(lib().ensi_ipc_close(self.h, C.c_void_p(ptr)))

    def peer_signal(self, flag_ptrs, slot: int, epoch: int, stream=None):
        """flag_ptrs: device pointers or 32-bit CUDA tensors (this GPU's and the peers' flag arrays)."""
        arr = (C.c_void_p * len(flag_ptrs))(*[f.data_ptr() if hasattr(f, "data_ptr") else int(f) for f in flag_ptrs])
        self._check(lib().ensi_peer_signal(self.h, arr, len(flag_ptrs), slot, epoch, _stream_ptr(stream)))

    def peer_wait(self, flags, n: int, epoch: int, stream=None):
        if not (flags.is_cuda and flags.dtype.itemsize == 4 and flags.numel() >= n):
            raise ValueError("flags must be a CUDA tensor of >= n 32-bit words")
        self._check(lib().ensi_peer_wait(self.h, C.c_void_p(flags.data_ptr()), n, epoch, _stream_ptr(stream)))

    # ---- compact wire format (host transfers)
    def wire_widths(self, level: int):
        return [(int(q).bit_length() + 7) // 8 for q in self.moduli[:level]]

    def wire_bytes(self, level: int) -> int:
        return int(lib().ensi_wire_bytes(self.h, level))

    def pcmm_ternary_host_wire(self, x_wire: np.ndarray, w: Weights, y_wire: np.ndarray, level: int,
                               kernel: int = 0, stream=None, log2_scale: float = 40.0):
        """End-to-end Layout A on host buffers in the wire format (uint8, pinned recommended)."""
        wb = self.wire_bytes(level)
        if not (x_wire.dtype == np.uint8 and y_wire.dtype == np.uint8 and x_wire.flags.c_contiguous
                and y_wire.flags.c_contiguous):
            raise ValueError("wire buffers must be C-contiguous uint8 arrays")
        if x_wire.size != w.d * wb or y_wire.size != w.m * wb:
            raise ValueError(f"wire buffers must hold d / m ciphertexts of {wb} bytes")
        self._check(lib().ensi_pcmm_ternary_host_wire(self.h, _np_ptr(x_wire), level, log2_scale, w.h,
                                                      _np_ptr(y_wire), kernel, _stream_ptr(stream)))

    def _wire_buf(self, t, count: int, level: int, what: str):
        need = count * self.wire_bytes(level)
        if not (t.is_cuda and t.is_contiguous() and t.dtype.itemsize == 1):
            raise ValueError(f"{what} must be a contiguous 8-bit CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"{what} on cuda:{t.device.index}, context on cuda:{self.device}")
        if t.numel() != need:
            raise ValueError(f"{what} must hold {count} x {self.wire_bytes(level)} bytes, got {t.numel()}")
        return C.c_void_p(t.data_ptr())

    def wire_pack(self, x, out, level: int, stream=None):
        xv = self.view(x, level)
        op = self._wire_buf(out, xv.count, level, "wire output")
        self._check(lib().ensi_wire_pack(self.h, C.byref(xv), op, _stream_ptr(stream)))

    def wire_unpack(self, inp, y, level: int, stream=None):
        yv = self.view(y, level)
        ip = self._wire_buf(inp, yv.count, level, "wire input")
        self._check(lib().ensi_wire_unpack(self.h, ip, C.byref(yv), _stream_ptr(stream)))

    # ---- primitives (rows a5-a7, a4, a10)
    def ntt(self, data, limb_of_row, inverse: bool = False, stream=None):
        lm = np.ascontiguousarray(limb_of_row, np.uint32)
        rows = data.numel() // self.n
        self._check(lib().ensi_ntt(self.h, C.c_void_p(data.data_ptr()), rows, _np_ptr(lm), lm.shape[0],
                                   1 if inverse else 0, _stream_ptr(stream)))

    def rotate_hoisted(self, x, galois, y, level: int, stream=None):
        ga = np.ascontiguousarray(galois, np.uint64)
        xv, yv = self.view(x, level), self.view(y, level)
        self._check(lib().ensi_rotate_hoisted(self.h, C.byref(xv), ga.shape[0], _np_ptr(ga), C.byref(yv),
                                              _stream_ptr(stream)))

    def rotate_batch(self, x, galois, y, level: int, stream=None):
        """y[c * len(galois) + r] = Rot_{galois[r]}(x[c]) for every input c (hoisted, key-stationary)."""
        ga = np.ascontiguousarray(galois, np.uint64)
        xv, yv = self.view(x, level), self.view(y, level)
        self._check(lib().ensi_rotate_batch(self.h, C.byref(xv), ga.shape[0], _np_ptr(ga), C.byref(yv),
                                            _stream_ptr(stream)))

    def rescale(self, x, y, level: int, log2_scale: float = 80.0, stream=None) -> float:
        xv, yv = self.view(x, level, log2_scale), self.view(y, level - 1)
        self._check(lib().ensi_rescale(self.h, C.byref(xv), C.byref(yv), _stream_ptr(stream)))
        return yv.log2_scale

    # ---- CCMM (R18)
    def load_relin_key(self, key):
        """key [dnum][2][num_q+num_p][N']: numpy (host, copied) or torch CUDA tensor (device, referenced)."""
        words = self.dnum * 2 * (self.L + self.A) * self.n
        if (key.size if isinstance(key, np.ndarray) else key.numel()) != words:
            raise ValueError(f"relinearisation key must hold dnum x 2 x (num_q + num_p) x N' = {words} words")
        if isinstance(key, np.ndarray):
            k = np.ascontiguousarray(key, np.uint64)
            self._check(lib().ensi_load_relin_key(self.h, k.ctypes.data, MEM_HOST))
        else:
            if not (key.is_cuda and key.is_contiguous() and key.dtype.itemsize == 8):
                raise ValueError("device relinearisation key must be a contiguous 64-bit CUDA tensor")
            self._keep_relin = key
            self._check(lib().ensi_load_relin_key(self.h, key.data_ptr(), MEM_DEVICE))

    @staticmethod
    def _dev_words(t, shape, what):
        if not (t.is_cuda and t.is_contiguous() and t.dtype.itemsize == 8) or tuple(t.shape) != tuple(shape):
            raise ValueError(f"{what} must be a contiguous 64-bit CUDA tensor of shape {tuple(shape)}")
        return t.data_ptr()

    def mul_plain(self, x, pt, y, level: int, log2_scale: float = 40.0, pt_log2_scale: float = 40.0,
                  stream=None) -> float:
        xv, yv = self.view(x, level, log2_scale), self.view(y, level)
        pp = self._dev_words(pt, (level, self.n), "plaintext")
        self._check(lib().ensi_mul_plain(self.h, C.byref(xv), pp, pt_log2_scale, C.byref(yv), _stream_ptr(stream)))
        return yv.log2_scale

    def mul_relin(self, a, b, y, level: int, log2_scale: float = 40.0, stream=None) -> float:
        av, bv, yv = self.view(a, level, log2_scale), self.view(b, level, log2_scale), self.view(y, level)
        self._check(lib().ensi_mul_relin(self.h, C.byref(av), C.byref(bv), C.byref(yv), _stream_ptr(stream)))
        return yv.log2_scale

    def ccmm(self, a, src, mask_pt, y, form: int, block_s: int, d: int, m: int, level: int,
             log2_scale: float = 40.0, col0: int = 0, cols: int = 0, stream=None) -> float:
        """y = CCMM(a, src) (R18): form 2 C = A.B, form 1 C = A.K^T, per head block of block_s slots;
        output columns [col0, col0 + cols) (cols = 0: to m)."""
        av, sv = self.view(a, level, log2_scale), self.view(src, level, log2_scale)
        yv = self.view(y, level - 2)
        mp = self._dev_words(mask_pt, (level, self.n), "mask plaintext")
        opts = CcmmOpts(form, block_s, d, m, col0, cols)
        self._check(lib().ensi_ccmm(self.h, C.byref(av), C.byref(sv), mp, C.byref(yv), C.byref(opts),
                                    _stream_ptr(stream)))
        return yv.log2_scale

    def decrypt_debug(self, ct, index: int, level: int, log2_scale: float = 40.0, want_coeffs: bool = False):
        cv = self.view(ct, level, log2_scale)
        slots = np.zeros(self.n // 2, np.float64)
        coeffs = np.zeros((level, self.n), np.uint64) if want_coeffs else None
        self._check(lib().ensi_decrypt_debug(self.h, C.byref(cv), index,
                                             _np_ptr(coeffs) if want_coeffs else None, _np_ptr(slots)))
        return (slots, coeffs) if want_coeffs else slots


def wire_pack_host(x: np.ndarray, widths) -> np.ndarray:
    """Host-side wire packing of [count][2][level][N'] uint64 words (the client's serialisation; numpy only):
    limb r keeps the low widths[r] bytes of each little-endian word."""
    x = np.ascontiguousarray(x, np.uint64)
    cnt, _, level, n = x.shape
    b = x.view(np.uint8).reshape(cnt, 2, level, n, 8)
    parts = [b[:, :, r, :, :widths[r]].reshape(cnt, 2, -1) for r in range(level)]
    return np.ascontiguousarray(np.concatenate(parts, axis=2).reshape(cnt, -1))


def wire_unpack_host(wb: np.ndarray, widths, level: int, n: int) -> np.ndarray:
    """Inverse of wire_pack_host: [count][wire bytes] -> [count][2][level][N'] uint64."""
    cnt = wb.shape[0]
    w2 = wb.reshape(cnt, 2, -1)
    out = np.zeros((cnt, 2, level, n, 8), np.uint8)
    off = 0
    for r in range(level):
        out[:, :, r, :, :widths[r]] = w2[:, :, off:off + n * widths[r]].reshape(cnt, 2, n, widths[r])
        off += n * widths[r]
    return out.reshape(cnt, 2, level, n * 8).view(np.uint64).reshape(cnt, 2, level, n)


def galois_elt(log_n: int, r: int) -> int:
    """g = 5^r mod 2N' (left rotation by r); host helper for building key lists."""
    half = 1 << (log_n - 1)
    return pow(5, r % half, 2 << log_n)
