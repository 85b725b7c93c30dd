"""Thin ctypes binding of libmoe (include/moe.h).  Argument marshalling only:
every step of the layer runs in the library's sm_100a kernels.  Torch supplies
device memory, streams and (for world > 1) the broadcast of the NCCL unique id.

There is no fallback: if libmoe.so is missing or fails to load, importing this
module raises.
"""

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoe.so")

MOE_OK = 0
ABI_VERSION = 3  # include/moe.h MOE_ABI_VERSION
STATUS = {0: "MOE_OK", 1: "MOE_ERR_INVALID_ARG", 2: "MOE_ERR_CUDA", 3: "MOE_ERR_NCCL", 4: "MOE_ERR_CAPACITY",
          5: "MOE_ERR_UNSUPPORTED", 6: "MOE_ERR_DEVICE", 7: "MOE_ERR_TIMEOUT"}

# Every symbol include/moe.h declares (checked by tests/test_abi_cpu.py).
EXPORTS = ["moe_get_unique_id", "moe_ctx_create", "moe_ctx_create_group", "moe_ctx_destroy", "moe_ctx_sync", "moe_status_str",
           "moe_last_error", "moe_abi_version", "moe_route", "moe_route_stats", "moe_stats_allreduce", "moe_stats_allreduce_layers",
           "moe_dispatch", "moe_dispatch_from", "moe_set_output_mode", "moe_expert_ffn", "moe_combine", "moe_pack_w13", "moe_placement_contiguous",
           "moe_layout_host", "moe_debug_plan", "moe_debug_identity_ffn", "moe_debug_recv", "moe_debug_send", "moe_kernel_launches",
           "moe_ffn_timing_enable", "moe_ffn_timing_read", "moe_timeline_enable", "moe_timeline_read"]


class MoeError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("max_tokens", ctypes.c_int32), ("hidden", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("num_experts", ctypes.c_int32), ("max_k", ctypes.c_int32), ("world", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("device", ctypes.c_int32), ("virtual_ranks", ctypes.c_int32),
                ("a2a_mode", ctypes.c_int32), ("tp", ctypes.c_int32)]


class DispatchInfo(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("num_local_experts", ctypes.c_int32), ("recv_rows", ctypes.c_int64),
                ("send_counts", ctypes.c_int32 * 64), ("recv_counts", ctypes.c_int32 * 64)]


def load_library(path=LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"libmoe.so not found at {path}: build it with "
                          f"`python -m paper_2502_06643_b200.build` (no fallback path exists)")
    lib = ctypes.CDLL(path)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "moe_get_unique_id": [P],
        "moe_ctx_create": [ctypes.POINTER(Config), P, ctypes.POINTER(P)],
        "moe_ctx_create_group": [ctypes.POINTER(Config), I32, P, P],
        "moe_ctx_destroy": [P],
        "moe_ctx_sync": [P],
        "moe_route": [P, P, I32, I32, I32, P, P, P],
        "moe_route_stats": [P, P, P, I32, I32, I32, P, P, P],
        "moe_stats_allreduce": [P, P, P, I32, P],
        "moe_stats_allreduce_layers": [P, P, P, I32, I32, P],
        "moe_dispatch": [P, P, P, I32, I32, P, P, P],
        "moe_expert_ffn": [P, P, P, I32, P],
        "moe_dispatch_from": [P, P, P, P, I32, I32, P, P],
        "moe_set_output_mode": [P, I32],
        "moe_combine": [P, P, P, P],
        "moe_pack_w13": [P, P, I32, I32, I32, P, P],
        "moe_placement_contiguous": [I32, I32, P],
        "moe_layout_host": [I32, I32, P, P, P, P, P, P],
        "moe_debug_plan": [P, P, P, P, P],
        "moe_debug_identity_ffn": [P, P],
        "moe_debug_recv": [P, P, I64, P],
        "moe_debug_send": [P, P, I64, P],
        "moe_ffn_timing_enable": [P, I32],
        "moe_ffn_timing_read": [P, P, I32, P],
        "moe_timeline_enable": [P, I32],
        "moe_timeline_read": [P, P, I32, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.moe_status_str.argtypes = [ctypes.c_int]
    lib.moe_status_str.restype = ctypes.c_char_p
    lib.moe_last_error.argtypes = [P]
    lib.moe_last_error.restype = ctypes.c_char_p
    lib.moe_abi_version.restype = ctypes.c_int32
    if lib.moe_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI version {lib.moe_abi_version()} != {ABI_VERSION} (rebuild libmoe)")
    lib.moe_kernel_launches.argtypes = [P]
    lib.moe_kernel_launches.restype = ctypes.c_int64
    return lib


_lib = load_library()


def lib():
    return _lib


def _check(status, ctx=None):
    if status != MOE_OK:
        msg = _lib.moe_last_error(ctx).decode(errors="replace")
        raise MoeError(status, msg)


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _dev(t, dtype, device, name, ndim=None):
    """Device pointer of a tensor argument after checking what the C ABI assumes
    (dtype, dense row-major, on this context's device); None passes through."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise MoeError(1, f"{name}: expected a torch tensor, got {type(t).__name__}")
    if t.dtype != dtype:
        raise MoeError(1, f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise MoeError(1, f"{name}: must be contiguous")
    if t.device != device:
        raise MoeError(1, f"{name}: on {t.device}, the context is on {device}")
    if ndim is not None and t.dim() != ndim:
        raise MoeError(1, f"{name}: {t.dim()} dims, expected {ndim}")
    return ctypes.c_void_p(t.data_ptr())


def _np_ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def placement_contiguous(E, G):
    out = np.zeros(E, dtype=np.int32)
    _check(_lib.moe_placement_contiguous(E, G, _np_ptr(out)))
    return out


def layout_host(P, cnt):
    """Host layout (see moe_layout_host): returns seg_start, recv_base, recv_rows, send_base."""
    P = np.ascontiguousarray(P, dtype=np.int32)
    cnt = np.ascontiguousarray(cnt, dtype=np.int32)
    G, E = cnt.shape
    seg = np.zeros(E, np.int32)
    rb = np.zeros((G, E), np.int32)
    rr = np.zeros(G, np.int32)
    sb = np.zeros((G, E), np.int32)
    _check(_lib.moe_layout_host(E, G, _np_ptr(P), _np_ptr(cnt), _np_ptr(seg), _np_ptr(rb), _np_ptr(rr), _np_ptr(sb)))
    return seg, rb, rr, sb


def get_unique_id():
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.moe_get_unique_id(buf))
    return bytes(buf)


def pack_w13(w1, w3, stream=None):
    """w1, w3: bf16 [n][F][H] on the device -> w13 [n][2F][H] (moe_pack_w13)."""
    n, F, H = w1.shape
    w13 = torch.empty(n, 2 * F, H, dtype=torch.bfloat16, device=w1.device)
    _check(_lib.moe_pack_w13(_ptr(w1), _ptr(w3), n, F, H, _ptr(w13), _stream(stream)))
    return w13


def tp_slice_weights(w1, w3, w2, tp, q, stream=None):
    """TP slice q of tp (moe.h, moe_expert_ffn): w1, w3 bf16 [n][F][H], w2 [n][H][F]
    on the device -> (w13_q [n][2F/tp][H] packed, w2_q [n][H][F/tp] contiguous)."""
    F = w1.shape[1]
    f = F // tp
    sl = slice(q * f, (q + 1) * f)
    return (pack_w13(w1[:, sl].contiguous(), w3[:, sl].contiguous(), stream),
            w2[:, :, sl].contiguous())


class MoeLayer:
    """One libmoe context (one EP rank, or G virtual ranks on one GPU).

    tp > 1: tensor parallelism inside the experts (moe.h; reading G20) -- the G
    ranks form G/tp EP groups, the placement maps experts to groups.
    MoeLayer.group(n, ...): the n ranks of an EP group as n contexts of this
    process (moe_ctx_create_group), e.g. all on one GPU."""

    def __init__(self, *, max_tokens, hidden, ffn, num_experts, max_k, world=1, rank=0, device=0,
                 virtual_ranks=1, uid=None, a2a="nccl", tp=1, _handle=None):
        mode = {"nccl": 0, "p2p": 1}[a2a]
        self.cfg = Config(max_tokens, hidden, ffn, num_experts, max_k, world, rank, device, virtual_ranks, mode, tp)
        self.a2a = a2a
        self.tp = tp
        self.rank = rank
        self.E, self.H, self.F = num_experts, hidden, ffn
        self.G = virtual_ranks if virtual_ranks > 1 else world
        self.device = torch.device("cuda", device)
        self._placements = {}
        self._last = None
        if _handle is not None:
            self._ctx = _handle
            return
        h = ctypes.c_void_p()
        uid_buf = None
        if uid is not None:
            uid_buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(_lib.moe_ctx_create(ctypes.byref(self.cfg), uid_buf, ctypes.byref(h)))
        self._ctx = h

    @classmethod
    def group(cls, n, *, max_tokens, hidden, ffn, num_experts, max_k, devices=None, tp=1):
        """The n ranks of an EP group as n contexts of this process (moe.h,
        moe_ctx_create_group; P2P data plane, peer pointers without IPC/NCCL).
        devices: list of n device ordinals (default: all on the current device)."""
        dev0 = torch.cuda.current_device() if devices is None else int(devices[0])
        cfg = Config(max_tokens, hidden, ffn, num_experts, max_k, n, 0, dev0, 1, 1, tp)
        hs = (ctypes.c_void_p * n)()
        darr = None if devices is None else (ctypes.c_int32 * n)(*[int(d) for d in devices])
        _check(_lib.moe_ctx_create_group(ctypes.byref(cfg), n, darr, hs))
        return [cls(max_tokens=max_tokens, hidden=hidden, ffn=ffn, num_experts=num_experts, max_k=max_k, world=n,
                    rank=r, device=dev0 if devices is None else int(devices[r]), a2a="p2p", tp=tp,
                    _handle=ctypes.c_void_p(hs[r])) for r in range(n)]

    def close(self):
        if self._ctx:
            _lib.moe_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, status):
        _check(status, self._ctx)

    @property
    def kernel_launches(self):
        return int(_lib.moe_kernel_launches(self._ctx))

    def ffn_timing(self, max_records):
        """Arm per-call K5/K6 event records for the next max_records expert_ffn calls."""
        self._c(_lib.moe_ffn_timing_enable(self._ctx, int(max_records)))
        self._timing_max = int(max_records)

    def ffn_timing_read(self):
        """[(k5_ms, k6_ms)] of the recorded calls (synchronises; re-arms)."""
        n = getattr(self, "_timing_max", 0)
        ms = (ctypes.c_float * (2 * max(n, 1)))()
        got = ctypes.c_int32()
        self._c(_lib.moe_ffn_timing_read(self._ctx, ms, n, ctypes.byref(got)))
        return [(float(ms[2 * i]), float(ms[2 * i + 1])) for i in range(got.value)]

    TIMELINE = ("dispatch", "layout", "scatter_local", "scatter_peers", "ffn", "k5", "k6", "combine")

    def timeline(self, max_records):
        """Arm the 8-event layer timeline for the next max_records layers (moe.h)."""
        self._c(_lib.moe_timeline_enable(self._ctx, int(max_records)))
        self._tl_max = int(max_records)

    def timeline_read(self):
        """[[ms of each TIMELINE event after dispatch entry] per recorded layer]."""
        n = getattr(self, "_tl_max", 0)
        ms = (ctypes.c_float * (8 * max(n, 1)))()
        got = ctypes.c_int32()
        self._c(_lib.moe_timeline_read(self._ctx, ms, n, ctypes.byref(got)))
        return [[float(ms[8 * i + j]) for j in range(8)] for i in range(got.value)]

    def sync(self):
        self._c(_lib.moe_ctx_sync(self._ctx))

    # a1
    def route(self, logits, k, idx=None, w=None, stream=None):
        T, E = logits.shape
        if idx is None:
            idx = torch.empty(T, k, dtype=torch.int32, device=logits.device)
        if w is None:
            w = torch.empty(T, k, dtype=torch.float32, device=logits.device)
        d = self.device
        self._c(_lib.moe_route(self._ctx, _dev(logits, torch.float32, d, "logits", 2), T, E, k,
                               _dev(idx, torch.int32, d, "idx", 2), _dev(w, torch.float32, d, "w", 2),
                               _stream(stream)))
        return idx, w

    # a2
    def route_stats(self, idx_l, idx_l1, load, coact, stream=None):
        T, k = idx_l.shape
        d = self.device
        self._c(_lib.moe_route_stats(self._ctx, _dev(idx_l, torch.int32, d, "idx_l", 2),
                                     _dev(idx_l1, torch.int32, d, "idx_l1", 2), T, self.E, k,
                                     _dev(load, torch.int64, d, "load"), _dev(coact, torch.int64, d, "coact"),
                                     _stream(stream)))

    def stats_allreduce(self, load, coact, stream=None):
        d = self.device
        self._c(_lib.moe_stats_allreduce(self._ctx, _dev(load, torch.int64, d, "load"),
                                         _dev(coact, torch.int64, d, "coact"), self.E, _stream(stream)))

    def stats_allreduce_layers(self, load, coact, stream=None):
        """load int64 [L][E], coact int64 [L-1][E][E] (or None): one collective."""
        L = load.shape[0]
        d = self.device
        self._c(_lib.moe_stats_allreduce_layers(self._ctx, _dev(load, torch.int64, d, "load"),
                                                _dev(coact, torch.int64, d, "coact"), self.E, L, _stream(stream)))

    def placement(self, expert_to_rank):
        """The device int32 [E] placement array moe_dispatch reads.  A torch tensor on
        this device passes through; a host sequence is uploaded once and cached (by
        value), so repeated dispatches with the same placement copy nothing."""
        if isinstance(expert_to_rank, torch.Tensor) and expert_to_rank.is_cuda:
            return expert_to_rank
        P = np.ascontiguousarray(np.asarray(expert_to_rank), dtype=np.int32)
        key = P.tobytes()
        t = self._placements.get(key)
        if t is None:
            t = torch.from_numpy(P.copy()).to(self.device)
            self._placements[key] = t
        return t

    # a3-a5
    def dispatch(self, x, idx, expert_to_rank, info=False, stream=None):
        T, k = idx.shape
        d = self.device
        P = self.placement(expert_to_rank)
        inf = DispatchInfo() if info else None
        self._c(_lib.moe_dispatch(self._ctx, _dev(x, torch.bfloat16, d, "x", 2), _dev(idx, torch.int32, d, "idx", 2),
                                  T, k, _dev(P, torch.int32, d, "expert_to_rank", 1),
                                  ctypes.byref(inf) if inf is not None else None, _stream(stream)))
        self._last = (T, k)
        return inf

    def dispatch_from(self, prev, w_prev, idx, expert_to_rank, stream=None):
        """NEXT-4 direct dispatch (moe.h, moe_dispatch_from): this layer's receive rows
        are combined on the hosting ranks from layer `prev`'s expert outputs (prev:
        the MoeLayer of layer l on this rank, run with output_mode("stay"))."""
        T, k = idx.shape
        d = self.device
        P = self.placement(expert_to_rank)
        self._c(_lib.moe_dispatch_from(self._ctx, prev._ctx, _dev(w_prev, torch.float32, d, "w_prev", 2),
                                       _dev(idx, torch.int32, d, "idx", 2), T, k,
                                       _dev(P, torch.int32, d, "expert_to_rank", 1), _stream(stream)))
        self._last = (T, k)

    def output_mode(self, mode):
        """"home" (default: moe_combine returns the outputs) or "stay" (they stay on the
        hosting ranks for the next layer's dispatch_from)."""
        self._c(_lib.moe_set_output_mode(self._ctx, {"home": 0, "stay": 1}[mode]))

    # a6
    def expert_ffn(self, w13, w2, stream=None):
        """w13 bf16 [n_w][2F][H] (pack_w13), w2 bf16 [n_w][H][F]: the experts the last
        dispatch's placement hosts here (n_w may be 0: w13 = w2 = None)."""
        d = self.device
        n_w = 0 if w13 is None else int(w13.shape[0])
        self._c(_lib.moe_expert_ffn(self._ctx, _dev(w13, torch.bfloat16, d, "w13", 3),
                                    _dev(w2, torch.bfloat16, d, "w2", 3), n_w, _stream(stream)))

    def identity_ffn(self, stream=None):
        self._c(_lib.moe_debug_identity_ffn(self._ctx, _stream(stream)))

    # a7-a8
    def combine(self, w, out=None, stream=None):
        T, k = self._last
        if out is None:
            out = torch.empty(T, self.H, dtype=torch.bfloat16, device=self.device)
        d = self.device
        self._c(_lib.moe_combine(self._ctx, _dev(w, torch.float32, d, "w", 2), _dev(out, torch.bfloat16, d, "out", 2),
                                 _stream(stream)))
        return out

    # debug views
    def debug_plan(self):
        T, k = self._last
        dr = np.zeros((T, k), np.int32)
        rp = np.zeros((T, k), np.int32)
        ss = np.zeros((T, k), np.int32)
        cnt = np.zeros((self.G, self.E), np.int32)
        self._c(_lib.moe_debug_plan(self._ctx, _np_ptr(dr), _np_ptr(rp), _np_ptr(ss), _np_ptr(cnt)))
        return dr, rp, ss, cnt

    def debug_recv(self):
        n = ctypes.c_int64()
        self._c(_lib.moe_debug_recv(self._ctx, None, 0, ctypes.byref(n)))
        buf = np.zeros((max(n.value, 1), self.H), np.uint16)
        self._c(_lib.moe_debug_recv(self._ctx, _np_ptr(buf), n.value, ctypes.byref(n)))
        return buf[:n.value]

    def debug_send(self):
        """NCCL mode: this rank's compact send buffer (remote rows in C3 send order);
        copy-engine mode: the staging buffer indexed by the C3 send slot (moe.h)."""
        n = ctypes.c_int64()
        self._c(_lib.moe_debug_send(self._ctx, None, 0, ctypes.byref(n)))
        buf = np.zeros((max(n.value, 1), self.H), np.uint16)
        self._c(_lib.moe_debug_send(self._ctx, _np_ptr(buf), n.value, ctypes.byref(n)))
        return buf[:n.value]
