"""Thin ctypes binding of the C ABI in include/fastformers.h.

Argument marshalling only: every step of the forward pass runs in the sm_100a
kernels of ``libfastformers.so``.  PyTorch is used for device memory (the two
caller-owned arenas and the ids / mask / logits tensors) and streams.  If the
library is missing or the device is not a B200 this module raises -- there is
no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# FF_LIB_PATH: load another build of the library (A/B experiments, tools/ab_lib.py)
LIB_PATH = os.environ.get("FF_LIB_PATH") or os.path.join(_PKG, "libfastformers.so")

FF_OK, FF_E_INVALID, FF_E_SHAPE, FF_E_STATE, FF_E_CUDA, FF_E_INPUT, FF_E_UNSUPPORTED, FF_E_NOMEM = range(8)
FF_F16, FF_I8 = 0, 1
FF_OPT_GRAPHS = 1
FF_OPT_CTA_PAIRS = 2
FF_OPT_ATTN_TC = 3
FF_OPT_FUSED_EPILOGUES = 4
FF_OPT_PDL = 5
FF_OPT_ACT_QUANT = 6
FF_OPT_FUSED_MASK = 8
FF_OPT_PDL_RR = 9
FF_OPT_CLS_LAST_LAYER = 13
FF_OPT_ROW_DIRS = 14
FF_SCORER_OPT_TC_LINEARS = 1  # ff_scorer_set_option
KERNEL_KINDS = ["embed_ln", "gemm_f16", "gemm_i8", "attention", "quant_rows", "add_ln", "head", "gemm_rr_f16",
                "gemm_rr_i8"]
STATUS_NAMES = ["FF_OK", "FF_E_INVALID", "FF_E_SHAPE", "FF_E_STATE", "FF_E_CUDA", "FF_E_INPUT", "FF_E_UNSUPPORTED",
                "FF_E_NOMEM"]

EXPORTED = ["ff_abi_version", "ff_last_error", "ff_model_create", "ff_model_memory", "ff_bind_memory",
            "ff_load_weights", "ff_finalize", "ff_encode", "ff_encode_host", "ff_encode_host_async", "ff_check", "ff_set_option", "ff_get_option",
            "ff_model_destroy", "ff_launch_count", "ff_profile", "ff_encode_trace", "ff_debug_gemm", "ff_debug_quant_rows",
            "ff_debug_attention", "ff_debug_attention_q8", "ff_debug_set_trace",
            "ff_scorer_last_error", "ff_scorer_create", "ff_scorer_memory", "ff_scorer_bind_memory",
            "ff_scorer_load_weights", "ff_scorer_finalize", "ff_score_batch", "ff_scorer_check", "ff_scorer_set_option", "ff_debug_gemm_x3",
            "ff_scorer_destroy"]


class FFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


class FFConfig(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("num_layers", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("vocab_size", ctypes.c_int32), ("max_positions", ctypes.c_int32),
                ("num_classes", ctypes.c_int32), ("ln_eps", ctypes.c_float), ("act", ctypes.c_int32),
                ("heads", ctypes.POINTER(ctypes.c_int32)), ("ffn_dim", ctypes.POINTER(ctypes.c_int32)),
                ("dtype", ctypes.POINTER(ctypes.c_int32)), ("max_tokens", ctypes.c_int32)]


_lib = None


def lib():
    """Load libfastformers.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FFError(FF_E_CUDA, f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        L.ff_abi_version.restype = i32
        L.ff_last_error.restype = ctypes.c_char_p
        L.ff_model_create.argtypes = [ctypes.POINTER(FFConfig), i32, ctypes.POINTER(vp)]
        L.ff_model_memory.argtypes = [vp, ctypes.POINTER(sz), ctypes.POINTER(sz)]
        L.ff_bind_memory.argtypes = [vp, vp, sz, vp, sz, vp]
        L.ff_load_weights.argtypes = [vp, ctypes.c_char_p, vp, ctypes.POINTER(ctypes.c_int64), i32, vp]
        L.ff_finalize.argtypes = [vp, vp]
        L.ff_encode.argtypes = [vp, vp, vp, i32, i32, vp, vp]
        L.ff_encode_host.argtypes = [vp, vp, vp, i32, i32, vp, vp]
        L.ff_encode_host_async.argtypes = [vp, vp, vp, i32, i32, vp, vp]
        L.ff_check.argtypes = [vp, vp]
        L.ff_set_option.argtypes = [vp, i32, ctypes.c_int64]
        L.ff_get_option.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_int64)]
        L.ff_model_destroy.argtypes = [vp]
        L.ff_model_destroy.restype = None
        L.ff_launch_count.argtypes = [vp, i32, i32, ctypes.POINTER(i32)]
        L.ff_profile.argtypes = [vp, vp, vp, i32, i32, vp, i32, vp, vp, ctypes.POINTER(i32), vp]
        L.ff_encode_trace.argtypes = [vp, vp, vp, i32, i32, vp, i32, ctypes.POINTER(vp), vp]
        L.ff_debug_gemm.argtypes = [i32, vp, i32, vp, i32, i32, i32, i32, i32, vp, i32, vp, vp, vp, i32, vp]
        L.ff_debug_quant_rows.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp]
        L.ff_debug_attention.argtypes = [vp, vp, i32, i32, i32, i32, vp, i32, vp]
        L.ff_debug_attention_q8.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp]
        L.ff_debug_set_trace.argtypes = [vp, i32]
        L.ff_scorer_last_error.restype = ctypes.c_char_p
        L.ff_scorer_create.argtypes = [ctypes.POINTER(FFConfig), i32, ctypes.POINTER(vp)]
        L.ff_scorer_memory.argtypes = [vp, ctypes.POINTER(sz), ctypes.POINTER(sz)]
        L.ff_scorer_bind_memory.argtypes = [vp, vp, sz, vp, sz]
        L.ff_scorer_load_weights.argtypes = [vp, ctypes.c_char_p, vp, ctypes.POINTER(ctypes.c_int64), i32, vp]
        L.ff_scorer_finalize.argtypes = [vp, vp]
        L.ff_score_batch.argtypes = [vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]
        L.ff_scorer_check.argtypes = [vp, vp]
        L.ff_scorer_set_option.argtypes = [vp, i32, i32]
        L.ff_debug_gemm_x3.argtypes = [vp, i32, vp, i32, i32, i32, i32, vp, vp, i32, i32, i32, vp]
        L.ff_scorer_destroy.argtypes = [vp]
        L.ff_scorer_destroy.restype = None
        for name in EXPORTED:
            if name not in ("ff_abi_version", "ff_last_error", "ff_model_destroy", "ff_scorer_last_error",
                            "ff_scorer_destroy"):
                getattr(L, name).restype = i32
        _lib = L
    return _lib


def check(status: int):
    if status != FF_OK:
        raise FFError(status, lib().ff_last_error().decode(errors="replace"))


def _stream_ptr(stream=None, device=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _check_tensor(t, dtype, device, what):
    """Argument marshalling guard: the C ABI reads raw pointers, so a wrong
    dtype / layout / device would be silently misread."""
    assert t.dtype == dtype, f"{what}: expected {dtype}, got {t.dtype}"
    assert t.is_contiguous(), f"{what} must be contiguous"
    if device is not None:
        assert t.device == device, f"{what} must be on {device}, is on {t.device}"
    else:
        assert t.device.type == "cpu", f"{what} must be a host tensor"


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class Encoder:
    """One FastFormers encoder model on one GPU (weights packed once at load)."""

    def __init__(self, cfg, weights: Dict[str, np.ndarray], max_tokens: Optional[int] = None, device: int = 0,
                 use_graphs: bool = True, cta_pairs: bool = True, attn_tc: bool = True, fused=None,
                 act_quant: int = 0, cls_last: bool = False):
        import torch
        L = lib()
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        self._heads = (ctypes.c_int32 * cfg.num_layers)(*cfg.heads)
        self._ffn = (ctypes.c_int32 * cfg.num_layers)(*cfg.ffn_dim)
        self._dt = (ctypes.c_int32 * cfg.num_layers)(*cfg.dtype)
        self.max_tokens = int(max_tokens or cfg.batch * cfg.seq)
        c = FFConfig(1, cfg.num_layers, cfg.hidden, cfg.head_dim, cfg.vocab_size, cfg.max_positions,
                     cfg.num_classes, float(cfg.ln_eps), int(cfg.act), self._heads, self._ffn, self._dt,
                     self.max_tokens)
        h = ctypes.c_void_p()
        check(L.ff_model_create(ctypes.byref(c), device, ctypes.byref(h)))
        self.h = h
        wb, wsb = ctypes.c_size_t(), ctypes.c_size_t()
        check(L.ff_model_memory(self.h, ctypes.byref(wb), ctypes.byref(wsb)))
        with torch.cuda.device(self.device):
            self.weight_arena = torch.empty(wb.value, dtype=torch.uint8, device=self.device)
            self.workspace = torch.empty(wsb.value, dtype=torch.uint8, device=self.device)
            st = _stream_ptr()
            check(L.ff_bind_memory(self.h, _ptr(self.weight_arena), wb.value, _ptr(self.workspace), wsb.value, st))
            for name, w in weights.items():
                a = np.ascontiguousarray(w, dtype=np.float32)
                shape = (ctypes.c_int64 * a.ndim)(*a.shape)
                check(L.ff_load_weights(self.h, name.encode(), ctypes.c_void_p(a.ctypes.data), shape, a.ndim, st))
            check(L.ff_finalize(self.h, st))
        if not use_graphs:
            check(L.ff_set_option(self.h, FF_OPT_GRAPHS, 0))
        if not attn_tc:
            check(L.ff_set_option(self.h, FF_OPT_ATTN_TC, 0))
        # fused: None = library default (FF_OPT_FUSED_MASK 2: FFN1 + requant), False / True
        # (none / all three fusions) or a FF_OPT_FUSED_MASK bitmask
        if fused is None:
            pass
        elif isinstance(fused, bool):
            check(L.ff_set_option(self.h, FF_OPT_FUSED_EPILOGUES, 1 if fused else 0))
        else:
            check(L.ff_set_option(self.h, FF_OPT_FUSED_MASK, int(fused)))
        self.fused = fused
        # int8 activation quantizer: 0 per-row s8 (default), 1 per-tensor u8 + zero point
        check(L.ff_set_option(self.h, FF_OPT_ACT_QUANT, int(act_quant)))
        self.act_quant = act_quant
        if not cta_pairs:
            check(L.ff_set_option(self.h, FF_OPT_CTA_PAIRS, 0))
        # FF_OPT_CLS_LAST_LAYER: last layer's row-local steps on the first tokens only
        if cls_last:
            check(L.ff_set_option(self.h, FF_OPT_CLS_LAST_LAYER, 1))

    def get_option(self, option: int) -> int:
        v = ctypes.c_int64()
        check(lib().ff_get_option(self.h, option, ctypes.byref(v)))
        return v.value

    def fused_mask(self) -> int:
        """FF_OPT_FUSED_MASK in effect."""
        return self.get_option(FF_OPT_FUSED_MASK)

    def set_fused(self, mask: int):
        """FF_OPT_FUSED_MASK: bit 0 out-proj+LN1, bit 1 FFN1+requant, bit 2 FFN2+LN2."""
        check(lib().ff_set_option(self.h, FF_OPT_FUSED_MASK, int(mask)))
        self.fused = mask

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.ff_model_destroy(h)
            self.h = None

    def encode(self, ids, mask, logits=None, stream=None):
        """ids, mask: int32 [B, S] CUDA tensors -> logits fp32 [B, C] (async on the stream;
        default: the current stream of the model's device)."""
        import torch
        B, S = ids.shape
        _check_tensor(ids, torch.int32, self.device, "ids")
        _check_tensor(mask, torch.int32, self.device, "mask")
        if logits is None:
            logits = torch.empty((B, self.cfg.num_classes), dtype=torch.float32, device=ids.device)
        _check_tensor(logits, torch.float32, self.device, "logits")
        assert tuple(logits.shape) == (B, self.cfg.num_classes), "logits must be [B, num_classes]"
        check(lib().ff_encode(self.h, _ptr(ids), _ptr(mask), B, S, _ptr(logits), _stream_ptr(stream, self.device)))
        return logits

    def encode_host(self, ids, mask, logits=None, stream=None):
        """End-to-end: host (ideally pinned) int32 ids / mask -> host fp32 logits."""
        import torch
        B, S = ids.shape
        if logits is None:
            logits = torch.empty((B, self.cfg.num_classes), dtype=torch.float32).pin_memory()
        for t, dt, n in ((ids, torch.int32, "ids"), (mask, torch.int32, "mask"), (logits, torch.float32, "logits")):
            _check_tensor(t, dt, None, n)
        check(lib().ff_encode_host(self.h, _ptr(ids), _ptr(mask), B, S, _ptr(logits), _stream_ptr(stream, self.device)))
        return logits

    def encode_host_async(self, ids, mask, logits, stream=None):
        """ff_encode_host_async: pinned host ids / mask -> pinned host logits, enqueued
        without synchronizing (read `logits` only after the stream is synchronized)."""
        import torch
        B, S = ids.shape
        for t, dt, n in ((ids, torch.int32, "ids"), (mask, torch.int32, "mask"), (logits, torch.float32, "logits")):
            _check_tensor(t, dt, None, n)
        check(lib().ff_encode_host_async(self.h, _ptr(ids), _ptr(mask), B, S, _ptr(logits),
                                         _stream_ptr(stream, self.device)))
        return logits

    def check_inputs(self, stream=None):
        check(lib().ff_check(self.h, _stream_ptr(stream)))

    def launch_count(self, B, S):
        n = ctypes.c_int32()
        check(lib().ff_launch_count(self.h, B, S, ctypes.byref(n)))
        return n.value

    def profile(self, ids, mask, logits=None, stream=None):
        """One un-graphed forward with CUDA events around every launch.
        Returns a list of (kind, ms) with kind in KERNEL_KINDS."""
        import torch
        B, S = ids.shape
        if logits is None:
            logits = torch.empty((B, self.cfg.num_classes), dtype=torch.float32, device=ids.device)
        cap = 4096
        kinds = (ctypes.c_int32 * cap)()
        ms = (ctypes.c_float * cap)()
        n = ctypes.c_int32()
        check(lib().ff_profile(self.h, _ptr(ids), _ptr(mask), B, S, _ptr(logits), cap, ctypes.cast(kinds, ctypes.c_void_p),
                               ctypes.cast(ms, ctypes.c_void_p), ctypes.byref(n), _stream_ptr(stream)))
        return [(KERNEL_KINDS[kinds[i]], ms[i]) for i in range(n.value)]

    def trace(self, ids, mask, layer: int):
        """Run the forward and return layer `layer`'s fp16 stage tensors (packed, on device)."""
        import torch
        cfg = self.cfg
        B, S = ids.shape
        M, H = B * S, cfg.hidden
        D, F = cfg.heads[layer] * cfg.head_dim, cfg.ffn_dim[layer]
        names = ["x_in", "qkv", "ctx", "o", "h1", "i", "y", "x_out"]
        cols = [H, 3 * D, D, H, H, F, H, H]
        bufs = [torch.empty((M, c), dtype=torch.float16, device=ids.device) for c in cols]
        ptrs = (ctypes.c_void_p * 8)(*[b.data_ptr() for b in bufs])
        logits = torch.empty((B, cfg.num_classes), dtype=torch.float32, device=ids.device)
        check(lib().ff_encode_trace(self.h, _ptr(ids), _ptr(mask), B, S, _ptr(logits), layer, ptrs, _stream_ptr()))
        out = dict(zip(names, bufs))
        out["logits"] = logits
        return out


# ------------------------------------------------------------ debug entry points
def gemm(A, W, out_mode=0, bias=None, sx=None, sw=None, act=-1, out=None, cta_pair=None):
    """C = A W^T through the production tcgen05 kernel.  A [M,K], W [N,K]: both
    int8 (kind::i8) or both fp16 (kind::f16) CUDA tensors with 16-byte aligned rows."""
    import torch
    M, K = A.shape
    N = W.shape[0]
    i8 = A.dtype == torch.int8
    if out is None:
        if out_mode == 0:
            out = torch.empty((M, N), dtype=torch.int32 if i8 else torch.float32, device=A.device)
        else:
            out = torch.empty((M, N), dtype=torch.float16, device=A.device)
    nul = ctypes.c_void_p(None)
    mode = out_mode | (0 if cta_pair is None else (16 if cta_pair else 32))
    check(lib().ff_debug_gemm(FF_I8 if i8 else FF_F16, _ptr(A), A.stride(0), _ptr(W), W.stride(0), M, N, K, mode,
                              _ptr(out), out.stride(0), _ptr(bias) if bias is not None else nul,
                              _ptr(sx) if sx is not None else nul, _ptr(sw) if sw is not None else nul, act,
                              _stream_ptr()))
    return out


def quant_rows(x16):
    import torch
    M, K = x16.shape
    ldq = (K + 15) // 16 * 16
    q = torch.empty((M, ldq), dtype=torch.int8, device=x16.device)
    s = torch.empty(M, dtype=torch.float32, device=x16.device)
    check(lib().ff_debug_quant_rows(_ptr(x16), M, K, x16.stride(0), _ptr(q), ldq, _ptr(s), _stream_ptr()))
    return q[:, :K], s


def attention(qkv16, mask, A, d, impl=0):
    """impl: 0 auto, 1 mma.sync kernel, 2 tcgen05 kernel (head_dim 64 or even <= 32, S <= 128)."""
    import torch
    B, S = mask.shape
    ctx = torch.empty((B * S, A * d), dtype=torch.float16, device=qkv16.device)
    check(lib().ff_debug_attention(_ptr(qkv16), _ptr(mask), B, S, A, d, _ptr(ctx), impl, _stream_ptr()))
    return ctx


def attention_q8(qkv16, mask, A, d, with_ctx16=True, trace=None):
    """tcgen05 attention with the int8 ctx requant fused: (ctx16 or None, q s8, scales).
    trace: optional int64 CUDA tensor [min(B,148), 32, 8] for event timestamps."""
    import torch
    B, S = mask.shape
    dev = qkv16.device
    ctx = torch.empty((B * S, A * d), dtype=torch.float16, device=dev) if with_ctx16 else None
    q = torch.empty((B * S, A * d), dtype=torch.int8, device=dev)
    s = torch.empty(B * S, dtype=torch.float32, device=dev)
    check(lib().ff_debug_attention_q8(_ptr(qkv16), _ptr(mask), B, S, A, d, _ptr(ctx) if ctx is not None else None,
                                      _ptr(q), _ptr(s), _ptr(trace) if trace is not None else None,
                                      _stream_ptr()))
    return ctx, q, s


def set_gemm_trace(trace=None, which=0):
    """Debug: record per-tile timestamps into `trace` (zeroed int64 CUDA tensor
    [grid, 64, 24]) — which = 0: subsequent debug GEMMs; 1/2/3: the layer-0
    fused out-proj+LN / FFN1+requant / FFN2+LN of subsequent forwards."""
    check(lib().ff_debug_set_trace(_ptr(trace) if trace is not None else None, which))


def _scheck(status: int):
    if status != FF_OK:
        raise FFError(status, lib().ff_scorer_last_error().decode(errors="replace"))


def gemm_x3(A, B, bias=None, out=None, accumulate=False, kc=2):
    """ff_debug_gemm_x3: C (+)= A B^T (+ bias) on the scorer's 3xFP16 tcgen05
    GEMM; A [M, K], B [N, K] fp32 CUDA tensors (unit column stride)."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    if out is None:
        out = torch.zeros((M, N), dtype=torch.float32, device=A.device)
    nul = ctypes.c_void_p(None)
    _scheck(lib().ff_debug_gemm_x3(_ptr(A), A.stride(0), _ptr(B), B.stride(0), M, N, K,
                                   _ptr(bias) if bias is not None else nul, _ptr(out), out.stride(0),
                                   1 if accumulate else 0, kc, _stream_ptr()))
    return out


class Scorer:
    """Structured-pruning importance scorer on one GPU (C-ABI ff_scorer_*;
    SURVEY 8(f) NEXT-3).  Holds the UNPRUNED model in fp32;
    ``score(ids, mask, labels)`` adds |dL/dmask| of every head and FFN unit
    to ``head_scores`` [L, max heads] / ``ffn_scores`` [L, max ffn] (fp64,
    device) and returns the batch's mean cross-entropy (device scalar)."""

    def __init__(self, cfg, weights: Dict[str, np.ndarray], max_tokens: Optional[int] = None, device: int = 0,
                 tc_linears: bool = True):
        import torch
        L = lib()
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        self._heads = (ctypes.c_int32 * cfg.num_layers)(*cfg.heads)
        self._ffn = (ctypes.c_int32 * cfg.num_layers)(*cfg.ffn_dim)
        self._dt = (ctypes.c_int32 * cfg.num_layers)(*([0] * cfg.num_layers))
        self.max_tokens = int(max_tokens or cfg.batch * cfg.seq)
        c = FFConfig(1, cfg.num_layers, cfg.hidden, cfg.head_dim, cfg.vocab_size, cfg.max_positions,
                     cfg.num_classes, float(cfg.ln_eps), int(cfg.act), self._heads, self._ffn, self._dt,
                     self.max_tokens)
        h = ctypes.c_void_p()
        _scheck(L.ff_scorer_create(ctypes.byref(c), device, ctypes.byref(h)))
        self.h = h
        self.set_tc_linears(tc_linears)
        wb, wsb = ctypes.c_size_t(), ctypes.c_size_t()
        _scheck(L.ff_scorer_memory(self.h, ctypes.byref(wb), ctypes.byref(wsb)))
        with torch.cuda.device(self.device):
            self.weight_arena = torch.empty(wb.value, dtype=torch.uint8, device=self.device)
            self.workspace = torch.empty(wsb.value, dtype=torch.uint8, device=self.device)
            _scheck(L.ff_scorer_bind_memory(self.h, _ptr(self.weight_arena), wb.value, _ptr(self.workspace),
                                            wsb.value))
            st = _stream_ptr()
            for name, w in weights.items():
                a = np.ascontiguousarray(w, dtype=np.float32)
                shape = (ctypes.c_int64 * a.ndim)(*a.shape)
                _scheck(L.ff_scorer_load_weights(self.h, name.encode(), ctypes.c_void_p(a.ctypes.data), shape,
                                                 a.ndim, st))
            _scheck(L.ff_scorer_finalize(self.h, st))
            self.head_scores = torch.zeros((cfg.num_layers, max(cfg.heads)), dtype=torch.float64,
                                           device=self.device)
            self.ffn_scores = torch.zeros((cfg.num_layers, max(cfg.ffn_dim)), dtype=torch.float64,
                                          device=self.device)
            self.loss = torch.zeros(1, dtype=torch.float32, device=self.device)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.ff_scorer_destroy(h)

    def set_tc_linears(self, on: bool):
        """FF_SCORER_OPT_TC_LINEARS: 3xTF32 tcgen05 linears (default) or the SIMT SGEMM."""
        _scheck(lib().ff_scorer_set_option(self.h, FF_SCORER_OPT_TC_LINEARS, 1 if on else 0))

    def reset(self):
        self.head_scores.zero_()
        self.ffn_scores.zero_()

    def score(self, ids, mask, labels, logits=None, stream=None):
        """ids, mask [B, S], labels [B]: int32 tensors on the scorer's device."""
        import torch
        B, S = ids.shape
        for t, n in ((ids, "ids"), (mask, "mask"), (labels, "labels")):
            _check_tensor(t, torch.int32, self.device, n)
        assert labels.shape == (B,), "labels must be [B]"
        if logits is not None:
            _check_tensor(logits, torch.float32, self.device, "logits")
        nul = ctypes.c_void_p(None)
        _scheck(lib().ff_score_batch(self.h, _ptr(ids), _ptr(mask), _ptr(labels), B, S, _ptr(self.head_scores),
                                     _ptr(self.ffn_scores), _ptr(self.loss),
                                     _ptr(logits) if logits is not None else nul,
                                     _stream_ptr(stream, self.device)))
        return self.loss

    def check_inputs(self, stream=None):
        """ff_scorer_check: raises FFError(FF_E_INPUT) if a scored batch had invalid ids / mask / labels."""
        _scheck(lib().ff_scorer_check(self.h, _stream_ptr(stream)))

    def scores(self):
        """(head_scores [L][A_l], ffn_scores [L][F_l]) as numpy, trimmed per layer."""
        hs, fs = self.head_scores.cpu().numpy(), self.ffn_scores.cpu().numpy()
        return ([hs[l, :self.cfg.heads[l]] for l in range(self.cfg.num_layers)],
                [fs[l, :self.cfg.ffn_dim[l]] for l in range(self.cfg.num_layers)])
