"""CPU oracle for the FastFormers encoder forward -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
wraps ``oracle/oracle.cpp`` (plain C++, see that file's header for the modes
and citations) through ctypes and shares no code with the CUDA library.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

MODE_REF64 = 0
MODE_EMU = 1
ST_QKV, ST_ATTN, ST_OPROJ, ST_LN1, ST_FFN1, ST_FFN2, ST_LN2 = range(7)


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-O2, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               _SRC, "-o", _LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32p = ctypes.POINTER(ctypes.c_int32)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        i8p = ctypes.POINTER(ctypes.c_int8)
        i64p = ctypes.POINTER(ctypes.c_int64)
        c_int, c_float = ctypes.c_int, ctypes.c_float
        L.or_create.restype = P
        L.or_create.argtypes = [c_int] * 6 + [c_float, c_int, i32p, i32p, i32p]
        L.or_destroy.argtypes = [P]
        L.or_load.argtypes = [P, ctypes.c_char_p, f32p, i64p, c_int]
        L.or_finalize.argtypes = [P]
        L.or_encode.argtypes = [P, i32p, i32p, c_int, c_int, c_int, c_int, f32p, f64p, f32p]
        L.or_stage.argtypes = [P, c_int, c_int, f32p, f32p, i32p, c_int, c_int, c_int, f32p]
        L.or_embed.argtypes = [P, i32p, c_int, c_int, c_int, f32p]
        L.or_head.argtypes = [P, f32p, c_int, c_int, f32p]
        L.or_prepared_weight.argtypes = [P, c_int, c_int, i8p, f32p, f32p]
        L.or_q8row.argtypes = [f32p, c_int, c_int, i8p, f32p]
        L.or_quant_weight.argtypes = [f32p, c_int, c_int, i8p, f32p]
        L.or_q8tensor.argtypes = [f32p, c_int, c_int, ctypes.POINTER(ctypes.c_uint8), f32p, i32p]
        L.or_set_act_quant.argtypes = [P, c_int]
        L.or_gemm_s8.argtypes = [i8p, i8p, c_int, c_int, c_int, i32p]
        L.or_r16.argtypes = [f32p, ctypes.c_size_t, f32p]
        L.or_act.argtypes = [f32p, ctypes.c_size_t, c_int, f64p]
        L.or_layer_norm64.argtypes = [f64p, c_int, c_int, f32p, f32p, c_float, f64p]
        L.or_attention.argtypes = [f32p, i32p, c_int, c_int, c_int, c_int, c_int, f32p]
        L.or_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _check(rc: int):
    if rc != 0:
        raise RuntimeError(f"oracle error {rc}: {lib().or_last_error().decode()}")


class Oracle:
    """One oracle model.  ``cfg`` is a ``paper_2010_13382_b200.synth.ModelConfig``-like
    object with fields num_layers, hidden, head_dim, vocab_size, max_positions,
    num_classes, ln_eps, act, heads, ffn_dim, dtype (ints: 0 = f16, 1 = i8)."""

    def __init__(self, cfg, weights: dict | None = None, act_quant: int = 0):
        """act_quant: int8 activation quantizer, 0 = Q8row (per row, default),
        1 = Q8tensor (per tensor, u8 with zero point; DESIGN R22)."""
        L = lib()
        self.cfg = cfg
        heads = _i32(cfg.heads)
        ffn = _i32(cfg.ffn_dim)
        dt = _i32(cfg.dtype)
        self.h = L.or_create(cfg.num_layers, cfg.hidden, cfg.head_dim, cfg.vocab_size, cfg.max_positions,
                             cfg.num_classes, float(cfg.ln_eps), int(cfg.act), _p(heads, ctypes.c_int32),
                             _p(ffn, ctypes.c_int32), _p(dt, ctypes.c_int32))
        if not self.h:
            raise RuntimeError("or_create failed: " + L.or_last_error().decode())
        _check(L.or_set_act_quant(self.h, int(act_quant)))
        if weights is not None:
            self.load(weights)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_destroy(self.h)
            self.h = None

    def load(self, weights: dict):
        for name, w in weights.items():
            a = _f32(w)
            shape = np.asarray(a.shape, dtype=np.int64)
            _check(lib().or_load(self.h, name.encode(), _p(a, ctypes.c_float), _p(shape, ctypes.c_int64), a.ndim))
        _check(lib().or_finalize(self.h))

    def encode(self, ids, mask, mode=MODE_EMU, acc32=False, return_hidden=False, fp64_logits=False):
        ids, mask = _i32(ids), _i32(mask)
        B, S = ids.shape
        logits = np.zeros((B, self.cfg.num_classes), np.float32)
        l64 = np.zeros((B, self.cfg.num_classes), np.float64)
        hid = np.zeros((B * S, self.cfg.hidden), np.float32) if return_hidden else None
        _check(lib().or_encode(self.h, _p(ids, ctypes.c_int32), _p(mask, ctypes.c_int32), B, S, mode, int(acc32),
                               _p(logits, ctypes.c_float), _p(l64, ctypes.c_double),
                               _p(hid, ctypes.c_float) if hid is not None else None))
        out = l64 if fp64_logits else logits
        return (out, hid) if return_hidden else out

    def stage(self, layer: int, stage: int, a, b=None, mask=None, B=None, S=None, acc32=False):
        cfg = self.cfg
        a = _f32(a)
        M = a.shape[0]
        A, F, H, d = cfg.heads[layer], cfg.ffn_dim[layer], cfg.hidden, cfg.head_dim
        D = A * d
        ncol = {ST_QKV: 3 * D, ST_ATTN: D, ST_OPROJ: H, ST_LN1: H, ST_FFN1: F, ST_FFN2: H, ST_LN2: H}[stage]
        out = np.zeros((M, ncol), np.float32)
        if mask is None:
            mask = np.ones((B, S), np.int32) if B is not None else np.ones((1, M), np.int32)
        mask = _i32(mask)
        if B is None:
            B, S = mask.shape
        bb = _f32(b) if b is not None else None
        _check(lib().or_stage(self.h, layer, stage, _p(a, ctypes.c_float),
                              _p(bb, ctypes.c_float) if bb is not None else None, _p(mask, ctypes.c_int32), B, S,
                              int(acc32), _p(out, ctypes.c_float)))
        return out

    def embed(self, ids, acc32=False):
        ids = _i32(ids)
        B, S = ids.shape
        out = np.zeros((B * S, self.cfg.hidden), np.float32)
        _check(lib().or_embed(self.h, _p(ids, ctypes.c_int32), B, S, int(acc32), _p(out, ctypes.c_float)))
        return out

    def head(self, x, B, S):
        x = _f32(x)
        out = np.zeros((B, self.cfg.num_classes), np.float32)
        _check(lib().or_head(self.h, _p(x, ctypes.c_float), B, S, _p(out, ctypes.c_float)))
        return out

    def prepared_weight(self, layer: int, which: int):
        cfg = self.cfg
        D, F, H = cfg.heads[layer] * cfg.head_dim, cfg.ffn_dim[layer], cfg.hidden
        N, K = [(3 * D, H), (H, D), (F, H), (H, F)][which]
        q = np.zeros((N, K), np.int8)
        s = np.zeros(N, np.float32)
        w16 = np.zeros((N, K), np.float32)
        _check(lib().or_prepared_weight(self.h, layer, which, _p(q, ctypes.c_int8), _p(s, ctypes.c_float),
                                        _p(w16, ctypes.c_float)))
        return q, s, w16


# ---------------------------------------------------------------- primitives
def q8row(x):
    x = _f32(x)
    M, K = x.shape
    q = np.zeros((M, K), np.int8)
    s = np.zeros(M, np.float32)
    lib().or_q8row(_p(x, ctypes.c_float), M, K, _p(q, ctypes.c_int8), _p(s, ctypes.c_float))
    return q, s


def q8tensor(x):
    """Per-tensor u8 quantization with zero point (DESIGN R22): (q u8, scale, zp)."""
    x = _f32(x)
    M, K = x.shape if x.ndim == 2 else (1, x.size)
    q = np.zeros(x.shape, np.uint8)
    s = np.zeros(1, np.float32)
    z = np.zeros(1, np.int32)
    lib().or_q8tensor(_p(x, ctypes.c_float), M, K, _p(q, ctypes.c_uint8), _p(s, ctypes.c_float), _p(z, ctypes.c_int32))
    return q, float(s[0]), int(z[0])


def quant_weight(W):
    W = _f32(W)
    N, K = W.shape
    q = np.zeros((N, K), np.int8)
    s = np.zeros(N, np.float32)
    lib().or_quant_weight(_p(W, ctypes.c_float), N, K, _p(q, ctypes.c_int8), _p(s, ctypes.c_float))
    return q, s


def gemm_s8(A, W):
    A = np.ascontiguousarray(A, np.int8)
    W = np.ascontiguousarray(W, np.int8)
    M, K = A.shape
    N = W.shape[0]
    C = np.zeros((M, N), np.int32)
    lib().or_gemm_s8(_p(A, ctypes.c_int8), _p(W, ctypes.c_int8), M, N, K, _p(C, ctypes.c_int32))
    return C


def r16(x):
    x = _f32(x)
    y = np.zeros_like(x)
    lib().or_r16(_p(x, ctypes.c_float), x.size, _p(y, ctypes.c_float))
    return y


def act(x, kind):
    x = _f32(x)
    y = np.zeros(x.shape, np.float64)
    lib().or_act(_p(x, ctypes.c_float), x.size, int(kind), _p(y, ctypes.c_double))
    return y


def layer_norm64(x, g, b, eps):
    x = np.ascontiguousarray(x, np.float64)
    M, H = x.shape
    g, b = _f32(g), _f32(b)
    y = np.zeros_like(x)
    lib().or_layer_norm64(_p(x, ctypes.c_double), M, H, _p(g, ctypes.c_float), _p(b, ctypes.c_float),
                          float(eps), _p(y, ctypes.c_double))
    return y


def attention(qkv, mask, A, d, mode=MODE_EMU):
    qkv = _f32(qkv)
    mask = _i32(mask)
    B, S = mask.shape
    ctx = np.zeros((B * S, A * d), np.float32)
    lib().or_attention(_p(qkv, ctypes.c_float), _p(mask, ctypes.c_int32), B, S, A, d, mode, _p(ctx, ctypes.c_float))
    return ctx
