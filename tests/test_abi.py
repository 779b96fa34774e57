"""Host-side checks of the C ABI (no GPU needed): the library builds, loads and
exports every symbol include/fastformers.h declares; the header is valid C;
config validation happens before any device work."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2010_13382_b200 import fastformers as ffb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fastformers.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^FF_API\s+[\w\s\*]*?\b(ff_\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def built():
    import __graft_entry__
    __graft_entry__.build()
    return ffb.lib()


def test_header_is_valid_c():
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-x", "c", HEADER])


def test_every_declared_symbol_is_exported(built):
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.check_output(["nm", "-D", "--defined-only", ffb.LIB_PATH], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(ffb.EXPORTED) == syms


def test_abi_version(built):
    assert built.ff_abi_version() == 1


def test_library_targets_sm100a_only(built):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ffb.LIB_PATH], text=True)
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", ffb.LIB_PATH], text=True)
    assert "UTCHMMA" in sass or "UTCQMMA" in sass or "UTCIMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA loads
    assert "LDTM" in sass     # tcgen05.ld


def _cfg(**kw):
    heads = (ctypes.c_int32 * 2)(2, 1)
    ffn = (ctypes.c_int32 * 2)(256, 128)
    dt = (ctypes.c_int32 * 2)(1, 1)
    base = dict(abi_version=1, num_layers=2, hidden=128, head_dim=64, vocab_size=100, max_positions=64,
                num_classes=2, ln_eps=1e-12, act=0, heads=heads, ffn_dim=ffn, dtype=dt, max_tokens=128)
    base.update(kw)
    c = ffb.FFConfig(**{k: v for k, v in base.items()})
    return c, (heads, ffn, dt)


@pytest.mark.parametrize("field,value,status", [
    ("abi_version", 2, ffb.FF_E_INVALID),
    ("num_layers", 0, ffb.FF_E_INVALID),
    ("head_dim", 27, ffb.FF_E_INVALID),
    ("head_dim", 256, ffb.FF_E_INVALID),
    ("ln_eps", 0.0, ffb.FF_E_INVALID),
    ("act", 7, ffb.FF_E_INVALID),
    ("hidden", 100, ffb.FF_E_UNSUPPORTED),
    ("max_tokens", 0, ffb.FF_E_INVALID),
])
def test_config_validation_before_device(built, field, value, status):
    c, keep = _cfg(**{field: value})
    h = ctypes.c_void_p()
    assert built.ff_model_create(ctypes.byref(c), 0, ctypes.byref(h)) == status
    assert not h.value
    assert built.ff_last_error()


def test_bad_layer_arrays(built):
    heads = (ctypes.c_int32 * 2)(2, 0)
    c, keep = _cfg(heads=heads)
    h = ctypes.c_void_p()
    assert built.ff_model_create(ctypes.byref(c), 0, ctypes.byref(h)) == ffb.FF_E_INVALID


def test_null_model_calls_are_rejected(built):
    assert built.ff_encode(None, None, None, 1, 1, None, None) == ffb.FF_E_INVALID
    assert built.ff_check(None, None) == ffb.FF_E_INVALID
    assert built.ff_finalize(None, None) == ffb.FF_E_INVALID


def test_options_are_per_model(built):
    """Every option is per model (no process-wide state on the launch path):
    m = NULL is rejected, and the removed round-1 experiment ids (7, 10, 11,
    12) are unknown."""
    for opt in (ffb.FF_OPT_PDL, ffb.FF_OPT_PDL_RR, ffb.FF_OPT_FUSED_MASK, ffb.FF_OPT_GRAPHS, 7, 10, 11, 12, 999):
        assert built.ff_set_option(None, opt, 1) == ffb.FF_E_INVALID


def test_scorer_config_validation_before_device(built):
    c, keep = _cfg(num_classes=65)
    h = ctypes.c_void_p()
    assert built.ff_scorer_create(ctypes.byref(c), 0, ctypes.byref(h)) == ffb.FF_E_INVALID
    assert built.ff_scorer_last_error()
    assert built.ff_score_batch(None, None, None, None, 1, 1, None, None, None, None, None) == ffb.FF_E_INVALID
