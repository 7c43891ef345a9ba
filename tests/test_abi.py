"""CPU checks of the C ABI: the library builds for sm_100a, loads, exports
every symbol include/dynsplit.h declares, and its host-side queries and
argument validation work without a GPU (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dynsplit.h")


@pytest.fixture(scope="module")
def D():
    from paper_2602_03184_b200 import build, dynsplit
    build.build()
    dynsplit.lib()
    return dynsplit


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dynsplit_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(D):
    syms = declared_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", D.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dynsplit_[a-z0-9_]+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(D.SIGNATURES) == set(syms)          # the binding covers the whole ABI


def test_library_is_sm100a(D):
    out = subprocess.run(["cuobjdump", "--list-elf", D.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_config_and_bounds(D):
    c = D.default_config()
    assert (c.W, c.R, c.alpha_pen, c.C, c.delta, c.lambda_num, c.lambda_den, c.page_size, c.digest_mode) == \
        (8, 128, 1.0, 32, 14, 1, 2, 16, 0)
    # every non-final chunk has >= C - Delta tokens
    assert D.max_blocks(131072, c) == 131072 // 18 + 1 == 7282
    assert D.max_pages(131072, c) == 7282 + 8192
    assert D.max_selected(4096, 131072, c) == 4095 // 18 + 2
    assert D.lib().dynsplit_version().startswith(b"dynsplit-b200")


def test_host_validation_without_gpu(D):
    L = D.lib()
    c = D.default_config()
    bad = D.make_shape(1, 128, 6, 4)                      # Hq % Hkv != 0
    assert L.dynsplit_score_blocks(ctypes.byref(bad), ctypes.byref(c), None, None, None, None, None) == 2
    empty = D.make_shape(1, 0, 8, 8)
    assert L.dynsplit_segment(ctypes.byref(empty), ctypes.byref(c), None, None, 1, None, None, None,
                              None, 0, None) == 3
    ok = D.make_shape(1, 128, 8, 8)
    assert L.dynsplit_select(ctypes.byref(ok), ctypes.byref(c), 16, None, None, None, None, None, None,
                             None, None, None, None, None, None, 0, None) == 1
    c2 = D.default_config(delta=32)                       # Delta >= C
    assert L.dynsplit_workspace_bytes(D.OP_SELECT, ctypes.byref(ok), ctypes.byref(c2), 16) == 0
    assert D.workspace_bytes(D.OP_DECODE_ATTN, ok, c) > 0
    assert D.worklist_bytes(ok, c, 64) > 0
    assert L.dynsplit_status_string(4) == b"workspace too small"
    d64 = D.make_shape(1, 128, 8, 8, d=64)
    assert L.dynsplit_score_blocks(ctypes.byref(d64), ctypes.byref(c), None, None, None, None, None) == 2


def test_product_path_has_no_oracle_dependency():
    # The product package never imports the oracle (test infrastructure only).
    pkg = os.path.join(ROOT, "paper_2602_03184_b200")
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle|#include\s+.*oracle)", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not pat.search(src), f


def test_append_argument_validation(D):
    """NEXT-1 entry points reject bad lengths / configs before any launch."""
    import ctypes as C
    sh = D.make_shape(1, 1000, 8, 8, 128)
    cfg = D.default_config()
    lib = D.lib()
    p = C.c_void_p(16)  # never dereferenced: validation fails first
    bad = [(5, 3), (-1, 3), (0, 0), (10, 1001)]
    for lp, l in bad:
        st = lib.dynsplit_append_plan(C.byref(sh), C.byref(cfg), lp, l, p, p, 13, p, p, p, p, p, p, p, p,
                                      1 << 20, None)
        assert st != 0, (lp, l)
        st = lib.dynsplit_append_kv(C.byref(sh), C.byref(cfg), lp, l, p, p, p, p, p, p, p, p, p, None)
        assert st != 0, (lp, l)
    wide = D.default_config(C=200, delta=100)
    st = lib.dynsplit_append_plan(C.byref(sh), C.byref(wide), 0, 10, p, p, 13, p, p, p, p, p, p, p, p,
                                  1 << 20, None)
    assert st == 5  # DYNSPLIT_ERR_UNSUPPORTED (C + Delta above the staging bound)
    assert D.workspace_bytes(D.OP_APPEND, sh, cfg) > 0


def test_offload_abi_without_gpu(D):
    """NEXT-3 entry points: the cache-slot bound (per query head at most
    ceil(budget / P) + max_selected pages, times g, capped at max_pages), the
    workspace sizes, and host-side rejection of bad caches before any launch."""
    import ctypes as C
    lib = D.lib()
    c = D.default_config()
    sh = D.make_shape(1, 32768, 32, 8)
    g = 4
    per_head = (2048 + 15) // 16 + D.max_selected(2048, 32768, c)
    assert D.cache_slots(sh, c, 2048) == min(g * per_head, D.max_pages(32768, c))
    tiny = D.make_shape(1, 100, 32, 8)
    assert D.cache_slots(tiny, c, 4096) == D.max_pages(100, c)       # capped
    assert D.cache_slots(sh, c, 0) == 0                               # budget < 1
    assert D.workspace_bytes(D.OP_REUSE, sh, c) > 0
    assert D.workspace_bytes(D.OP_DECODE_OFFLOAD, sh, c, 2048) > D.workspace_bytes(D.OP_DECODE_ATTN, sh, c)
    p = C.c_void_p(16)  # never dereferenced: validation fails first
    ws_ok = D.workspace_bytes(D.OP_REUSE, sh, c)
    # null cache, zero / oversize slot counts, missing outputs -> INVALID_ARGUMENT (1)
    assert lib.dynsplit_reuse_plan(C.byref(sh), C.byref(c), p, 1, 1, None, p, ws_ok, None) == 1
    for n_slots in (0, D.max_pages(32768, c) + 1):
        k = D.KVCache(n_slots, p, p, p, p, p, p, p, p)
        assert lib.dynsplit_reuse_plan(C.byref(sh), C.byref(c), p, 1, 1, C.byref(k), p, ws_ok, None) == 1
    k = D.KVCache(64, p, p, p, None, p, p, p, p)
    assert lib.dynsplit_reuse_plan(C.byref(sh), C.byref(c), p, 1, 1, C.byref(k), p, ws_ok, None) == 1
    k = D.KVCache(64, p, p, p, p, p, p, p, p)
    assert lib.dynsplit_reuse_plan(C.byref(sh), C.byref(c), p, 1, 1, C.byref(k), p, ws_ok - 1, None) == 4
    # dense fetch needs n_slots == max_pages (DIMENSION_MISMATCH, 2)
    assert lib.dynsplit_fetch_pages(C.byref(sh), C.byref(c), p, p, p, p, 1, C.byref(k), None) == 2
