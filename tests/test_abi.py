"""The C-ABI library loads and exports every entry point include/*.h declares (CPU, no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

from conftest import ROOT

HEADERS = sorted((ROOT / "include").glob("*.h"))


def declared():
    names = []
    for h in HEADERS:
        text = h.read_text()
        names += re.findall(r"DS_API\s+[\w\s\*]+?\b(ds_\w+)\s*\(", text)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2411_02820_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2411_02820_b200 import _build
        _build.build()
    return _lib


def test_headers_declare_entry_points():
    names = declared()
    for must in ("ds_kv_ingest", "ds_partial_prefill", "ds_full_prefill", "ds_recompute_group", "ds_anchor",
                 "ds_workspace_size", "ds_last_error", "ds_abi_version"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    h = ctypes.CDLL(str(lib.LIB_PATH))
    missing = [n for n in declared() if not hasattr(h, n)]
    assert not missing, missing
    # the Python binding covers the same set
    assert sorted(lib.EXPORTED_SYMBOLS) == declared()


def test_host_only_entry_points(lib):
    L = lib.lib()
    assert L.ds_abi_version() == lib.ABI_VERSION == 2
    # anchor-shape override: returns the previous value, rejects unknown shapes
    prev = L.ds_set_anchor_shape(2)
    assert prev in (0, 1, 2)
    assert L.ds_set_anchor_shape(prev) == 2
    assert L.ds_set_anchor_shape(7) == -1
    with lib.anchor_shape("persistent"):
        assert L.ds_set_anchor_shape(1) == 1
    assert L.ds_set_anchor_shape(prev) == prev
    assert L.ds_fused_fallbacks() == 0
    dims = lib.Dims(32, 4096, 32, 8, 128, 14336, 128256, 8192)
    assert L.ds_workspace_size(ctypes.byref(dims), 8192) > 8192 * 4096 * 4
    assert L.ds_workspace_size(None, 8) == 0
    # argument validation happens before any device work and maps to ValueError
    rc = L.ds_kv_ingest(None, None, None, 0, 0, 8, 128, None, None)
    assert rc == lib.DS_ERR_INVALID
    with pytest.raises(ValueError):
        lib.check(rc)
    assert b"ingest" in L.ds_last_error()
    # profiling aids: no events recorded -> empty trace; bad arguments -> -1
    assert L.ds_trace_begin() == 0
    assert L.ds_trace_end(None, None, 0) == 0
    assert L.ds_anchor_placement(None, 8, None, None, 0) == -1
    assert b"placement" in L.ds_last_error()
    assert L.ds_anchor_timeline(ctypes.byref(dims), 0, None, None, 0) == -1


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    from paper_2411_02820_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "absent.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="not built"):
        _lib.lib()


def test_batch_entry_points_validate_on_host(lib):
    """ds_partial_prefill_batch validates every request (reference order,
    requests in order) before any device work and names the bad request."""
    L = lib.lib()
    C = ctypes
    dims = lib.Dims(4, 256, 4, 1, 64, 1024, 4096, 1024, 0)
    one = L.ds_workspace_size(C.byref(dims), 300)
    assert L.ds_workspace_size_batch(C.byref(dims), 300, 4) > one
    assert L.ds_workspace_size_batch(C.byref(dims), 300, 9) == 0
    assert L.ds_workspace_size_batch(C.byref(dims), 300, 0) == 0
    layers = (lib.LayerWeights * 4)()
    model = lib.Model(dims, None, None, None, None, None, C.cast(layers, C.POINTER(lib.LayerWeights)))
    import numpy as np
    toks = [np.arange(100, dtype=np.int64), np.arange(120, dtype=np.int64) % 4096]
    bad = toks[1].copy()
    bad[7] = 4096
    groups = (C.c_int32 * 2)(2, 3)
    fake = C.c_void_p(256)  # never dereferenced: validation fails first
    out = (lib.KvCache * 2)(*[lib.KvCache(fake, fake, 0, 64 * 64, 64 * 64, None, 4, 128, None, None)] * 2)
    nt = (C.c_int32 * 2)(100, 120)
    badreq, ml, mk = C.c_int32(-9), C.c_int32(-1), C.c_int32(0)

    def call(t, skv, g=groups):
        th = (C.c_void_p * 2)(*[x.ctypes.data for x in t])
        return L.ds_partial_prefill_batch(C.byref(model), 2, th, None, nt, g, 1, skv, None, None, out, fake,
                                          fake, None, 0, None, None, C.byref(badreq), C.byref(ml), C.byref(mk))

    # every layer recomputed (no export needed): request 1's ids are checked after request 0's
    rc = call([toks[0], bad], None, (C.c_int32 * 2)(0, 3))
    assert rc == lib.DS_ERR_INVALID and badreq.value == 1 and b"vocabulary" in L.ds_last_error()
    # ... and with everything valid, the missing workspace is the error (still no device work)
    rc = call(toks, None, (C.c_int32 * 2)(0, 3))
    assert rc == lib.DS_ERR_INVALID and badreq.value == -1 and b"workspace" in L.ds_last_error()
    # valid tokens, no sender export: KV miss at the first reused layer of request 0
    rc = call(toks, None)
    assert rc == lib.DS_ERR_CACHE_MISS and badreq.value == 0 and (ml.value, mk.value) == (0, 1)
    from paper_2411_02820_b200.errors import CacheMissError
    with pytest.raises(CacheMissError):
        lib.check(rc, ml.value, mk.value)
    # exports present, E missing for request 0's transition layer 2
    skv = (lib.KvCache * 2)(*[lib.KvCache(fake, fake, 0, 128 * 64, 64 * 64, None, 4, 128, None, None)] * 2)
    rc = call(toks, skv)
    assert rc == lib.DS_ERR_CACHE_MISS and badreq.value == 0 and (ml.value, mk.value) == (2, 2)
    assert L.ds_decode_greedy_batch(C.byref(model), 0, None, None, None, 1, None, None, 0, None) == lib.DS_ERR_INVALID
    assert L.ds_anchor_batch(C.byref(model), 9, None, None, None, None, None, None, 0, None) == lib.DS_ERR_INVALID
