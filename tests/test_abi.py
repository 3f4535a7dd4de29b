"""C-ABI library: loads without a GPU, exports every declared symbol, and
reports contract violations as EF_EINVAL before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1803_00430_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "echoforge_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t)\s+(ef_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_abi_version_and_error_channel():
    L = _lib.lib()
    assert L.ef_abi_version() == 1
    rc = L.ef_eval_sh_batch(None, 10, 7, None, None)
    assert rc == _lib.EF_EINVAL
    assert "order must be in [0, 4]" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_scene_create_validates_before_cuda():
    L = _lib.lib()
    h = ctypes.c_void_p()
    a = np.zeros((1, 4))
    rc = L.ef_scene_create(None, None, None, None, None, 0, _lib.host_ptr(a), _lib.host_ptr(a),
                           1, 9, ctypes.byref(h))
    assert rc == _lib.EF_EINVAL and "n_bands" in _lib.last_error()
    bad = np.full((1, 4), 1.5)
    rc = L.ef_scene_create(None, None, None, None, None, 0, _lib.host_ptr(bad), _lib.host_ptr(a),
                           1, 4, ctypes.byref(h))
    assert rc == _lib.EF_EINVAL and "[0, 1]" in _lib.last_error()
    v = np.zeros((1, 3))
    mi = np.array([3], np.int64)
    rc = L.ef_scene_create(_lib.host_ptr(v), _lib.host_ptr(v), _lib.host_ptr(v), _lib.host_ptr(v),
                           _lib.host_ptr(mi), 1, _lib.host_ptr(a), _lib.host_ptr(a), 1, 4,
                           ctypes.byref(h))
    assert rc == _lib.EF_EINVAL and "material index" in _lib.last_error()


def test_trace_config_layout_matches_header():
    # ef_trace_config: 4*i32, i64, 3*u32, i32, f64, 3*f64, f64, f32, i32
    assert ctypes.sizeof(_lib.TraceConfig) == 128
    assert _lib.TraceConfig.er_capacity.offset == 104
    assert _lib.ER_DTYPE.itemsize == 72
    assert _lib.TraceConfig.n_rays.offset == 16
    assert _lib.TraceConfig.bin_len.offset == 40
    assert _lib.TraceConfig.e0.offset == 80
    assert ctypes.sizeof(_lib.AnalysisConfig) == 32


def test_trace_rejects_bad_config_without_gpu():
    L = _lib.lib()
    cfg = _lib.TraceConfig()
    cfg.n_sources = 0
    assert L.ef_trace(ctypes.c_void_p(1), cfg, *([None] * 10)) == _lib.EF_EINVAL
    assert "source" in _lib.last_error()


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (cross-compiled here)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
