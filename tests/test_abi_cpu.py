"""CPU-side checks of the C ABI (-m "not gpu"): the library builds for sm_100a, loads,
exports every symbol include/hp.h declares, validates arguments, and its defaults
transcribe the paper's tables identically to the oracle's independent transcription."""
import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2005_07068_b200 as hp
from paper_2005_07068_b200 import build as hpbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "hp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\*?(hp_\w+)\s*\(", src, re.M)))


def test_library_builds_for_sm100a():
    lib = hpbuild.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


DEBUG_ONLY = {"hp_shard_loopback"}  # declared in hp.h for -DHP_LOOPBACK_TEST builds only


def test_every_header_symbol_is_exported():
    syms = _header_symbols()
    assert len(syms) >= 18
    L = hp.lib()
    for s in syms:
        assert hasattr(L, s) == (s not in DEBUG_ONLY), s
    assert sorted(hp.exported_symbols()) == sorted(set(syms) - DEBUG_ONLY)


def test_loopback_debug_build_exports_the_same_abi_plus_the_loopback_hook():
    path = hpbuild.build_loopback()
    L = hp.lib(path)
    for s in _header_symbols():
        assert hasattr(L, s), s


def test_sass_has_tma_loads():
    lib = hpbuild.build()
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # cp.async.bulk.tensor in the fused kernel


def test_defaults_match_oracle_transcription():
    lo, hi = hp.bounds()
    olo, ohi = O.bounds()
    assert np.array_equal(lo, olo) and np.array_equal(hi, ohi)
    d, od = hp.default_dims(), O.default_dims()
    assert [list(r) for r in d.base] == [list(r) for r in od.base]
    assert [list(r) for r in d.seg_len] == [list(r) for r in od.seg_len]
    assert [list(r) for r in d.radius] == [list(r) for r in od.radius]
    assert (d.palm_half_w, d.palm_half_t, d.palm_len, d.palm_cap_half_len) == (
        od.palm_half_w, od.palm_half_t, od.palm_len, od.palm_cap_half_len)
    c, oc = hp.default_cost(), O.default_cost()
    assert (c.d_m, c.d_M, c.lam, c.lambda_k, c.depth_scale) == (oc.d_m, oc.d_M, oc.lam,
                                                                 oc.lambda_k, oc.depth_scale)
    for w, h in ((160, 120), (320, 240), (640, 480)):
        i, oi = hp.default_intrinsics(w, h), O.camera(w, h)
        assert (i.fx, i.fy, i.cx, i.cy, i.z_near_mm, i.z_far_mm) == (oi.fx, oi.fy, oi.cx, oi.cy,
                                                                     oi.z_near, oi.z_far)


def test_create_validates_and_reports_no_device():
    L = hp.lib()
    h = C.c_void_p()
    bad = hp.default_intrinsics(160, 120)
    bad.fx = 0
    assert L.hp_create(C.byref(bad), None, None, 16, -1, C.byref(h)) == hp.hp.HP_ERR_INVALID_ARG
    assert b"fx" in L.hp_last_error(None)
    bad = hp.default_intrinsics(160, 120)
    bad.z_near_mm = 3000
    assert L.hp_create(C.byref(bad), None, None, 16, -1, C.byref(h)) == hp.hp.HP_ERR_INVALID_ARG
    ok = hp.default_intrinsics(160, 120)
    assert L.hp_create(C.byref(ok), None, None, 0, -1, C.byref(h)) == hp.hp.HP_ERR_INVALID_ARG
    huge = hp.default_intrinsics(8192, 4096)  # the ray table would not fit shared memory
    assert L.hp_create(C.byref(huge), None, None, 16, -1, C.byref(h)) == hp.hp.HP_ERR_INVALID_ARG
    assert b"too large" in L.hp_last_error(None)
    import torch

    if not torch.cuda.is_available():
        st = L.hp_create(C.byref(ok), None, None, 16, -1, C.byref(h))
        assert st == hp.hp.HP_ERR_NO_DEVICE
        with pytest.raises(hp.HPError):
            hp.Context(160, 120)


def test_null_ctx_calls_fail_cleanly():
    L = hp.lib()
    assert L.hp_eval_costs(None, None, 4, None, None) == hp.hp.HP_ERR_INVALID_ARG
    assert L.hp_pso_fit(None, None, None, None, None, None, None) == hp.hp.HP_ERR_INVALID_ARG
    assert L.hp_last_launch_count(None) == -1
    L.hp_destroy(None)


def test_binding_refuses_missing_library(tmp_path, monkeypatch):
    """No CPU fallback: without libhp.so the binding raises."""
    import importlib

    mod = importlib.import_module("paper_2005_07068_b200.hp")
    monkeypatch.setattr(mod, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(mod, "_libs", {})
    with pytest.raises(ImportError):
        mod.lib()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2005_07068_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).lower().replace(
                    "no oracle", ""), f


def test_constriction_host_formula_matches():
    # the library computes w on the host with the same closed form
    psi = 2.8 + 1.3
    w = 2.0 / abs(2.0 - psi - math.sqrt(psi * psi - 4.0 * psi))
    assert abs(w - O.constriction(2.8, 1.3)) == 0.0
