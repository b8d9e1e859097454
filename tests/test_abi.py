"""CPU checks of the C ABI: the library builds for sm_100a, loads without a GPU, and exports
every entry point declared in include/mmot.h (no compute calls)."""
import ctypes
import os
import re

import pytest

import paper_2405_19246_b200 as mm
from paper_2405_19246_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mmot.h")).read()
    return sorted(set(re.findall(r"MMOT_API\s+[\w\s\*]+?\b(mmot_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return mm.load_library()


def test_header_declares_entry_points():
    names = _declared()
    for n in ("mmot_create", "mmot_marginal", "mmot_sinkhorn", "mmot_cost", "mmot_destroy",
              "mmot_strerror", "mmot_init_uniform", "mmot_sinkhorn_host", "mmot_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    exported = set(mm.exported_symbols())
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    # no internal symbols leak (visibility hidden)
    assert all(s.startswith("mmot_") for s in exported)


def test_host_only_calls(lib):
    assert lib.mmot_version() == (0 << 16) | 1
    assert lib.mmot_strerror(0) == b"ok"
    assert b"overflow" in lib.mmot_strerror(6) or b"range" in lib.mmot_strerror(6)


def test_argument_errors_before_any_launch(lib):
    """mmot_create validates on the host (EINVAL / EUNSUPPORTED) without touching the device."""
    ctx = ctypes.c_void_p()
    g = mm._Grid(0.0, 1.0)
    assert lib.mmot_create(1, 10, 0.1, g, 0, None, None, ctypes.byref(ctx)) == 1       # l < 2
    assert lib.mmot_create(3, 0, 0.1, g, 0, None, None, ctypes.byref(ctx)) == 1        # N < 1
    assert lib.mmot_create(3, 10, -1.0, g, 0, None, None, ctypes.byref(ctx)) == 1      # eta <= 0
    assert lib.mmot_create(3, 10, float("nan"), g, 0, None, None, ctypes.byref(ctx)) == 1
    assert lib.mmot_create(3, 10, 0.1, mm._Grid(1.0, 0.0), 0, None, None, ctypes.byref(ctx)) == 1
    assert lib.mmot_create(9, 10, 0.1, g, 0, None, None, ctypes.byref(ctx)) == 1       # l > MMOT_MAX_L = 8
    assert lib.mmot_create(7, 10, 0.1, g, 1, None, None, ctypes.byref(ctx)) == 10      # l = 7, 8: MMOT_F64 only
    assert ctx.value is None
    assert lib.mmot_marginal(None, 0, None, None) == 1
    assert lib.mmot_sinkhorn(None, None, 1, 0.0, None, None) == 1


def test_batched_and_sharded_argument_errors(lib):
    """mmot_create_batched / mmot_create_sharded validate on the host before any device work."""
    ctx = ctypes.c_void_p()
    g = mm._Grid(0.0, 1.0)
    etas = (ctypes.c_double * 2)(0.1, -1.0)
    assert lib.mmot_create_batched(4, 100, 2, etas, g, 0, None, None, ctypes.byref(ctx)) == 1   # eta <= 0
    etas_ok = (ctypes.c_double * 2)(0.1, 0.2)
    assert lib.mmot_create_batched(4, 0, 2, etas_ok, g, 0, None, None, ctypes.byref(ctx)) == 1  # N < 1
    assert lib.mmot_create_batched(6, 100, 2, etas_ok, g, 1, None, None, ctypes.byref(ctx)) == 10  # l > 5: MMOT_F64 only
    uid = ctypes.create_string_buffer(128)
    assert lib.mmot_create_sharded(4, 100, 0.1, g, 0, uid, 2, 2, None, None, ctypes.byref(ctx)) == 1  # rank >= world
    assert lib.mmot_create_sharded(4, 100, 0.1, g, 0, None, 0, 1, None, None, ctypes.byref(ctx)) == 1  # no id
    assert ctx.value is None


def test_points_argument_errors(lib):
    """mmot_create_points validates the grid points on the host before any device work."""
    ctx = ctypes.c_void_p()
    bad = (ctypes.c_double * 4)(0.0, 0.5, 0.5, 1.0)      # not strictly increasing
    assert lib.mmot_create_points(3, 4, 0.1, bad, 0, None, None, ctypes.byref(ctx)) == 1
    nan = (ctypes.c_double * 3)(0.0, float("nan"), 1.0)
    assert lib.mmot_create_points(3, 3, 0.1, nan, 0, None, None, ctypes.byref(ctx)) == 1
    assert lib.mmot_create_points(3, 3, 0.1, None, 0, None, None, ctypes.byref(ctx)) == 1
    ok = (ctypes.c_double * 3)(0.0, 0.2, 1.0)
    assert lib.mmot_create_points(3, 3, -1.0, ok, 0, None, None, ctypes.byref(ctx)) == 1   # eta <= 0


def test_virtual_group_argument_errors(lib):
    """mmot_vgroup_create / mmot_create_sharded_virtual validate on the host (no device work)."""
    g = ctypes.c_void_p()
    assert lib.mmot_vgroup_create(0, ctypes.byref(g)) == 1
    assert lib.mmot_vgroup_create(17, ctypes.byref(g)) == 1
    assert g.value is None
    lib.mmot_vgroup_destroy(None)
    ctx = ctypes.c_void_p()
    assert lib.mmot_create_sharded_virtual(4, 100, 0.1, mm._Grid(0.0, 1.0), 0, None, 0, None, None,
                                           ctypes.byref(ctx)) == 1
    assert ctx.value is None
    assert lib.mmot_fallback_count(None) == 0
    assert lib.mmot_strerror(11) == b"single-walk precision guard tripped"
