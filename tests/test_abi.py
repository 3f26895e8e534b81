"""CPU-side checks of the C ABI: the library loads and exports every symbol that
include/feb200.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "feb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fe_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("fe_create_mesh_geometry", "fe_eval_element_matrices", "fe_eval_residual",
              "fe_assemble_vector", "fe_destroy_mesh", "fe_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_2107_04121_b200 as fe
    if not os.path.exists(fe.LIB_PATH):
        from paper_2107_04121_b200 import build
        build.build()
    lib = ctypes.CDLL(fe.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(fe.ABI_SYMBOLS)


def test_error_state_without_gpu():
    """Argument validation runs on the host: NULL handle -> FE_ERR_INVALID_ARG."""
    import paper_2107_04121_b200 as fe
    lib = fe.lib()
    st = lib.fe_eval_residual(None, 0, 0, None, None, 0, 0, None, None, None)
    assert st == fe.FE_ERR_INVALID_ARG
    assert b"NULL" in lib.fe_last_error()
    info = fe.fe_info()
    assert lib.fe_mesh_info(None, ctypes.byref(info)) == fe.FE_ERR_INVALID_ARG


def test_product_does_not_import_oracle():
    """The product package never references oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2107_04121_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "fe_oracle" not in txt, f


def test_new_entry_points_validate_on_host():
    """N3 / N4 entry points reject bad arguments before touching the device."""
    import paper_2107_04121_b200 as fe
    lib = fe.lib()
    INV = fe.FE_ERR_INVALID_ARG
    assert lib.fe_eval_stress(None, None, None, 0, 0, None, None) == INV
    out = ctypes.c_void_p()
    assert lib.fe_create_field(None, 1, 8, None, None, ctypes.byref(out)) == INV
    assert lib.fe_create_field(None, 1, 8, None, None, None) == INV
    assert lib.fe_destroy_field(None) == fe.FE_OK
    assert lib.fe_eval_coupling_matrices(None, None, 0, 0, 0, None, None) == INV
    assert lib.fe_eval_coupling_residual(None, None, 0, None, 0, 0, None, None, None) == INV
    assert lib.fe_eval_coupling_scalar(None, None, None, None, 0, 0, None, None) == INV
    offs = (ctypes.c_int64 * 3)()
    assert lib.fe_group_cells(None, 5, 2, None, offs, None) == INV      # NULL kind
    assert lib.fe_group_cells(None, 0, 0, None, offs, None) == INV      # no kinds
    assert lib.fe_group_cells(None, 0, 2, None, offs, None) == fe.FE_OK  # empty: offsets zero
    assert list(offs) == [0, 0, 0]
    assert lib.fe_gather_rows_f64(None, None, 3, None, 4, None, None) == INV
    assert lib.fe_gather_rows_i32(None, None, 3, None, -1, None, None) == INV
    assert lib.fe_gather_rows_i32(None, None, 3, None, 0, None, None) == fe.FE_OK
