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
    assert lib.fe_destroy_field(None, None) == fe.FE_OK
    assert lib.fe_destroy_mesh(None, None) == fe.FE_OK
    assert lib.fe_destroy_csr(None, None) == fe.FE_OK
    assert lib.fe_eval_stress_integral(None, None, None, 0, 0, None, None) == INV
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


def test_options_set_get_and_validate():
    """fe_set_option / fe_get_option (host only): values stick, out-of-range values and unknown
    options are rejected, the options context manager restores the previous values."""
    import paper_2107_04121_b200 as fe
    lib = fe.lib()
    before = fe.get_options()
    with fe.options(matrix_impl="dense", max_ctas=3, csr_impl="gather", residual_impl="sf"):
        assert fe.get_options() == {"matrix_impl": 2, "residual_impl": 1, "csr_impl": 1,
                                    "max_ctas": 3}
    assert fe.get_options() == before
    INV = fe.FE_ERR_INVALID_ARG
    assert lib.fe_set_option(fe.OPT_MATRIX_IMPL, 3) == INV
    assert lib.fe_set_option(fe.OPT_MAX_CTAS, -1) == INV
    assert lib.fe_set_option(99, 0) == INV
    assert lib.fe_get_option(0, None) == INV
    assert fe.get_options() == before


def test_options_read_from_environment_once():
    """Defaults come from FEB200_* at load (a fresh process), and the binding says so."""
    import subprocess
    import sys
    env = dict(os.environ, FEB200_MATRIX_IMPL="dense", FEB200_MAX_CTAS="7",
               FEB200_RESIDUAL_IMPL="sf", FEB200_CSR_IMPL="gather")
    code = ("import paper_2107_04121_b200 as fe, os; print(fe.get_options()); "
            "os.environ['FEB200_MATRIX_IMPL'] = 'sf1'; print(fe.get_options()['matrix_impl'])")
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert eval(lines[0]) == {"matrix_impl": 2, "residual_impl": 1, "csr_impl": 1, "max_ctas": 7}
    assert lines[1] == "2"          # no getenv after load
    assert "implementation options from the environment" in r.stderr


def test_every_working_entry_point_has_an_nvtx_range():
    """an NVTX range around every ABI call that queues or performs work."""
    pure = {"fe_last_error", "fe_last_error_element", "fe_launch_count", "fe_set_option",
            "fe_get_option", "fe_mesh_info", "fe_csr_info", "fe_csr_arrays"}
    csrc = os.path.join(ROOT, "paper_2107_04121_b200", "csrc")
    src = "".join(open(os.path.join(csrc, f)).read() for f in os.listdir(csrc)
                  if f.endswith((".cu", ".cpp")))
    for s in declared_symbols():
        if s in pure:
            continue
        assert f'FE_NVTX_RANGE("{s}")' in src, s
