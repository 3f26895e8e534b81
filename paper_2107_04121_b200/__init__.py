"""paper_2107_04121_b200 -- batched FE weak-form evaluation on B200 (sm_100a).

Thin ctypes binding of libfeb200.so (C ABI: include/feb200.h).  The functions
below carry the ABI's names and do argument marshalling only: every step of
the hot path (geometry, gradients, contractions, gather, scatter-add) runs in
the library's CUDA kernels.  PyTorch provides device memory and streams.

There is NO CPU fallback: if libfeb200.so is missing or fails to load, the
first call raises ImportError.  Build it with ``python -m paper_2107_04121_b200.build`` (or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FEB200_LIB_PATH selects another in-tree build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("FEB200_LIB_PATH", os.path.join(_HERE, "libfeb200.so"))

FE_OK, FE_ERR_INVALID_ARG, FE_ERR_UNSUPPORTED, FE_ERR_DEGENERATE, FE_ERR_CUDA, FE_ERR_OOM = range(6)
DIFFUSION, MASS, VECTOR_MASS, MASS_DIFFUSION, ELASTICITY, CONVECTIVE, WEIGHTED_DOT, DIVERGENCE = range(8)
F64, F32 = 0, 1
MAT_PER_QP, MAT_PER_ELEM, MAT_FULL_D = 0, 1, 2
NCOMP = {DIFFUSION: 1, MASS: 1, VECTOR_MASS: 3, MASS_DIFFUSION: 1, ELASTICITY: 3, CONVECTIVE: 3,
         WEIGHTED_DOT: 3, DIVERGENCE: 3}
_STATUS = {1: "FE_ERR_INVALID_ARG", 2: "FE_ERR_UNSUPPORTED", 3: "FE_ERR_DEGENERATE",
           4: "FE_ERR_CUDA", 5: "FE_ERR_OOM"}


class FEError(RuntimeError):
    def __init__(self, status: int, msg: str, element: int = -1):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.element = element


class fe_material(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("a", ctypes.c_void_p), ("b", ctypes.c_void_p)]


class fe_peer_window(ctypes.Structure):
    _fields_ = [("node_begin", ctypes.c_int64), ("node_end", ctypes.c_int64),
                ("dst", ctypes.c_void_p), ("dst_node_offset", ctypes.c_int64)]


class fe_info(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("q1d", ctypes.c_int32), ("nb", ctypes.c_int32),
                ("nq", ctypes.c_int32), ("n_vertices", ctypes.c_int64),
                ("n_elems", ctypes.c_int64), ("n_nodes", ctypes.c_int64),
                ("min_det_j", ctypes.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2107_04121_b200.build` "
                          "(no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    env = {k: v for k, v in os.environ.items() if k in (
        "FEB200_MATRIX_IMPL", "FEB200_RESIDUAL_IMPL", "FEB200_CSR_IMPL", "FEB200_MAX_CTAS")}
    if env:  # non-default kernels selected from the environment: say so (measured baselines)
        import sys
        print(f"paper_2107_04121_b200: implementation options from the environment: {env}",
              file=sys.stderr)
    P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    lib.fe_create_mesh_geometry.argtypes = [i64, P, i64, P, i32, i32, i64, P, P,
                                            ctypes.POINTER(P)]
    lib.fe_destroy_mesh.argtypes = [P, P]
    lib.fe_mesh_info.argtypes = [P, ctypes.POINTER(fe_info)]
    lib.fe_eval_element_matrices.argtypes = [P, i32, i32, ctypes.POINTER(fe_material), P, i64,
                                             i64, P, P]
    lib.fe_eval_residual.argtypes = [P, i32, i32, ctypes.POINTER(fe_material), P, i64, i64, P,
                                     P, P]
    lib.fe_assemble_vector.argtypes = [P, i32, i32, i64, i64, P, P, P]
    lib.fe_eval_scalar.argtypes = [P, i32, i32, ctypes.POINTER(fe_material), P, i64, i64, P, P]
    lib.fe_eval_matrix_residual.argtypes = [P, i32, i32, ctypes.POINTER(fe_material), P, i64,
                                            i64, P, P, P, P]
    lib.fe_eval_stress.argtypes = [P, ctypes.POINTER(fe_material), P, i64, i64, P, P]
    lib.fe_create_field.argtypes = [P, i32, i64, P, P, ctypes.POINTER(P)]
    lib.fe_destroy_field.argtypes = [P, P]
    lib.fe_eval_coupling_matrices.argtypes = [P, P, i32, i64, i64, P, P]
    lib.fe_eval_coupling_residual.argtypes = [P, P, i32, P, i64, i64, P, P, P]
    lib.fe_eval_coupling_scalar.argtypes = [P, P, P, P, i64, i64, P, P]
    lib.fe_group_cells.argtypes = [P, i64, i32, P, P, P]
    lib.fe_gather_rows_i32.argtypes = [P, P, i32, P, i64, P, P]
    lib.fe_gather_rows_f64.argtypes = [P, P, i32, P, i64, P, P]
    lib.fe_eval_residual_peer.argtypes = [P, i32, ctypes.POINTER(fe_material), P, i64, i64, P, P,
                                          ctypes.POINTER(fe_peer_window), i32, P]
    lib.fe_ipc_alloc.argtypes = [i64, ctypes.POINTER(P), ctypes.c_char_p]
    lib.fe_ipc_free.argtypes = [P]
    lib.fe_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(P)]
    lib.fe_ipc_close.argtypes = [P]
    lib.fe_create_csr.argtypes = [P, i32, P, ctypes.POINTER(P)]
    lib.fe_csr_info.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.fe_csr_arrays.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P)]
    lib.fe_csr_copy_arrays.argtypes = [P, P, P, P]
    lib.fe_assemble_matrix.argtypes = [P, P, i64, i64, P, P]
    lib.fe_destroy_csr.argtypes = [P, P]
    lib.fe_set_option.argtypes = [i32, i64]
    lib.fe_get_option.argtypes = [i32, ctypes.POINTER(i64)]
    lib.fe_eval_stress_integral.argtypes = [P, ctypes.POINTER(fe_material), P, i64, i64, P, P]
    lib.fe_geometry.argtypes = [P, P, P, P]
    lib.fe_last_error.restype = ctypes.c_char_p
    lib.fe_last_error_element.restype = i64
    lib.fe_launch_count.restype = i64
    for f in ("fe_create_mesh_geometry", "fe_destroy_mesh", "fe_mesh_info",
              "fe_eval_element_matrices", "fe_eval_residual", "fe_assemble_vector",
              "fe_geometry", "fe_eval_scalar", "fe_eval_matrix_residual", "fe_eval_stress", "fe_create_field", "fe_destroy_field",
              "fe_eval_coupling_matrices", "fe_eval_coupling_residual", "fe_eval_coupling_scalar",
              "fe_group_cells", "fe_gather_rows_i32", "fe_gather_rows_f64",
              "fe_eval_residual_peer", "fe_ipc_alloc", "fe_ipc_free", "fe_ipc_open", "fe_ipc_close",
              "fe_create_csr", "fe_csr_info", "fe_csr_arrays",
              "fe_csr_copy_arrays",
              "fe_assemble_matrix", "fe_destroy_csr", "fe_set_option", "fe_get_option",
              "fe_eval_stress_integral"):
        getattr(lib, f).restype = ctypes.c_int
    return lib


_lib_handle = None


class _LazyLib:
    """Loads libfeb200.so on first use and raises loudly if it is missing."""

    def __getattr__(self, name):
        global _lib_handle
        if _lib_handle is None:
            _lib_handle = _load()
        return getattr(_lib_handle, name)


_lib = _LazyLib()
ABI_SYMBOLS = ("fe_create_mesh_geometry", "fe_destroy_mesh", "fe_mesh_info",
               "fe_eval_element_matrices", "fe_eval_residual", "fe_assemble_vector", "fe_eval_scalar",
               "fe_eval_matrix_residual", "fe_eval_stress",
               "fe_create_field", "fe_destroy_field", "fe_eval_coupling_matrices",
               "fe_eval_coupling_residual", "fe_eval_coupling_scalar",
               "fe_group_cells", "fe_gather_rows_i32", "fe_gather_rows_f64",
               "fe_eval_residual_peer", "fe_ipc_alloc", "fe_ipc_free", "fe_ipc_open", "fe_ipc_close",
               "fe_geometry", "fe_last_error", "fe_last_error_element", "fe_launch_count",
               "fe_create_csr", "fe_csr_info", "fe_csr_arrays", "fe_csr_copy_arrays",
               "fe_assemble_matrix", "fe_destroy_csr", "fe_set_option", "fe_get_option",
               "fe_eval_stress_integral")


def lib():
    """The loaded ctypes library (raises ImportError if not built)."""
    global _lib_handle
    if _lib_handle is None:
        _lib_handle = _load()
    return _lib_handle


def _check(status: int):
    if status != FE_OK:
        raise FEError(status, _lib.fe_last_error().decode(), int(_lib.fe_last_error_element()))


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _dev(t: Optional[torch.Tensor], dtype=None, device="cuda"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    return t.to(device=device, dtype=dtype or t.dtype).contiguous()


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def fe_last_error() -> str:
    return _lib.fe_last_error().decode()


def fe_launch_count() -> int:
    return int(_lib.fe_launch_count())


def fe_create_mesh_geometry(coords: torch.Tensor, conn: torch.Tensor, order: int, q1d: int,
                            n_nodes: int, dof_conn: Optional[torch.Tensor] = None,
                            stream=None) -> int:
    """coords [V][3] f64, conn [E][8] i32, dof_conn [E][nb] i32 (device tensors)."""
    out = ctypes.c_void_p()
    _check(_lib.fe_create_mesh_geometry(coords.shape[0], _ptr(coords), conn.shape[0], _ptr(conn),
                                        order, q1d, n_nodes, _ptr(dof_conn), _stream(stream),
                                        ctypes.byref(out)))
    return out.value


def _release_stream(device):
    """Stream for the stream-ordered release of a handle: the current stream of its device
    (where the handle's work was queued in the usual single-stream use); NULL (legacy default
    stream) when torch cannot tell (interpreter shutdown)."""
    try:
        return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    except Exception:
        return None


def fe_destroy_mesh(handle: int, stream=None):
    _check(_lib.fe_destroy_mesh(handle, _stream(stream) if stream is not None else None))


# ---- process-wide implementation options (fe_set_option; include/feb200.h)
OPT_MATRIX_IMPL, OPT_RESIDUAL_IMPL, OPT_CSR_IMPL, OPT_MAX_CTAS = range(4)
_OPT_NAMES = {"matrix_impl": OPT_MATRIX_IMPL, "residual_impl": OPT_RESIDUAL_IMPL,
              "csr_impl": OPT_CSR_IMPL, "max_ctas": OPT_MAX_CTAS}
_OPT_VALUES = {OPT_MATRIX_IMPL: {"default": 0, "sf1": 1, "dense": 2},
               OPT_RESIDUAL_IMPL: {"default": 0, "sf": 1, "dense": 2},
               OPT_CSR_IMPL: {"atomic": 0, "gather": 1}}


def fe_set_option(option: int, value: int):
    _check(_lib.fe_set_option(option, int(value)))


def fe_get_option(option: int) -> int:
    v = ctypes.c_int64()
    _check(_lib.fe_get_option(option, ctypes.byref(v)))
    return v.value


def get_options() -> dict:
    """The active implementation options by name (values as set, 0 = default)."""
    return {k: fe_get_option(o) for k, o in _OPT_NAMES.items()}


class options:
    """Context manager that sets implementation options and restores them on exit, e.g.
    ``with fe.options(matrix_impl="dense", max_ctas=3): ...`` (values by name or number)."""

    def __init__(self, **kw):
        self.kw = kw
        self.saved = {}

    def __enter__(self):
        for k, v in self.kw.items():
            o = _OPT_NAMES[k]
            v = _OPT_VALUES.get(o, {}).get(v, v) if isinstance(v, str) else v
            self.saved[o] = fe_get_option(o)
            fe_set_option(o, v)
        return self

    def __exit__(self, *a):
        for o, v in self.saved.items():
            fe_set_option(o, v)


def fe_mesh_info(handle: int) -> fe_info:
    info = fe_info()
    _check(_lib.fe_mesh_info(handle, ctypes.byref(info)))
    return info


def _material(kind, a, b):
    return fe_material(kind, _ptr(a), _ptr(b))


def fe_eval_element_matrices(handle: int, form: int, dtype: int, mat_kind: int,
                             mat_a: Optional[torch.Tensor], mat_b: Optional[torch.Tensor],
                             state_u: Optional[torch.Tensor], elem_begin: int, elem_end: int,
                             K: torch.Tensor, stream=None):
    m = _material(mat_kind, mat_a, mat_b)
    _check(_lib.fe_eval_element_matrices(handle, form, dtype, ctypes.byref(m), _ptr(state_u),
                                         elem_begin, elem_end, _ptr(K), _stream(stream)))


def fe_eval_residual(handle: int, form: int, dtype: int, mat_kind: int,
                     mat_a: Optional[torch.Tensor], mat_b: Optional[torch.Tensor],
                     u: torch.Tensor, elem_begin: int, elem_end: int,
                     r_elem: Optional[torch.Tensor], r_global: Optional[torch.Tensor],
                     stream=None):
    m = _material(mat_kind, mat_a, mat_b)
    _check(_lib.fe_eval_residual(handle, form, dtype, ctypes.byref(m), _ptr(u), elem_begin,
                                 elem_end, _ptr(r_elem), _ptr(r_global), _stream(stream)))


def fe_eval_residual_peer(handle: int, form: int, mat_kind: int, mat_a, mat_b, u: torch.Tensor,
                          elem_begin: int, elem_end: int, r_elem, r_global, windows, stream=None):
    """C-ABI fe_eval_residual_peer: fp64 residual whose fused scatter also adds the nodes of up
    to two windows [(node_begin, node_end, dst_ptr, dst_node_offset), ...] into dst (peer memory
    of a neighbouring rank: the z-slab interface exchange inside the residual kernel)."""
    m = _material(mat_kind, mat_a, mat_b)
    arr = (fe_peer_window * 2)()
    for i, (lo, hi, dst, off) in enumerate(windows):
        arr[i] = fe_peer_window(lo, hi, dst, off)
    _check(_lib.fe_eval_residual_peer(handle, form, ctypes.byref(m), _ptr(u), elem_begin, elem_end,
                                      _ptr(r_elem), _ptr(r_global), arr, len(windows),
                                      _stream(stream)))


class IpcVector:
    """A device fp64 vector allocated with fe_ipc_alloc (shareable with other processes through
    its 64-byte handle); `tensor` views it as a torch tensor (CUDA array interface)."""

    def __init__(self, shape, device="cuda"):
        n = 1
        for s in shape:
            n *= s
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        with torch.cuda.device(device):
            _check(_lib.fe_ipc_alloc(8 * n, ctypes.byref(ptr), handle))
        self.ptr, self.handle, self.shape = ptr.value, handle.raw, tuple(shape)
        self.__cuda_array_interface__ = {"shape": self.shape, "typestr": "<f8",
                                         "data": (self.ptr, False), "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device=device)

    def close(self):
        if getattr(self, "ptr", None):
            self.tensor = None
            _lib.fe_ipc_free(self.ptr)
            self.ptr = None


def ipc_open(handle: bytes) -> int:
    """Map another process's fe_ipc_alloc buffer; returns the device pointer."""
    ptr = ctypes.c_void_p()
    _check(_lib.fe_ipc_open(handle, ctypes.byref(ptr)))
    return ptr.value


def ipc_close(ptr: int):
    _check(_lib.fe_ipc_close(ptr))


def fe_eval_matrix_residual(handle: int, form: int, dtype: int, mat_kind: int, mat_a, mat_b, u,
                            elem_begin: int, elem_end: int, K, r_elem, r_global, stream=None):
    """C-ABI fe_eval_matrix_residual: element matrices and r_e = K_e u_e in one kernel."""
    m = _material(mat_kind, mat_a, mat_b)
    _check(_lib.fe_eval_matrix_residual(handle, form, dtype, ctypes.byref(m), _ptr(u), elem_begin,
                                        elem_end, _ptr(K), _ptr(r_elem), _ptr(r_global),
                                        _stream(stream)))


def fe_assemble_vector(handle: int, dtype: int, ncomp: int, elem_begin: int, elem_end: int,
                       r_elem: torch.Tensor, r_global: torch.Tensor, stream=None):
    _check(_lib.fe_assemble_vector(handle, dtype, ncomp, elem_begin, elem_end, _ptr(r_elem),
                                   _ptr(r_global), _stream(stream)))


def fe_eval_scalar(handle: int, form: int, dtype: int, mat_kind: int,
                   mat_a: Optional[torch.Tensor], mat_b: Optional[torch.Tensor], u: torch.Tensor,
                   elem_begin: int, elem_end: int, value: torch.Tensor, stream=None):
    """value (1-element fp64 device tensor) += the form's integral with v = u (eval mode)."""
    m = _material(mat_kind, mat_a, mat_b)
    _check(_lib.fe_eval_scalar(handle, form, dtype, ctypes.byref(m), _ptr(u), elem_begin, elem_end,
                               _ptr(value), _stream(stream)))


def fe_eval_stress(handle: int, mat_kind: int, mat_a: Optional[torch.Tensor],
                   mat_b: Optional[torch.Tensor], u: torch.Tensor, elem_begin: int, elem_end: int,
                   sigma: torch.Tensor, stream=None):
    """sigma [E'][nq][6] (fp64 device) = D e(u) at the quadrature points (Tab. 2)."""
    m = _material(mat_kind, mat_a, mat_b)
    _check(_lib.fe_eval_stress(handle, ctypes.byref(m), _ptr(u), elem_begin, elem_end, _ptr(sigma),
                               _stream(stream)))


def fe_eval_stress_integral(handle: int, mat_kind: int, mat_a: Optional[torch.Tensor],
                            mat_b: Optional[torch.Tensor], u: torch.Tensor, elem_begin: int,
                            elem_end: int, sigma_int: torch.Tensor, stream=None):
    """sigma_int [E'][6] (fp64 device) = int_e sigma dx per cell ('eval' mode)."""
    m = _material(mat_kind, mat_a, mat_b)
    _check(_lib.fe_eval_stress_integral(handle, ctypes.byref(m), _ptr(u), elem_begin, elem_end,
                                        _ptr(sigma_int), _stream(stream)))


def fe_geometry(handle: int, detw: Optional[torch.Tensor], jinv: Optional[torch.Tensor],
                stream=None):
    _check(_lib.fe_geometry(handle, _ptr(detw), _ptr(jinv), _stream(stream)))


class PressureField:
    """Scalar pressure space Q_pp on the cells of a (velocity) Mesh (fe_create_field), and the
    Stokes coupling forms of Tab. 2 between the two."""

    def __init__(self, mesh: "Mesh", order: int, dof_conn, n_nodes: Optional[int] = None,
                 stream=None):
        dof_conn = _dev(dof_conn, torch.int32, mesh.device)
        n_nodes = int(dof_conn.max().item()) + 1 if n_nodes is None else n_nodes
        out = ctypes.c_void_p()
        _check(_lib.fe_create_field(mesh.handle, order, n_nodes, _ptr(dof_conn), _stream(stream),
                                    ctypes.byref(out)))
        self.handle, self.mesh, self.order, self.n_nodes = out.value, mesh, order, n_nodes
        self.nb = (order + 1) ** 3

    def coupling_matrices(self, transposed=False, elem_begin=0, elem_end=None, out=None,
                          stream=None):
        """B [E'][3 nbv][nbp] ('i.i,0', v, p) or, transposed, C [E'][nbp][3 nbv] ('i.i,0', u, q)."""
        m = self.mesh
        elem_end = m.n_elems if elem_end is None else elem_end
        shape = (self.nb, 3 * m.nb) if transposed else (3 * m.nb, self.nb)
        if out is None:
            out = torch.empty((max(elem_end - elem_begin, 0),) + shape, dtype=torch.float64,
                              device=m.device)
        _check(_lib.fe_eval_coupling_matrices(m.handle, self.handle, int(transposed), elem_begin,
                                              elem_end, _ptr(out), _stream(stream)))
        return out

    def coupling_residual(self, x, transposed=False, elem_begin=0, elem_end=None,
                          want_elem=False, want_global=True, r_elem=None, r_global=None,
                          stream=None):
        """transposed=False: x = pressure [n_p] -> r_v (velocity-shaped); True: x = velocity
        [n_v][3] -> r_q (pressure-shaped).  Returns (r_elem or None, r_global or None)."""
        m = self.mesh
        elem_end = m.n_elems if elem_end is None else elem_end
        n = max(elem_end - elem_begin, 0)
        if want_elem and r_elem is None:
            r_elem = torch.empty((n, self.nb if transposed else 3 * m.nb), dtype=torch.float64,
                                 device=m.device)
        if want_global and r_global is None:
            shape = (self.n_nodes,) if transposed else (m.n_nodes, 3)
            r_global = torch.zeros(shape, dtype=torch.float64, device=m.device)
        _check(_lib.fe_eval_coupling_residual(m.handle, self.handle, int(transposed), _ptr(x),
                                              elem_begin, elem_end, _ptr(r_elem), _ptr(r_global),
                                              _stream(stream)))
        return r_elem, r_global

    def coupling_eval(self, u, p, elem_begin=0, elem_end=None, stream=None):
        """int p_h div u_h (eval mode), a 1-element fp64 device tensor."""
        m = self.mesh
        elem_end = m.n_elems if elem_end is None else elem_end
        value = torch.zeros(1, dtype=torch.float64, device=m.device)
        _check(_lib.fe_eval_coupling_scalar(m.handle, self.handle, _ptr(u), _ptr(p), elem_begin,
                                            elem_end, _ptr(value), _stream(stream)))
        return value

    def close(self):
        if getattr(self, "handle", None):
            _check(_lib.fe_destroy_field(self.handle, _release_stream(self.mesh.device)))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fe_group_cells(kind: torch.Tensor, n_kinds: int, stream=None):
    """Stable grouping of cells by kind (GPU): (perm int64 device [E], offsets list [n_kinds+1])."""
    kind = kind.to(dtype=torch.int32).contiguous()
    perm = torch.empty(kind.numel(), dtype=torch.int64, device=kind.device)
    offs = (ctypes.c_int64 * (n_kinds + 1))()
    _check(_lib.fe_group_cells(_ptr(kind), kind.numel(), n_kinds, _ptr(perm), offs,
                               _stream(stream)))
    return perm, list(offs)


def fe_gather_rows(src: torch.Tensor, width: int, perm: torch.Tensor, row_ptr=None, stream=None):
    """out[i][j] = src[row_ptr[perm[i]] + j] (or src[perm[i] * width + j]); int32 or fp64."""
    n = perm.numel()
    out = torch.empty((n, width), dtype=src.dtype, device=src.device)
    f = _lib.fe_gather_rows_i32 if src.dtype == torch.int32 else _lib.fe_gather_rows_f64
    if src.dtype not in (torch.int32, torch.float64):
        raise TypeError("fe_gather_rows: int32 or float64 only")
    _check(f(_ptr(src), _ptr(row_ptr), width, _ptr(perm), n, _ptr(out), _stream(stream)))
    return out


class MixedMesh:
    """A p-mixed hexahedral mesh evaluated group by group.

    orders[E] (1..4) per cell; dof_ptr[E+1] / dof_idx: each cell's (order+1)^3 node ids
    (CSR rows, lexicographic local order).  Cells are grouped by order with fe_group_cells;
    each group is a Mesh of one order built from rows gathered by fe_gather_rows, and every
    evaluation runs the single-kind kernels per group.  No conformity constraints between
    orders are applied (the paper's setting has none)."""

    def __init__(self, coords, conn, orders, dof_ptr, dof_idx, n_nodes: int, device="cuda",
                 stream=None):
        coords = _dev(coords, torch.float64, device)
        conn = _dev(conn, torch.int32, device)
        orders = _dev(orders, torch.int32, device)
        dof_ptr = _dev(dof_ptr, torch.int64, device)
        dof_idx = _dev(dof_idx, torch.int32, device)
        self.device, self.n_nodes, self.n_elems = device, n_nodes, conn.shape[0]
        self.perm, offs = fe_group_cells(orders - 1, 4, stream)
        self.groups = []   # (order, begin, end, Mesh, perm slice)
        for g in range(4):
            b, e = offs[g], offs[g + 1]
            if e <= b:
                continue
            p = g + 1
            pg = self.perm[b:e]
            cg = fe_gather_rows(conn, 8, pg, stream=stream)
            dg = fe_gather_rows(dof_idx, (p + 1) ** 3, pg, row_ptr=dof_ptr, stream=stream)
            m = Mesh(coords, cg, p, dof_conn=dg, n_nodes=n_nodes, device=device, stream=stream)
            self.groups.append((p, b, e, m, pg))

    def group_material(self, arr, row_ptr=None, stream=None):
        """Per-group blocks of a per-cell array in original cell order: `arr` [E][w] fixed
        width (row_ptr None), or ragged rows (e.g. per-qp values, (p+1)^3 per cell)."""
        out = []
        for p, b, e, m, pg in self.groups:
            w = (p + 1) ** 3 if row_ptr is not None else arr.shape[1] if arr.dim() > 1 else 1
            out.append(fe_gather_rows(arr.reshape(arr.shape[0], -1) if row_ptr is None else arr,
                                      w, pg, row_ptr=row_ptr, stream=stream))
        return out

    def element_matrices(self, form, mat_kind=MAT_PER_QP, mats_a=None, mats_b=None, stream=None):
        """List of per-group K blocks [E_g][D nb_g][D nb_g]; group g's cells are
        perm[begin_g:end_g]."""
        out = []
        for i, (p, b, e, m, pg) in enumerate(self.groups):
            out.append(m.element_matrices(form, mat_kind, None if mats_a is None else mats_a[i],
                                          None if mats_b is None else mats_b[i], stream=stream))
        return out

    def residual(self, form, u, mat_kind=MAT_PER_QP, mats_a=None, mats_b=None, r_global=None,
                 stream=None):
        """Global residual: the per-group kernels scatter-add into one vector."""
        if r_global is None:
            r_global = torch.zeros((self.n_nodes, NCOMP[form]), dtype=u.dtype, device=self.device)
        for i, (p, b, e, m, pg) in enumerate(self.groups):
            m.residual(form, u, mat_kind, None if mats_a is None else mats_a[i],
                       None if mats_b is None else mats_b[i], r_global=r_global, stream=stream)
        return r_global


class CSR:
    """Global sparse matrix pattern (fe_create_csr) and assembly (fe_assemble_matrix)."""

    def __init__(self, mesh: "Mesh", ncomp: int, stream=None):
        out = ctypes.c_void_p()
        _check(_lib.fe_create_csr(mesh.handle, ncomp, _stream(stream), ctypes.byref(out)))
        self.handle, self.mesh, self.ncomp = out.value, mesh, ncomp
        nr, nz = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.fe_csr_info(self.handle, ctypes.byref(nr), ctypes.byref(nz)))
        self.n_rows, self.nnz = nr.value, nz.value

    def arrays(self):
        """(row_ptr int64 [n_rows+1], col_idx int32 [nnz]) copied to host numpy arrays."""
        import numpy as np
        row_ptr = torch.empty(self.n_rows + 1, dtype=torch.int64, device=self.mesh.device)
        col = torch.empty(self.nnz, dtype=torch.int32, device=self.mesh.device)
        _check(_lib.fe_csr_copy_arrays(self.handle, _ptr(row_ptr), _ptr(col), _stream(None)))
        return row_ptr.cpu().numpy(), col.cpu().numpy().astype(np.int64)

    def assemble(self, K, elem_begin=0, elem_end=None, values=None, stream=None):
        elem_end = self.mesh.n_elems if elem_end is None else elem_end
        if values is None:
            values = torch.zeros(self.nnz, dtype=torch.float64, device=self.mesh.device)
        _check(_lib.fe_assemble_matrix(self.handle, _ptr(K), elem_begin, elem_end, _ptr(values),
                                       _stream(stream)))
        return values

    def close(self):
        if getattr(self, "handle", None):
            _check(_lib.fe_destroy_csr(self.handle, _release_stream(self.mesh.device)))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Mesh:
    """Owning wrapper of an fe_mesh handle plus convenience evaluators.

    All evaluation goes through the C ABI; this class only allocates outputs."""

    def __init__(self, coords, conn, order: int, q1d: Optional[int] = None,
                 dof_conn=None, n_nodes: Optional[int] = None, device="cuda", stream=None):
        q1d = order + 1 if q1d is None else q1d
        coords = _dev(coords, torch.float64, device)
        conn = _dev(conn, torch.int32, device)
        dof_conn = None if (dof_conn is None or order == 1 and dof_conn is None) else _dev(
            dof_conn, torch.int32, device)
        if n_nodes is None:
            n_nodes = coords.shape[0] if dof_conn is None else int(dof_conn.max().item()) + 1
        self.device = device
        self.handle = fe_create_mesh_geometry(coords, conn, order, q1d, n_nodes, dof_conn, stream)
        info = fe_mesh_info(self.handle)
        self.order, self.q1d, self.nb, self.nq = info.order, info.q1d, info.nb, info.nq
        self.n_elems, self.n_nodes, self.n_vertices = info.n_elems, info.n_nodes, info.n_vertices
        self.min_det_j = info.min_det_j

    def close(self):
        if getattr(self, "handle", None):
            _check(_lib.fe_destroy_mesh(self.handle, _release_stream(self.device)))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def element_matrices(self, form, mat_kind=MAT_PER_QP, mat_a=None, mat_b=None, state_u=None,
                         elem_begin=0, elem_end=None, out=None, stream=None):
        """K [E'][ndof][ndof]; fp32 coefficient arrays select the FE_F32 path (fp32 K)."""
        elem_end = self.n_elems if elem_end is None else elem_end
        ndof = NCOMP[form] * self.nb
        f32 = mat_a is not None and mat_a.dtype == torch.float32
        if out is None:
            out = torch.empty((elem_end - elem_begin, ndof, ndof),
                              dtype=torch.float32 if f32 else torch.float64, device=self.device)
        fe_eval_element_matrices(self.handle, form, F32 if f32 else F64, mat_kind, mat_a, mat_b,
                                 state_u, elem_begin, elem_end, out, stream)
        return out

    def residual(self, form, u, mat_kind=MAT_PER_QP, mat_a=None, mat_b=None, elem_begin=0,
                 elem_end=None, r_elem=None, r_global=None, want_elem=False, want_global=True,
                 stream=None):
        elem_end = self.n_elems if elem_end is None else elem_end
        dt = F64 if u.dtype == torch.float64 else F32
        D = NCOMP[form]
        if want_elem and r_elem is None:
            r_elem = torch.empty((elem_end - elem_begin, D * self.nb), dtype=u.dtype,
                                 device=self.device)
        if want_global and r_global is None:
            r_global = torch.zeros((self.n_nodes, D), dtype=u.dtype, device=self.device)
        fe_eval_residual(self.handle, form, dt, mat_kind, mat_a, mat_b, u, elem_begin, elem_end,
                         r_elem, r_global, stream)
        return r_elem, r_global

    def matrix_residual(self, form, u, mat_kind=MAT_PER_QP, mat_a=None, mat_b=None, elem_begin=0,
                        elem_end=None, K=None, r_elem=None, r_global=None, want_elem=False,
                        stream=None):
        """Element matrices and the residual r_e = K_e u_e of a linear scalar form, one pass."""
        elem_end = self.n_elems if elem_end is None else elem_end
        n = elem_end - elem_begin
        if K is None:
            K = torch.empty((n, self.nb, self.nb), dtype=torch.float64, device=self.device)
        if want_elem and r_elem is None:
            r_elem = torch.empty((n, self.nb), dtype=torch.float64, device=self.device)
        if r_global is None:
            r_global = torch.zeros((self.n_nodes, 1), dtype=torch.float64, device=self.device)
        fe_eval_matrix_residual(self.handle, form, F64, mat_kind, mat_a, mat_b, u, elem_begin,
                                elem_end, K, r_elem, r_global, stream)
        return K, r_elem, r_global

    def assemble(self, r_elem, ncomp, r_global=None, elem_begin=0, elem_end=None, stream=None):
        elem_end = self.n_elems if elem_end is None else elem_end
        if r_global is None:
            r_global = torch.zeros((self.n_nodes, ncomp), dtype=r_elem.dtype, device=self.device)
        dt = F64 if r_elem.dtype == torch.float64 else F32
        fe_assemble_vector(self.handle, dt, ncomp, elem_begin, elem_end, r_elem, r_global, stream)
        return r_global

    def eval_scalar(self, form, u, mat_kind=MAT_PER_QP, mat_a=None, mat_b=None, elem_begin=0,
                    elem_end=None, stream=None):
        elem_end = self.n_elems if elem_end is None else elem_end
        value = torch.zeros(1, dtype=torch.float64, device=self.device)
        dt = F64 if u.dtype == torch.float64 else F32
        fe_eval_scalar(self.handle, form, dt, mat_kind, mat_a, mat_b, u, elem_begin, elem_end,
                       value, stream)
        return value

    def stress(self, u, mat_kind=MAT_PER_QP, mat_a=None, mat_b=None, elem_begin=0, elem_end=None,
               stream=None):
        elem_end = self.n_elems if elem_end is None else elem_end
        sigma = torch.empty((max(elem_end - elem_begin, 0), self.nq, 6), dtype=torch.float64,
                            device=self.device)
        fe_eval_stress(self.handle, mat_kind, mat_a, mat_b, u, elem_begin, elem_end, sigma, stream)
        return sigma

    def stress_integral(self, u, mat_kind=MAT_PER_QP, mat_a=None, mat_b=None, elem_begin=0,
                        elem_end=None, stream=None):
        elem_end = self.n_elems if elem_end is None else elem_end
        out = torch.empty((max(elem_end - elem_begin, 0), 6), dtype=torch.float64,
                          device=self.device)
        fe_eval_stress_integral(self.handle, mat_kind, mat_a, mat_b, u, elem_begin, elem_end, out,
                                stream)
        return out

    def geometry(self, stream=None):
        detw = torch.empty((self.n_elems, self.nq), dtype=torch.float64, device=self.device)
        jinv = torch.empty((self.n_elems, self.nq, 3, 3), dtype=torch.float64, device=self.device)
        fe_geometry(self.handle, detw, jinv, stream)
        return detw, jinv
