"""ctypes front-end of the C oracle (oracle/fe_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2107_04121_b200) never imports this module, and this module never
imports the product package; they share only fe_inputs (seeded inputs).

Every function here is argument marshalling around the plain C definition of
PAPER.md Alg. 1 / Alg. 2; see fe_oracle.c for the citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fe_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK = 0
ERR_ARG = -1
ERR_DEGENERATE = -3


# ORACLE_SANITIZE=1 in the environment: an AddressSanitizer + UndefinedBehaviorSanitizer build of
# the same source (liboracle_san.so), used by tests/test_oracle_sanitized.py in a subprocess with
# libasan preloaded (an ASan/UBSan host build of the oracle).
_SANITIZE = os.environ.get("ORACLE_SANITIZE", "") not in ("", "0")
_LIB_SAN = os.path.join(_HERE, "liboracle_san.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, IEEE fp64, no fast-math, OpenMP over cells)."""
    if _SANITIZE:
        if force or not os.path.exists(_LIB_SAN) or os.path.getmtime(_LIB_SAN) < os.path.getmtime(_SRC):
            cmd = ["gcc", "-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
                   "-fno-sanitize-recover=undefined", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                   "-Wall", "-o", _LIB_SAN, _SRC, "-lm"]
            subprocess.run(cmd, check=True)
        return _LIB_SAN
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        ci = ctypes.c_int
        _lib.oracle_gauss_legendre.argtypes = [ci, P, P]
        _lib.oracle_lagrange_1d.argtypes = [ci, ctypes.c_double, P, P]
        _lib.oracle_tables.argtypes = [ci, ci, P, P, P, P]
        _lib.oracle_geometry.argtypes = [ci, i64, P, P, P, P]
        _lib.oracle_eval_matrix.argtypes = [ci, ci, ci, i64, P, P, P, ci, P, P, P, P]
        _lib.oracle_eval_residual.argtypes = [ci, ci, ci, i64, P, P, P, ci, P, P, P, i64, i64, P]
        _lib.oracle_assemble.argtypes = [i64, ci, ci, P, P, P]
        _lib.oracle_isotropic_D.argtypes = [ctypes.c_double, ctypes.c_double, P]
        _lib.oracle_eval_scalar.argtypes = [ci, ci, ci, i64, P, P, P, ci, P, P, P, i64, i64, P]
        _lib.oracle_eval_scalar.restype = ci
        _lib.oracle_eval_stress.argtypes = [ci, ci, i64, P, P, P, ci, P, P, P, i64, i64, P]
        _lib.oracle_eval_stress.restype = ci
        _lib.oracle_eval_stress_integral.argtypes = [ci, ci, i64, P, P, P, ci, P, P, P, i64, i64, P]
        _lib.oracle_eval_stress_integral.restype = ci
        _lib.oracle_coupling_matrix.argtypes = [ci, ci, ci, ci, i64, P, P, i64, i64, P]
        _lib.oracle_coupling_residual.argtypes = [ci, ci, ci, ci, i64, P, P, P, P, P, P, i64, i64, P]
        _lib.oracle_coupling_eval.argtypes = [ci, ci, ci, i64, P, P, P, P, P, P, i64, i64, P]
        for f in ("oracle_coupling_matrix", "oracle_coupling_residual", "oracle_coupling_eval"):
            getattr(_lib, f).restype = ci
        _lib.oracle_bad_element.restype = i64
        for f in ("oracle_gauss_legendre", "oracle_lagrange_1d", "oracle_tables", "oracle_geometry",
                  "oracle_eval_matrix", "oracle_eval_residual", "oracle_assemble"):
            getattr(_lib, f).restype = ci
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status: int, element: int = -1):
        super().__init__(f"oracle status {status}" + (f" (element {element})" if element >= 0 else ""))
        self.status = status
        self.element = element


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's cell loops (timing only); returns the active count."""
    f = lib().oracle_set_threads
    f.restype = ctypes.c_int
    return int(f(int(n)))


def _check(st):
    if st != OK:
        raise OracleError(st, int(lib().oracle_bad_element()))


def gauss_legendre(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    _check(lib().oracle_gauss_legendre(n, _ptr(x), _ptr(w)))
    return x, w


def lagrange_1d(p: int, t: float):
    phi = np.zeros(p + 1)
    dphi = np.zeros(p + 1)
    _check(lib().oracle_lagrange_1d(p, float(t), _ptr(phi), _ptr(dphi)))
    return phi, dphi


def tables(p: int, q1d: int):
    nb, nq = (p + 1) ** 3, q1d ** 3
    xi = np.zeros((nq, 3))
    w = np.zeros(nq)
    Phi = np.zeros((nq, nb))
    dPhi = np.zeros((nq, 3, nb))
    _check(lib().oracle_tables(p, q1d, _ptr(xi), _ptr(w), _ptr(Phi), _ptr(dPhi)))
    return xi, w, Phi, dPhi


def isotropic_D(lam: float, mu: float):
    D = np.zeros((6, 6))
    lib().oracle_isotropic_D(float(lam), float(mu), _ptr(D))
    return D


def geometry(q1d: int, coords, conn):
    coords, conn = _f64(coords), _i32(conn)
    E = conn.shape[0]
    nq = q1d ** 3
    detw = np.zeros((E, nq))
    Jinv = np.zeros((E, nq, 3, 3))
    _check(lib().oracle_geometry(q1d, E, _ptr(coords), _ptr(conn), _ptr(detw), _ptr(Jinv)))
    return detw, Jinv


def _ncomp(form):
    return 3 if form in (2, 4, 5, 6, 7) else 1


def eval_matrix(form, p, q1d, coords, conn, dof_conn=None, mat_kind=0, mat_a=None, mat_b=None,
                u_state=None):
    """Element matrices K[E][ndof][ndof] (Alg. 2)."""
    coords, conn, dof_conn = _f64(coords), _i32(conn), _i32(dof_conn)
    mat_a, mat_b, u_state = _f64(mat_a), _f64(mat_b), _f64(u_state)
    E = conn.shape[0]
    ndof = _ncomp(form) * (p + 1) ** 3
    K = np.zeros((E, ndof, ndof))
    _check(lib().oracle_eval_matrix(form, p, q1d, E, _ptr(coords), _ptr(conn), _ptr(dof_conn),
                                    mat_kind, _ptr(mat_a), _ptr(mat_b), _ptr(u_state), _ptr(K)))
    return K


def eval_residual(form, p, q1d, coords, conn, dof_conn, u, mat_kind=0, mat_a=None, mat_b=None,
                  elem_begin=0, elem_end=None):
    """Element residuals r_elem[E'][ndof] (Alg. 1) over cells [elem_begin, elem_end)."""
    coords, conn, dof_conn = _f64(coords), _i32(conn), _i32(dof_conn)
    mat_a, mat_b, u = _f64(mat_a), _f64(mat_b), _f64(u)
    E = conn.shape[0]
    elem_end = E if elem_end is None else elem_end
    ndof = _ncomp(form) * (p + 1) ** 3
    r = np.zeros((max(elem_end - elem_begin, 0), ndof))
    _check(lib().oracle_eval_residual(form, p, q1d, E, _ptr(coords), _ptr(conn), _ptr(dof_conn),
                                      mat_kind, _ptr(mat_a), _ptr(mat_b), _ptr(u),
                                      elem_begin, elem_end, _ptr(r)))
    return r


def eval_scalar(form, p, q1d, coords, conn, dof_conn, u, mat_kind=0, mat_a=None, mat_b=None,
                elem_begin=0, elem_end=None):
    """'eval' mode: the form's integral with the test function replaced by u."""
    coords, conn, dof_conn = _f64(coords), _i32(conn), _i32(dof_conn)
    mat_a, mat_b, u = _f64(mat_a), _f64(mat_b), _f64(u)
    E = conn.shape[0]
    elem_end = E if elem_end is None else elem_end
    out = np.zeros(1)
    _check(lib().oracle_eval_scalar(form, p, q1d, E, _ptr(coords), _ptr(conn), _ptr(dof_conn),
                                    mat_kind, _ptr(mat_a), _ptr(mat_b), _ptr(u), elem_begin,
                                    elem_end, _ptr(out)))
    return float(out[0])


def eval_stress(p, q1d, coords, conn, dof_conn, u, mat_kind=1, mat_a=None, mat_b=None,
                elem_begin=0, elem_end=None):
    """Cauchy stress sigma = D e(u) (Tab. 2) at every qp: [E'][nq][6] (Voigt)."""
    coords, conn, dof_conn = _f64(coords), _i32(conn), _i32(dof_conn)
    mat_a, mat_b, u = _f64(mat_a), _f64(mat_b), _f64(u)
    E = conn.shape[0]
    elem_end = E if elem_end is None else elem_end
    sig = np.zeros((max(elem_end - elem_begin, 0), q1d ** 3, 6))
    _check(lib().oracle_eval_stress(p, q1d, E, _ptr(coords), _ptr(conn), _ptr(dof_conn), mat_kind,
                                    _ptr(mat_a), _ptr(mat_b), _ptr(u), elem_begin, elem_end,
                                    _ptr(sig)))
    return sig


def eval_stress_integral(p, q1d, coords, conn, dof_conn, u, mat_kind=1, mat_a=None, mat_b=None,
                         elem_begin=0, elem_end=None):
    """Cauchy stress in 'eval' mode: per cell int_e sigma dx, [E'][6] (Voigt)."""
    coords, conn, dof_conn = _f64(coords), _i32(conn), _i32(dof_conn)
    mat_a, mat_b, u = _f64(mat_a), _f64(mat_b), _f64(u)
    E = conn.shape[0]
    elem_end = E if elem_end is None else elem_end
    sig = np.zeros((max(elem_end - elem_begin, 0), 6))
    _check(lib().oracle_eval_stress_integral(p, q1d, E, _ptr(coords), _ptr(conn), _ptr(dof_conn),
                                             mat_kind, _ptr(mat_a), _ptr(mat_b), _ptr(u),
                                             elem_begin, elem_end, _ptr(sig)))
    return sig


def coupling_matrix(pv, pp, q1d, coords, conn, transposed=False, elem_begin=0, elem_end=None):
    """Stokes coupling matrices (Tab. 2 'i.i,0'): B [E'][3 nbv][nbp] (test v,
    trial p) or, transposed, C [E'][nbp][3 nbv] (test q, trial u)."""
    coords, conn = _f64(coords), _i32(conn)
    E = conn.shape[0]
    elem_end = E if elem_end is None else elem_end
    nbv, nbp = (pv + 1) ** 3, (pp + 1) ** 3
    shape = (nbp, 3 * nbv) if transposed else (3 * nbv, nbp)
    out = np.zeros((max(elem_end - elem_begin, 0),) + shape)
    _check(lib().oracle_coupling_matrix(int(transposed), pv, pp, q1d, E, _ptr(coords), _ptr(conn),
                                        elem_begin, elem_end, _ptr(out)))
    return out


def coupling_residual(pv, pp, q1d, coords, conn, dof_v, dof_p, u=None, p=None, transposed=False,
                      elem_begin=0, elem_end=None):
    """Residual of the Stokes coupling (r_v = int div v p_h, input p) or of the transposed
    coupling (r_q = int q div u_h, input u)."""
    coords, conn, dof_v, dof_p = _f64(coords), _i32(conn), _i32(dof_v), _i32(dof_p)
    u, p = _f64(u), _f64(p)
    E = conn.shape[0]
    elem_end = E if elem_end is None else elem_end
    n = (pp + 1) ** 3 if transposed else 3 * (pv + 1) ** 3
    out = np.zeros((max(elem_end - elem_begin, 0), n))
    _check(lib().oracle_coupling_residual(int(transposed), pv, pp, q1d, E, _ptr(coords), _ptr(conn),
                                          _ptr(dof_v), _ptr(dof_p), _ptr(u), _ptr(p), elem_begin,
                                          elem_end, _ptr(out)))
    return out


def coupling_eval(pv, pp, q1d, coords, conn, dof_v, dof_p, u, p, elem_begin=0, elem_end=None):
    """'eval' mode of the coupling: int p_h div u_h."""
    coords, conn, dof_v, dof_p = _f64(coords), _i32(conn), _i32(dof_v), _i32(dof_p)
    u, p = _f64(u), _f64(p)
    E = conn.shape[0]
    elem_end = E if elem_end is None else elem_end
    out = np.zeros(1)
    _check(lib().oracle_coupling_eval(pv, pp, q1d, E, _ptr(coords), _ptr(conn), _ptr(dof_v),
                                      _ptr(dof_p), _ptr(u), _ptr(p), elem_begin, elem_end,
                                      _ptr(out)))
    return float(out[0])


def problem_stress(prob):
    return eval_stress(prob.p, prob.q1d, prob.coords, prob.conn, prob.dof_conn, prob.u,
                       prob.mat_kind, prob.mat_a, prob.mat_b)


def problem_eval_scalar(prob):
    return eval_scalar(prob.form, prob.p, prob.q1d, prob.coords, prob.conn, prob.dof_conn, prob.u,
                       prob.mat_kind, prob.mat_a, prob.mat_b)


def assemble(r_elem, dof_conn, n_nodes, ncomp, r_global=None):
    """Serial scatter-add r_global[dof_conn[e][k]*D + a] += r_elem[e][a*nb + k]."""
    r_elem, dof_conn = _f64(r_elem), _i32(dof_conn)
    E, nb = dof_conn.shape
    if r_global is None:
        r_global = np.zeros(n_nodes * ncomp)
    _check(lib().oracle_assemble(E, nb, ncomp, _ptr(dof_conn), _ptr(r_elem), _ptr(r_global)))
    return r_global


def problem_matrix(prob):
    """eval_matrix on a fe_inputs.Problem."""
    return eval_matrix(prob.form, prob.p, prob.q1d, prob.coords, prob.conn, prob.dof_conn,
                       prob.mat_kind, prob.mat_a, prob.mat_b,
                       prob.u if prob.form == 5 else None)


def problem_residual(prob, elem_begin=0, elem_end=None):
    return eval_residual(prob.form, prob.p, prob.q1d, prob.coords, prob.conn, prob.dof_conn,
                         prob.u, prob.mat_kind, prob.mat_a, prob.mat_b, elem_begin, elem_end)


def problem_assembled_residual(prob):
    r = problem_residual(prob)
    return assemble(r, prob.dof_conn, prob.n_nodes, prob.ncomp)
