"""ctypes loader for the CPU oracle (oracle/hom2d_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs are the only permitted importers.  The
product package (paper_1709_01619_b200) never imports this module.

The oracle is a plain fp64 C program compiled with ``-O2 -ffp-contract=off``;
see the header of hom2d_oracle.c for the paper passages each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "hom2d_oracle.c")
LIB = os.path.join(HERE, "liboracle_hom2d.so")

FV, CPR, DG, NDG, SD = 0, 1, 2, 3, 4
PERIODIC, TRANSMISSIVE = 0, 1
VORTEX, SHOCK = 0, 1
METHODS = {"fv": FV, "cpr": CPR, "dg": DG, "ndg": NDG, "sd": SD}


class OrcConfig(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32),
        ("xmin", C.c_double), ("xmax", C.c_double),
        ("ymin", C.c_double), ("ymax", C.c_double),
        ("bc", C.c_int32), ("method", C.c_int32), ("k", C.c_int32),
        ("gamma", C.c_double), ("cfl", C.c_double),
        ("limiter", C.c_int32), ("limiter_eps", C.c_double),
        ("cpr_chain_rule", C.c_int32),
        ("physics", C.c_int32), ("adv_a", C.c_double), ("adv_b", C.c_double),
        ("dt_fixed", C.c_double),
        ("limiter_per_step", C.c_int32), ("limiter_all_vars", C.c_int32), ("fv_unlimited", C.c_int32),
        ("limiter_characteristic", C.c_int32), ("fv_error_recon", C.c_int32),
        ("dg_overintegrate", C.c_int32),
    ]


def build(force: bool = False) -> str:
    """Compile liboracle_hom2d.so (plain C, fp64, no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-fopenmp", "-fPIC", "-shared",
             "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        d, i32, i64, vp = C.c_double, C.c_int32, C.c_int64, C.c_void_p
        P = C.POINTER
        cfgp = P(OrcConfig)
        L.orc_nodes.argtypes = [C.c_int, C.c_int, vp, vp]
        L.orc_lagrange.argtypes = [C.c_int, vp, d, vp]
        L.orc_lagrange_deriv.argtypes = [C.c_int, vp, d, vp]
        L.orc_radau_dgR.argtypes = [C.c_int, d]
        L.orc_radau_dgR.restype = d
        for fn in ("orc_flux", "orc_jacobian_apply"):
            getattr(L, fn).argtypes = [cfgp, C.c_int, vp, vp] + ([vp] if fn == "orc_jacobian_apply" else [])
        L.orc_rusanov.argtypes = [cfgp, C.c_int, vp, vp, vp]
        L.orc_wave_speed.argtypes = [cfgp, vp]
        L.orc_wave_speed.restype = d
        L.orc_pressure.argtypes = [cfgp, vp]
        L.orc_pressure.restype = d
        L.orc_minmod2.argtypes = [d, d]
        L.orc_minmod2.restype = d
        L.orc_minmod3.argtypes = [d, d, d]
        L.orc_minmod3.restype = d
        L.orc_muscl_face.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp]
        L.orc_muscl_face_unlimited.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp]
        L.orc_char_vectors.argtypes = [cfgp, C.c_int, vp, vp, vp]
        L.orc_residual.argtypes = [cfgp, vp, vp, vp]
        L.orc_residual_map.argtypes = [cfgp, vp, vp, vp, vp]
        L.orc_averages.argtypes = [cfgp, vp, vp]
        L.orc_limit.argtypes = [cfgp, vp, vp, vp]
        L.orc_max_wave_speed.argtypes = [cfgp, vp]
        L.orc_max_wave_speed.restype = d
        L.orc_dt.argtypes = [cfgp, vp]
        L.orc_dt.restype = d
        L.orc_ssprk3.argtypes = [vp, i64, d, vp, vp, vp]
        L.orc_run.argtypes = [cfgp, vp, i32, d, P(d), P(i64), vp]
        L.orc_run_map.argtypes = [cfgp, vp, i32, d, P(d), P(i64), vp, vp]
        L.orc_vortex_state.argtypes = [cfgp, d, d, d, vp]
        L.orc_shock_state.argtypes = [cfgp, d, d, vp]
        L.orc_init_case.argtypes = [cfgp, C.c_int, vp]
        L.orc_point_coords.argtypes = [cfgp, vp, vp]
        L.orc_error.argtypes = [cfgp, vp, C.c_int, d, C.c_int, P(d), P(d), P(d)]
        L.orc_fv_recon_points.argtypes = [cfgp, vp, C.c_int, vp]
        L.orc_residual_dg_quad.argtypes = [cfgp, C.c_int, vp, vp]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        L.orc_set_threads(1)  # definitional single thread unless asked (bench's nproc leg)
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype in (np.float64, np.int64, np.int32) and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def config(nx=10, ny=10, method="cpr", k=1, bc=PERIODIC, box=(-5.0, 5.0, -5.0, 5.0), gamma=1.4,
           cfl=0.24, limiter=0, limiter_eps=1e-3, cpr_chain_rule=1, physics=0, adv=(1.0, 0.5),
           dt_fixed=0.0, limiter_per_step=0, limiter_all_vars=0, fv_unlimited=0,
           limiter_characteristic=0, fv_error_recon=0, dg_overintegrate=0) -> OrcConfig:
    m = METHODS[method] if isinstance(method, str) else int(method)
    return OrcConfig(nx, ny, box[0], box[1], box[2], box[3], bc, m, k, gamma, cfl, limiter,
                     limiter_eps, cpr_chain_rule, physics, adv[0], adv[1], dt_fixed,
                     limiter_per_step, limiter_all_vars, fv_unlimited, limiter_characteristic,
                     fv_error_recon, dg_overintegrate)


def npts(cfg: OrcConfig) -> int:
    return 1 if cfg.method == FV else (cfg.k + 1) ** 2


def nvalues(cfg: OrcConfig) -> int:
    return 4 * cfg.nx * cfg.ny * npts(cfg)


def _chk(st):
    if st != 0:
        raise RuntimeError(f"oracle status {st}")


def nodes(kind: int, n: int):
    xi, w = np.zeros(n), np.zeros(n)
    _chk(lib().orc_nodes(kind, n, _p(xi), _p(w)))
    return xi, w


def lagrange(xi, x):
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    out = np.zeros(len(xi))
    lib().orc_lagrange(len(xi), _p(xi), float(x), _p(out))
    return out


def lagrange_deriv(xi, x):
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    out = np.zeros(len(xi))
    lib().orc_lagrange_deriv(len(xi), _p(xi), float(x), _p(out))
    return out


def radau_dgR(k, x):
    return lib().orc_radau_dgR(k, float(x))


def _v4(q):
    return np.ascontiguousarray(q, dtype=np.float64)


def flux(cfg, dir, q):
    q = _v4(q); f = np.zeros(4)
    lib().orc_flux(C.byref(cfg), dir, _p(q), _p(f))
    return f


def rusanov(cfg, dir, qL, qR):
    qL, qR = _v4(qL), _v4(qR); F = np.zeros(4)
    lib().orc_rusanov(C.byref(cfg), dir, _p(qL), _p(qR), _p(F))
    return F


def char_vectors(cfg, dir, q):
    """(R, L) 4x4: right / left eigenvectors of the flux Jacobian along axis dir at q."""
    R, Lm = np.zeros(16), np.zeros(16)
    lib().orc_char_vectors(C.byref(cfg), dir, _p(_v4(q)), _p(R), _p(Lm))
    return R.reshape(4, 4), Lm.reshape(4, 4)


def jacobian_apply(cfg, dir, q, d):
    q, d = _v4(q), _v4(d); o = np.zeros(4)
    lib().orc_jacobian_apply(C.byref(cfg), dir, _p(q), _p(d), _p(o))
    return o


def wave_speed(cfg, q):
    return lib().orc_wave_speed(C.byref(cfg), _p(_v4(q)))


def pressure(cfg, q):
    return lib().orc_pressure(C.byref(cfg), _p(_v4(q)))


def minmod2(a, b):
    return lib().orc_minmod2(float(a), float(b))


def minmod3(a, b, c):
    return lib().orc_minmod3(float(a), float(b), float(c))


def muscl_face(order, qm1, q0, q1, q2, unlimited=False):
    qW, qE = np.zeros(4), np.zeros(4)
    fn = lib().orc_muscl_face_unlimited if unlimited else lib().orc_muscl_face
    fn(order, _p(_v4(qm1)), _p(_v4(q0)), _p(_v4(q1)), _p(_v4(q2)), _p(qW), _p(qE))
    return qW, qE


def residual(cfg, q, counts=None, emap=None):
    """R(q).  emap (int64 per cell, FV): per-cell minmod outcomes accumulated
    (1 << 16*slot; slot 0 -> 0, 1 -> first argument, 2 -> second, 3 tie)."""
    q = _v4(q); r = np.zeros_like(q)
    _chk(lib().orc_residual_map(C.byref(cfg), _p(q), _p(r), _p(counts) if counts is not None else None,
                                _p(emap) if emap is not None else None))
    return r


def averages(cfg, q):
    q = _v4(q); qb = np.zeros(4 * cfg.nx * cfg.ny)
    _chk(lib().orc_averages(C.byref(cfg), _p(q), _p(qb)))
    return qb


def limit(cfg, q, counts=None):
    """Returns (limited copy, marks[int32 per element])."""
    q = np.array(q, dtype=np.float64, copy=True)
    marks = np.zeros(cfg.nx * cfg.ny, dtype=np.int32)
    _chk(lib().orc_limit(C.byref(cfg), _p(q), _p(marks), _p(counts) if counts is not None else None))
    return q, marks


def max_wave_speed(cfg, q):
    return lib().orc_max_wave_speed(C.byref(cfg), _p(_v4(q)))


def dt(cfg, q):
    return lib().orc_dt(C.byref(cfg), _p(_v4(q)))


RHS = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)


def ssprk3(q, dt, rhs):
    """One SSP-RK3 step of q' = rhs(q) through the oracle's own RK routine."""
    q = np.array(q, dtype=np.float64, copy=True)
    n = q.size

    def _cb(qp, rp, _ctx):
        qa = np.ctypeslib.as_array(qp, shape=(n,))
        ra = np.ctypeslib.as_array(rp, shape=(n,))
        ra[:] = rhs(qa.copy())

    cb = RHS(_cb)
    lib().orc_ssprk3(_p(q), n, float(dt), C.cast(cb, C.c_void_p), None, None)
    return q


def run(cfg, q, max_steps, t_end=float("inf"), t0=0.0, counts=None, emap=None):
    """March; returns (q, t, steps).  Raises on non-physical state.  emap (int64
    per element, accumulated): HO limiter runs -- the number of limiter passes
    that marked the element; FV -- per-cell minmod outcomes (see residual)."""
    q = np.array(q, dtype=np.float64, copy=True)
    t = C.c_double(t0); s = C.c_int64(0)
    if emap is not None:
        assert emap.dtype == np.int64 and emap.size == cfg.nx * cfg.ny
    st = lib().orc_run_map(C.byref(cfg), _p(q), int(max_steps), float(t_end), C.byref(t), C.byref(s),
                           _p(counts) if counts is not None else None, _p(emap) if emap is not None else None)
    if st == 4:
        raise FloatingPointError("oracle: non-physical state")
    _chk(st)
    return q, t.value, s.value


def vortex_state(cfg, x, y, t=0.0):
    q = np.zeros(4)
    lib().orc_vortex_state(C.byref(cfg), float(x), float(y), float(t), _p(q))
    return q


def shock_state(cfg, x, y):
    q = np.zeros(4)
    lib().orc_shock_state(C.byref(cfg), float(x), float(y), _p(q))
    return q


def init_case(cfg, case_id=VORTEX):
    q = np.zeros(nvalues(cfg))
    _chk(lib().orc_init_case(C.byref(cfg), case_id, _p(q)))
    return q


def point_coords(cfg):
    n = cfg.nx * cfg.ny * npts(cfg)
    X, Y = np.zeros(n), np.zeros(n)
    _chk(lib().orc_point_coords(C.byref(cfg), _p(X), _p(Y)))
    return X, Y


def fv_recon_points(cfg, q, var=0):
    """FV reconstructed solution at the 3x3 Gauss-Legendre points of every cell
    (reading R22): array [ny*nx, 3 (eta), 3 (xi)]."""
    out = np.zeros(cfg.nx * cfg.ny * 9)
    _chk(lib().orc_fv_recon_points(C.byref(cfg), _p(_v4(q)), var, _p(out)))
    return out.reshape(cfg.nx * cfg.ny, 3, 3)


def set_threads(n: int):
    """OpenMP threads of the oracle (timing only; results are bitwise those of 1)."""
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def residual_dg_quad(cfg, q, nq):
    """DG residual of Eq. (19) with nq-point Gauss-Legendre integrals (f3)."""
    r = np.zeros(nvalues(cfg))
    _chk(lib().orc_residual_dg_quad(C.byref(cfg), int(nq), _p(_v4(q)), _p(r)))
    return r


def error(cfg, q, t, case_id=VORTEX, var=0):
    l1, l2, li = C.c_double(), C.c_double(), C.c_double()
    _chk(lib().orc_error(C.byref(cfg), _p(_v4(q)), case_id, float(t), var, C.byref(l1), C.byref(l2),
                         C.byref(li)))
    return l1.value, l2.value, li.value
