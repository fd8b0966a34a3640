"""1-D reference solutions for the radial shock tube (TEST INFRASTRUCTURE ONLY).

Only tests/ may import this module; the product package never does.

The paper's discontinuous case ("Discontinuous Problem"): on
[-1,1]^2, (rho, p) = (1, 1) inside r < 0.4 and (0.125, 0.1) outside, at rest,
run to t = 0.25 and "the density is compared along the centerline, y = 0"
against Toro's reference solution (Fig. 5(b)).  The digitised
curve is not in PAPER.md, so this module recomputes that reference the way it
is defined for a radially symmetric flow: the 1-D Euler equations in r with the
geometric source term of cylindrical symmetry,

    U_t + F(U)_r = -(alpha / r) G(U),   U = (rho, rho u, E),
    F = (rho u, rho u^2 + p, u (E + p)),  G = (rho u, rho u^2, u (E + p)),

alpha = 1 (cylindrical; alpha = 0 is the planar 1-D Euler system of Eqs.
(1)-(5), restricted to one direction), p = (gamma - 1)(E - rho u^2/2),
gamma = 1.4 (R1).  It is solved on a fine radial mesh (cell-centred
finite volumes, componentwise minmod-MUSCL reconstruction, Rusanov flux as in
P:869-870, SSP-RK3 as in P:868, reflective centre, transmissive outer end).

Pins (tests/test_radial_reference.py):
  * riemann_exact(): Toro's exact Riemann solver (pressure function + Newton),
    checked against the star-state values Toro tabulates for Sod's problem
    (p* = 0.30313, u* = 0.92745, rho*_L = 0.42632, rho*_R = 0.26557) and the
    textbook closed forms of the rarefaction fan;
  * solve(alpha=0) converges to riemann_exact() (first order in L1 at the
    discontinuities) -- an independent check of the 1-D scheme;
  * solve(alpha=1): the cylindrical mass  sum rho_i r_i dr  drifts only by
    the discretisation error of the cell-centred source term, and that drift
    falls under mesh refinement (no wave leaves the mesh by t = 0.25).
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = 1.4


# --------------------------------------------------------------------------
# Exact Riemann solver for the 1-D Euler equations (Toro, Riemann Solvers and
# Numerical Methods for Fluid Dynamics, ch. 4: pressure function f_K, Newton
# iteration for p*, sampling of the self-similar solution).
# --------------------------------------------------------------------------
def _fK(p, rhoK, pK, cK, g):
    """Toro Eq. (4.6)/(4.7): f_K(p) and its derivative."""
    if p > pK:  # shock
        A = 2.0 / ((g + 1.0) * rhoK)
        B = (g - 1.0) / (g + 1.0) * pK
        s = math.sqrt(A / (p + B))
        return (p - pK) * s, s * (1.0 - 0.5 * (p - pK) / (B + p))
    # rarefaction
    r = (p / pK) ** ((g - 1.0) / (2.0 * g))
    return 2.0 * cK / (g - 1.0) * (r - 1.0), 1.0 / (rhoK * cK) * (p / pK) ** (-(g + 1.0) / (2.0 * g))


def star_state(WL, WR, g=GAMMA, tol=1e-14):
    """(p*, u*) of the Riemann problem with primitive states W = (rho, u, p)."""
    rL, uL, pL = WL
    rR, uR, pR = WR
    cL, cR = math.sqrt(g * pL / rL), math.sqrt(g * pR / rR)
    p = max(tol, 0.5 * (pL + pR) - 0.125 * (uR - uL) * (rL + rR) * (cL + cR))  # PVRS guess (Toro 4.47)
    for _ in range(100):
        fL, dL = _fK(p, rL, pL, cL, g)
        fR, dR = _fK(p, rR, pR, cR, g)
        pn = max(tol, p - (fL + fR + uR - uL) / (dL + dR))
        if abs(pn - p) <= tol * 0.5 * (pn + p):
            p = pn
            break
        p = pn
    fL, _ = _fK(p, rL, pL, cL, g)
    fR, _ = _fK(p, rR, pR, cR, g)
    return p, 0.5 * (uL + uR) + 0.5 * (fR - fL)


def riemann_exact(WL, WR, s, g=GAMMA):
    """Primitive solution (rho, u, p) at the similarity coordinates s = x/t
    (array), Toro section 4.5 sampling."""
    rL, uL, pL = WL
    rR, uR, pR = WR
    cL, cR = math.sqrt(g * pL / rL), math.sqrt(g * pR / rR)
    ps, us = star_state(WL, WR, g)
    gm = (g - 1.0) / (g + 1.0)
    out = np.empty((3, len(s)))
    for i, S in enumerate(np.asarray(s, dtype=float)):
        if S <= us:  # left of the contact
            if ps > pL:  # left shock
                SL = uL - cL * math.sqrt((g + 1) / (2 * g) * ps / pL + (g - 1) / (2 * g))
                W = (rL * (ps / pL + gm) / (gm * ps / pL + 1), us, ps) if S >= SL else (rL, uL, pL)
            else:  # left rarefaction
                SHL, STL = uL - cL, us - cL * (ps / pL) ** ((g - 1) / (2 * g))
                if S <= SHL:
                    W = (rL, uL, pL)
                elif S >= STL:
                    W = (rL * (ps / pL) ** (1 / g), us, ps)
                else:
                    f = 2 / (g + 1) + gm / cL * (uL - S)
                    W = (rL * f ** (2 / (g - 1)), 2 / (g + 1) * (cL + (g - 1) / 2 * uL + S), pL * f ** (2 * g / (g - 1)))
        else:  # right of the contact
            if ps > pR:  # right shock
                SR = uR + cR * math.sqrt((g + 1) / (2 * g) * ps / pR + (g - 1) / (2 * g))
                W = (rR * (ps / pR + gm) / (gm * ps / pR + 1), us, ps) if S <= SR else (rR, uR, pR)
            else:  # right rarefaction
                SHR, STR = uR + cR, us + cR * (ps / pR) ** ((g - 1) / (2 * g))
                if S >= SHR:
                    W = (rR, uR, pR)
                elif S <= STR:
                    W = (rR * (ps / pR) ** (1 / g), us, ps)
                else:
                    f = 2 / (g + 1) - gm / cR * (uR - S)
                    W = (rR * f ** (2 / (g - 1)), 2 / (g + 1) * (-cR + (g - 1) / 2 * uR + S), pR * f ** (2 * g / (g - 1)))
        out[:, i] = W
    return out


# --------------------------------------------------------------------------
# 1-D finite-volume solver with the geometric source term
# --------------------------------------------------------------------------
def _minmod(a, b):
    """minmod(a, b) of P:349 (0 if the signs differ or an argument is 0)."""
    return np.where((a > 0) & (b > 0), np.minimum(a, b), np.where((a < 0) & (b < 0), np.maximum(a, b), 0.0))


def _flux(U, g):
    rho, m, E = U
    u = m / rho
    p = (g - 1.0) * (E - 0.5 * m * u)
    return np.array([m, m * u + p, u * (E + p)]), np.abs(u) + np.sqrt(g * p / rho), p


def _rhs(U, r, dr, alpha, g, left):
    """-dF/dr - (alpha/r) G for the interior cells; two ghost cells per end:
    left = 'reflect' (centre r = 0: rho, E even, rho u odd) or 'copy'
    (transmissive, as the far end)."""
    n = U.shape[1]
    Ug = np.empty((3, n + 4))
    Ug[:, 2:-2] = U
    if left == "reflect":
        Ug[:, 1] = U[:, 0] * np.array([1.0, -1.0, 1.0])
        Ug[:, 0] = U[:, 1] * np.array([1.0, -1.0, 1.0])
    else:
        Ug[:, 0] = Ug[:, 1] = U[:, 0]
    Ug[:, -1] = Ug[:, -2] = U[:, -1]
    dm, dp = Ug[:, 1:-1] - Ug[:, :-2], Ug[:, 2:] - Ug[:, 1:-1]
    sig = _minmod(dm, dp)                       # cells 1 .. n+2 of Ug
    UL = Ug[:, 1:-2] + 0.5 * sig[:, :-1]        # face i+1/2 left state, faces between Ug cells 1..n+2
    UR = Ug[:, 2:-1] - 0.5 * sig[:, 1:]
    fL, aL, _ = _flux(UL, g)
    fR, aR, _ = _flux(UR, g)
    lam = np.maximum(aL, aR)
    F = 0.5 * (fL + fR) - 0.5 * lam * (UR - UL)  # n+1 faces: r_{1/2} .. r_{n+1/2}
    R = -(F[:, 1:] - F[:, :-1]) / dr
    if alpha:
        rho, m, E = U
        u = m / rho
        p = (g - 1.0) * (E - 0.5 * m * u)
        R -= alpha / r * np.array([m, m * u, u * (E + p)])
    return R


def solve(W_in, W_out, r0, t_end, alpha=1, R=1.5, n=3000, cfl=0.4, g=GAMMA, xmin=None):
    """Solve to t_end.  alpha = 1: radial problem on r in [0, R], state W_in for
    r < r0 and W_out outside (primitive (rho, u, p)).  alpha = 0: planar problem
    on [xmin, R] (xmin defaults to -R) with the initial jump at r0, transmissive
    ends.  Returns (cell centres, primitive W[3, n], steps)."""
    lo = 0.0 if alpha else (-R if xmin is None else xmin)
    dr = (R - lo) / n
    r = lo + (np.arange(n) + 0.5) * dr
    W = np.where(r < r0, np.array(W_in, dtype=float)[:, None], np.array(W_out, dtype=float)[:, None])
    U = np.array([W[0], W[0] * W[1], W[2] / (g - 1.0) + 0.5 * W[0] * W[1] ** 2])
    left = "reflect" if alpha else "copy"
    t, steps = 0.0, 0
    while t < t_end:
        _, a, _ = _flux(U, g)
        dt = min(cfl * dr / a.max(), t_end - t)
        U1 = U + dt * _rhs(U, r, dr, alpha, g, left)
        U2 = 0.75 * U + 0.25 * (U1 + dt * _rhs(U1, r, dr, alpha, g, left))
        U = U / 3.0 + 2.0 / 3.0 * (U2 + dt * _rhs(U2, r, dr, alpha, g, left))
        t += dt
        steps += 1
    rho, m, E = U
    u = m / rho
    return r, np.array([rho, u, (g - 1.0) * (E - 0.5 * m * u)]), steps


def radial_shock_density(t_end=0.25, n=3000, R=1.5):
    """Reference centreline density of the paper's case:
    rho(r, t_end) on the radial cell centres."""
    r, W, _ = solve((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), 0.4, t_end, alpha=1, R=R, n=n)
    return r, W[0]
