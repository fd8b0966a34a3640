"""Pins for the paper's discontinuous case (Fig. 5(b)):
the centreline density at t = 0.25 is compared with a radially symmetric 1-D
reference (oracle/radial1d.py), which is itself pinned to Toro's exact Riemann
solution (Sod's problem: the planar reduction of the same data).

What a plausible mistake in the 2-D oracle's shock workflow (initial radius,
transmissive boundary, gamma, a flux sign, the limiter) would do: move or
deform the shock / contact / rarefaction by O(1) cells, so the centreline L1
difference would stop halving under mesh refinement."""
import math

import numpy as np
import pytest

import oracle
from oracle import radial1d as R1

SOD_L, SOD_R = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)


def test_exact_riemann_sod_star_state():
    # Toro, Riemann Solvers..., Table 4.3, test 1 (Sod): p* = 0.30313,
    # u* = 0.92745, rho*_L = 0.42632, rho*_R = 0.26557 (5 printed digits)
    ps, us = R1.star_state(SOD_L, SOD_R)
    assert abs(ps - 0.30313) < 5e-6 and abs(us - 0.92745) < 5e-6
    W = R1.riemann_exact(SOD_L, SOD_R, np.array([us - 1e-9, us + 1e-9]))
    assert abs(W[0, 0] - 0.42632) < 5e-6 and abs(W[0, 1] - 0.26557) < 5e-6
    assert np.allclose(W[2], ps, rtol=0, atol=1e-14) and np.allclose(W[1], us, rtol=0, atol=1e-14)


def test_exact_riemann_closed_forms():
    g = 1.4
    cL = math.sqrt(g)
    ps, us = R1.star_state(SOD_L, SOD_R)
    # undisturbed states outside the fan / shock
    W = R1.riemann_exact(SOD_L, SOD_R, np.array([-cL - 1e-3, 5.0]))
    assert np.allclose(W[:, 0], SOD_L) and np.allclose(W[:, 1], SOD_R)
    # inside the left rarefaction: u - c = s and the Riemann invariant u + 2c/(g-1) = 2 cL/(g-1)
    s = np.linspace(-cL + 1e-6, us - math.sqrt(g * ps / 0.42632) - 1e-3, 7)
    W = R1.riemann_exact(SOD_L, SOD_R, s)
    c = np.sqrt(g * W[2] / W[0])
    assert np.allclose(W[1] - c, s, atol=1e-12)
    assert np.allclose(W[1] + 2 * c / (g - 1), 2 * cL / (g - 1), atol=1e-12)
    assert np.allclose(W[2] / W[0] ** g, 1.0, atol=1e-12)  # isentropic fan
    # Rankine-Hugoniot mass balance across the right shock
    rR, pR = SOD_R[0], SOD_R[2]
    cR = math.sqrt(g * pR / rR)
    SR = cR * math.sqrt((g + 1) / (2 * g) * ps / pR + (g - 1) / (2 * g))
    rs = R1.riemann_exact(SOD_L, SOD_R, np.array([SR - 1e-9]))[0, 0]
    assert abs(rs * (us - SR) - rR * (0.0 - SR)) < 1e-12


def test_planar_solver_converges_to_exact():
    """alpha = 0 is Sod's problem: the 1-D scheme's L1 error falls ~first order."""
    errs = []
    for n in (400, 800):
        x, W, _ = R1.solve(SOD_L, SOD_R, 0.0, 0.2, alpha=0, R=0.5, n=n)
        errs.append(np.abs(W - R1.riemann_exact(SOD_L, SOD_R, x / 0.2)).mean(axis=1))
    assert np.all(errs[1] < 0.7 * errs[0])
    assert np.all(errs[1] < 4e-3)


def test_radial_mass_drift_converges():
    drifts = []
    for n in (500, 1000):
        r, W, _ = R1.solve((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), 0.4, 0.25, alpha=1, R=1.5, n=n)
        m0 = (np.where(r < 0.4, 1.0, 0.125) * r).sum()
        drifts.append(abs((W[0] * r).sum() - m0) / m0)
    assert drifts[1] < 0.7 * drifts[0] and drifts[1] < 3e-4


@pytest.fixture(scope="module")
def reference():
    return R1.radial_shock_density(t_end=0.25, n=3000)


def _centreline_l1(method, k, n, cfl, ref):
    oc = oracle.config(nx=n, ny=n, method=method, k=k, bc=oracle.TRANSMISSIVE, box=(-1.0, 1.0, -1.0, 1.0),
                       cfl=cfl, limiter=1)
    q, t, _ = oracle.run(oc, oracle.init_case(oc, oracle.SHOCK), 10**6, t_end=0.25)
    assert t == 0.25
    X, Y = oracle.point_coords(oc)
    rho = q.reshape(4, -1)[0]
    sel = np.abs(Y) <= 1.0 / n + 1e-12  # points within half a cell / on the element edge at y = 0
    r, rho_ref = ref
    x, d = X[sel], rho[sel]
    diff = d - np.interp(np.abs(x), r, rho_ref)
    # the shock: the outermost x where the density exceeds the ambient 0.125 by 0.05
    xs = np.abs(x[d > 0.175]).max()
    return np.abs(diff).mean(), xs


# (method, k, coarse n, CFL of Table 4, bound on the fine-grid L1)
CASES = [("fv", 1, 100, 0.58, 0.013), ("cpr", 1, 50, 0.2, 0.025), ("dg", 1, 50, 0.22, 0.025),
         ("sd", 1, 50, 0.3, 0.025)]


@pytest.mark.parametrize("method,k,n,cfl,bound", CASES)
def test_centreline_converges_to_radial_reference(reference, method, k, n, cfl, bound):
    l1c, _ = _centreline_l1(method, k, n, cfl, reference)
    l1f, xs = _centreline_l1(method, k, 2 * n, cfl, reference)
    assert l1f < 0.65 * l1c, (l1c, l1f)
    assert l1f < bound, l1f
    r, rho_ref = reference
    xs_ref = r[rho_ref > 0.175].max()
    assert abs(xs - xs_ref) < 3 * 2.0 / (2 * n), (xs, xs_ref)
