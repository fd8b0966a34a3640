"""Pins of the oracle's FV reconstructed-solution error (P:879-880:
"For P^2 FV, the error was computed by reconstructing the solution along element
faces, and then using a quadrature rule to compute an averaged solution";
reading R22 in DESIGN.md).

What fixes it without the oracle itself:
* exactness: cell averages of a (monotone) quadratic -- MUSCL-3's face states are
  then the quadratic's face values (kappa = 1/3), so the reconstructed
  solution IS the quadratic at every Gauss point (1-D sum form x^2 + y^2); the
  same with linear data for MUSCL-2 and for the unlimited kappa-schemes;
* mean preservation: 3-point Gauss quadrature of the reconstructed cell solution
  returns the cell average (the quadratic's (3s^2-1) mode has zero mean);
* the face values themselves: the reconstructed solution extrapolated to s = +-1
  equals the oracle's muscl_face states (checked through orc_muscl_face);
* order of accuracy on the smooth vortex at t = 0 (the error of representing the
  exact cell averages): MUSCL-2 slope 2, MUSCL-3 above 2 (limited at extrema);
* closed forms of L1 / L2 / Linf for a state whose reconstruction is known.
"""
import numpy as np
import pytest

import oracle as O

XG, WG = np.polynomial.legendre.leggauss(3)


def _avg_quad(x0, x1, c2, c1, c0):
    """exact average over [x0, x1] of c0 + c1 x + c2 x^2"""
    return c0 + c1 * (x0 + x1) / 2 + c2 * (x1 ** 3 - x0 ** 3) / (3 * (x1 - x0))


def _quad_state(nx, ny, dx, dy, coef):
    a, b, c, d, e = coef
    ax = np.array([_avg_quad(i * dx, (i + 1) * dx, c, b, 0.0) for i in range(nx)])
    ay = np.array([_avg_quad(j * dy, (j + 1) * dy, e, d, 0.0) for j in range(ny)])
    q = np.zeros((4, ny * nx))
    q[0] = (a + ay[:, None] + ax[None, :]).ravel()
    q[1], q[2], q[3] = 0.1, -0.05, 5.0
    return q.ravel()


@pytest.mark.parametrize("k,unl,coef", [
    (1, 0, (2.0, 0.5, 0.0, -0.4, 0.0)),      # MUSCL-2: linear data
    (2, 0, (2.0, 0.5, 0.3, -0.4, 0.1)),      # MUSCL-3: monotone quadratic (limiter inactive)
    (2, 1, (2.0, 0.5, -0.9, -0.4, 0.7)),     # unlimited kappa = 1/3: any quadratic
    (1, 1, (1.0, -0.7, 0.0, 0.2, 0.0)),      # unlimited kappa = 0: linear
])
def test_recon_exact_on_quadratics(k, unl, coef):
    nx, ny, L = 12, 10, 1.2
    dx, dy = L / nx, 1.0 / ny
    cf = O.config(nx=nx, ny=ny, method="fv", k=k, bc=1, box=(0.0, L, 0.0, 1.0), fv_unlimited=unl)
    r = O.fv_recon_points(cf, _quad_state(nx, ny, dx, dy, coef), 0)
    a, b, c, d, e = coef
    err = 0.0
    for j in range(2, ny - 2):      # transmissive ghosts copy the boundary cell: stay 2 cells inside
        for i in range(2, nx - 2):
            x = (i + 0.5) * dx + 0.5 * dx * XG[None, :]
            y = (j + 0.5) * dy + 0.5 * dy * XG[:, None]
            err = max(err, np.abs(r[j * nx + i] - (a + b * x + c * x * x + d * y + e * y * y)).max())
    assert err < 1e-13


def test_recon_preserves_the_average_and_hits_the_face_states():
    """3-point Gauss quadrature of the cell's reconstructed solution = the cell value;
    the x-quadratic through the Gauss values, extrapolated to s = +-1, gives the
    MUSCL-3 face states of P:346-351 (orc_muscl_face) on rough data."""
    from paper_1709_01619_b200.inputs import perturb
    nx = ny = 9
    for k in (1, 2):
        cf = O.config(nx=nx, ny=ny, method="fv", k=k, bc=0)
        q = perturb(O.init_case(cf), seed=4, amp=0.2)
        for var in range(4):
            r = O.fv_recon_points(cf, q, var)
            qv = q.reshape(4, -1)[var]
            avg = np.einsum("mba,b,a->m", r, WG / 2, WG / 2)
            np.testing.assert_allclose(avg, qv, rtol=0, atol=1e-13 * np.abs(qv).max())
            # the cell's solution has the form qbar + al xi + be (3 xi^2 - 1) + ga eta
            # + de (3 eta^2 - 1): fit it through the 9 Gauss values (exact), then
            # its x-face values qbar -+ al + 2 be at one interior cell (i, j) = (4, 5)
            i, j = 4, 5
            m = j * nx + i
            X, Y = np.meshgrid(XG, XG)  # [b, a]
            A = np.stack([np.ones(9), X.ravel(), 3 * X.ravel() ** 2 - 1, Y.ravel(), 3 * Y.ravel() ** 2 - 1], 1)
            cfit, res, *_ = np.linalg.lstsq(A, r[m].ravel(), rcond=None)
            assert np.abs(A @ cfit - r[m].ravel()).max() <= 1e-13 * np.abs(r[m]).max()
            lo_x = cfit[0] - cfit[1] + 2 * cfit[2]
            hi_x = cfit[0] + cfit[1] + 2 * cfit[2]
            s = [q.reshape(4, -1)[:, j * nx + ((i + t) % nx)].copy() for t in (-2, -1, 0, 1, 2)]
            _, qE = O.muscl_face(k, s[0], s[1], s[2], s[3])
            qW, _ = O.muscl_face(k, s[1], s[2], s[3], s[4])
            assert abs(lo_x - qE[var]) <= 1e-12 * abs(qE[var]) + 1e-15
            assert abs(hi_x - qW[var]) <= 1e-12 * abs(qW[var]) + 1e-15


@pytest.mark.parametrize("k,lo,hi", [(1, 1.9, 2.1), (2, 2.2, 3.1)])
def test_recon_error_order_on_the_vortex(k, lo, hi):
    """t = 0, exact cell averages: the error is the reconstruction's, O(h^2) for the
    piecewise-linear MUSCL-2 and above that for MUSCL-3 (3rd order away from the
    extrema the minmod flattens)."""
    e = []
    for n in (40, 80):
        cf = O.config(nx=n, ny=n, method="fv", k=k, fv_error_recon=1)
        e.append(O.error(cf, O.init_case(cf), 0.0)[1])
    slope = np.log2(e[0] / e[1])
    assert lo <= slope <= hi, slope
    # the plain convention (cell value vs exact average) is exactly 0 at t = 0
    cf0 = O.config(nx=40, ny=40, method="fv", k=k)
    assert O.error(cf0, O.init_case(cf0), 0.0) == (0.0, 0.0, 0.0)


def test_recon_error_norms_closed_form():
    """A uniform state q = (rho0, ...) reconstructs to rho0 everywhere, so the error
    is the exact vortex density's deviation from rho0 at the 3x3 Gauss points of
    every cell: L1 = sum w|d| / Ne, L2 = sqrt(sum w d^2 / Ne), Linf = max|d|,
    computed here from the closed-form vortex directly."""
    n = 16
    cf = O.config(nx=n, ny=n, method="fv", k=2, fv_error_recon=1)
    q = np.zeros((4, n * n))
    q[0], q[1], q[2], q[3] = 1.1, 1.1, 0.0, 3.0
    t = 0.3
    l1, l2, li = O.error(cf, q.ravel(), t)
    g, eps = 1.4, 5.0
    h = 10.0 / n
    s1 = s2 = mx = 0.0
    for j in range(n):
        for i in range(n):
            for b in range(3):
                for a in range(3):
                    x = -5 + (i + 0.5) * h + 0.5 * h * XG[a] - t
                    y = -5 + (j + 0.5) * h + 0.5 * h * XG[b]
                    x = x - 10 * np.floor((x + 5) / 10)
                    T = 1 - (g - 1) * eps ** 2 / (8 * g * np.pi ** 2) * np.exp(1 - x * x - y * y)
                    d = 1.1 - T ** (1 / (g - 1))
                    w = WG[a] * WG[b] / 4
                    s1 += w * abs(d)
                    s2 += w * d * d
                    mx = max(mx, abs(d))
    assert abs(l1 - s1 / n ** 2) <= 1e-13 * l1
    assert abs(l2 - np.sqrt(s2 / n ** 2)) <= 1e-13 * l2
    assert abs(li - mx) <= 1e-14
