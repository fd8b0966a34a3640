"""Linear stability of the oracle's element operators (reading R9, SD flux points;
VERDICT r1 "settle SD at k >= 3").

On a periodic 1-D grid of unit elements with linear advection f = q (a = 1,
upwind Rusanov interface flux), the semi-discrete operator L of each method is
assembled column by column from the oracle's own residual (physics = 1) and its
spectrum checked against what the mathematics fixes:

* CPR, NDG, DG (all the FR/DG g_DG operator, P6-P7): the spectrum lies in the
  closed left half plane and the largest SSP-RK3 time step is the textbook
  RKDG limit: CFL 0.409 (P1) and 0.209 (P2) (Cockburn & Shu, RKDG CFL table),
  0.130 / 0.089 at P3 / P4 (computed here, no external figure);
* SD with the Chebyshev-Gauss-Lobatto flux points of reading R9 (which reproduce
  Table 3's SD P2 column): stable at P1, where every choice of 3
  flux points is {-1, 0, 1}; from P2 on the spectrum has a small positive real
  part (a weak semi-discrete growth, max Re(lambda) dx / a = 0.0028, 0.0135,
  0.027 at P2, P3, P4), and an independent numpy assembly of Eqs. (30)-(34) with
  Legendre-Gauss + end points (Huynh's g2, the provably stable choice) is stable.
  The growth is far below what the t = 1 vortex runs can see (e^(0.027 * t / dx)
  - 1 < 3 % on the 20x20 grid at P4); R9 records the consequence;
* the paper's "SD ... larger time-steps" (Table 1: SD 0.3 / 0.2 vs 0.24 /
  0.13 at P1 / P2): the largest RK3 step of the SD operator over its
  non-growing modes is 1.4-1.9 x the DG one at every order.
"""
import numpy as np
import pytest
from numpy.polynomial import legendre as L

import oracle as O


def op_1d(method, k, nx=12):
    """1-D operator of the oracle on element row 0, solution row b = 0, built from
    y-uniform unit data (the y fluxes vanish: advection velocity (1, 0))."""
    cf = O.config(nx=nx, ny=2, method=method, k=k, box=(0.0, float(nx), 0.0, 2.0), physics=1, adv=(1.0, 0.0))
    n = k + 1
    N = nx * 2 * n * n
    cols = [(i, a) for i in range(nx) for a in range(n)]
    idx = [i * n * n + a for i, a in cols]
    M = np.zeros((len(cols), len(cols)))
    for col, (i, a) in enumerate(cols):
        q = np.zeros((4, N))
        for j in range(2):
            for b in range(n):
                q[0, (j * nx + i) * n * n + b * n + a] = 1.0
        M[:, col] = O.residual(cf, q.ravel()).reshape(4, N)[0][idx]
    return M


def rk3_limit(ev, growth_ok=False):
    """largest c with |R(c lambda)| <= 1 for all eigenvalues (growth_ok: <= e^(Re c lambda)
    for the modes that grow in the semi-discretisation itself), R the SSP-RK3 polynomial"""
    lo, hi = 0.0, 3.0
    for _ in range(60):
        m = 0.5 * (lo + hi)
        z = m * ev
        bound = np.exp(np.maximum(z.real, 0.0)) * (1 + 1e-9) + 1e-12 if growth_ok else 1 + 1e-12
        if (np.abs(1 + z + z * z / 2 + z ** 3 / 6) <= bound).all():
            lo = m
        else:
            hi = m
    return lo


def _lagr(nodes, x):
    out = np.ones((len(x), len(nodes)))
    for j in range(len(nodes)):
        for m in range(len(nodes)):
            if m != j:
                out[:, j] *= (x - nodes[m]) / (nodes[j] - nodes[m])
    return out


def _dlagr(nodes, x):
    n = len(nodes)
    out = np.zeros((len(x), n))
    for j in range(n):
        for m in range(n):
            if m == j:
                continue
            t = np.ones(len(x)) / (nodes[j] - nodes[m])
            for r in range(n):
                if r not in (j, m):
                    t *= (x - nodes[r]) / (nodes[j] - nodes[r])
            out[:, j] += t
    return out


def sd_numpy(k, flux_nodes, nel=12):
    """Eqs. (30)-(34) for q_t + q_x = 0 on unit elements: interpolate to the flux
    nodes, upwind value at the left end, differentiate the flux polynomial at the
    Gauss-Legendre solution points."""
    n = k + 1
    xs = L.leggauss(n)[0]
    I = _lagr(xs, flux_nodes)        # (n+1) x n
    D = _dlagr(flux_nodes, xs)       # n x (n+1)
    M = np.zeros((nel * n, nel * n))
    for e in range(nel):
        for a in range(n):
            for r in range(n + 1):
                src, row = ((e - 1) % nel, I[n]) if r == 0 else (e, I[r])
                M[e * n + a, src * n:(src + 1) * n] -= 2.0 * D[a, r] * row
    return M


def cgl(m):
    return -np.cos(np.pi * np.arange(m) / (m - 1))


def gauss_ends(m):
    return np.concatenate([[-1.0], L.leggauss(m - 2)[0], [1.0]])


@pytest.mark.parametrize("method", ["cpr", "ndg", "dg"])
def test_dg_family_spectrum_and_rk3_limit(method):
    lim = {1: 0.409, 2: 0.209, 3: 0.130, 4: 0.0898}
    for k in (1, 2, 3, 4):
        ev = np.linalg.eigvals(op_1d(method, k, nx=24))
        assert ev.real.max() <= 1e-12
        c = rk3_limit(ev)
        assert abs(c - lim[k]) <= 0.004 * lim[k] + 1e-3, (k, c)


def test_sd_cgl_flux_points_weak_growth_and_independent_assembly():
    growth = {1: 0.0, 2: 0.0028, 3: 0.0135, 4: 0.0272}
    for k in (1, 2, 3, 4):
        M = op_1d("sd", k)
        # the oracle's SD operator IS the definition with CGL flux points (R9)
        np.testing.assert_allclose(M, sd_numpy(k, cgl(k + 2)), rtol=0, atol=1e-12 * np.abs(M).max())
        g = np.linalg.eigvals(M).real.max()
        if k == 1:
            assert g <= 1e-12
        else:
            assert 0.0 < g and abs(g - growth[k]) <= 0.05 * growth[k], (k, g)
        # Legendre-Gauss + end points: the stable alternative
        assert np.linalg.eigvals(sd_numpy(k, gauss_ends(k + 2))).real.max() <= 1e-12


def test_sd_takes_larger_time_steps_than_cpr():
    """P:964 / Table 1 (SD 0.3 vs CPR 0.24 at P1; 0.2 vs 0.13 at P2): the SD RK3
    step over its non-growing modes exceeds the CPR one by 1.4-1.9x at every order,
    and Table 1's P2 ratio 0.2 / 0.13 = 1.54 lies between the CGL (1.65) and the
    Legendre-Gauss + ends (1.53) flux-point readings."""
    for k in (1, 2, 3, 4):
        c_cpr = rk3_limit(np.linalg.eigvals(op_1d("cpr", k)))
        c_sd = rk3_limit(np.linalg.eigvals(op_1d("sd", k)), growth_ok=True)
        assert 1.4 <= c_sd / c_cpr <= 1.9, (k, c_sd, c_cpr)
    c2 = rk3_limit(np.linalg.eigvals(op_1d("cpr", 2)))
    r_cgl = rk3_limit(np.linalg.eigvals(op_1d("sd", 2)), growth_ok=True) / c2
    r_ge = rk3_limit(np.linalg.eigvals(sd_numpy(2, gauss_ends(4)))) / c2
    assert r_ge <= 0.2 / 0.13 + 0.02 and r_cgl >= 0.2 / 0.13 - 0.02
