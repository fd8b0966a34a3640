"""Pins of the oracle's DG with (k+2)-point Gauss-Legendre over-integration (SURVEY
8(f) f3; SPEC's alternative to the collocated integrals of Eq. (20), P:255-260;
Eq. (19)).

* with nq = n points the quadrature form IS the collocation DG (C6) to rounding;
* linear advection (f = a q): the integrands are polynomials of degree <= 2k, so
  every rule with nq >= n integrates them exactly and over-integration changes
  nothing;
* an independent numpy evaluation of Eq. (19) -- q_h interpolated to the
  (k+2)^2 Gauss points and to k+2 points along each edge, the Euler fluxes there
  (the oracle's pinned flux / Rusanov exports), integrals by the (k+2)-point rule,
  exact diagonal mass -- on a 3 x 2 periodic grid;
* conservation (periodic: sum_m sum_ab w_a w_b R_ab = 0) and free stream;
* Tables 2-3's DG column is reproduced by both forms (the paper cannot tell them
  apart on the smooth vortex: they differ by < 0.2 % there).
"""
import itertools

import numpy as np
import pytest
from numpy.polynomial import legendre as L

import oracle as O
from paper_1709_01619_b200.inputs import perturb


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_collocation_rule_is_the_dg_residual(k):
    cf = O.config(nx=5, ny=4, method="dg", k=k)
    q = perturb(O.init_case(cf), seed=3, amp=1e-2)
    r0 = O.residual(cf, q)
    np.testing.assert_allclose(O.residual_dg_quad(cf, q, k + 1), r0, rtol=0, atol=1e-13 * np.abs(r0).max())
    # and the switch selects the (k+2)-point rule
    cfo = O.config(nx=5, ny=4, method="dg", k=k, dg_overintegrate=1)
    np.testing.assert_array_equal(O.residual(cfo, q), O.residual_dg_quad(cf, q, k + 2))
    assert np.abs(O.residual(cfo, q) - r0).max() > 1e-6 * np.abs(r0).max()  # a different operator on Euler


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_linear_advection_is_integrated_exactly(k):
    cf = O.config(nx=4, ny=3, method="dg", k=k, physics=1, adv=(1.0, -0.6))
    cfo = O.config(nx=4, ny=3, method="dg", k=k, physics=1, adv=(1.0, -0.6), dg_overintegrate=1)
    q = perturb(O.init_case(O.config(nx=4, ny=3, method="dg", k=k)), seed=5, amp=0.3)
    r0 = O.residual(cf, q)
    np.testing.assert_allclose(O.residual(cfo, q), r0, rtol=0, atol=1e-13 * np.abs(r0).max())


def _lag(nodes, x):
    return np.array([np.prod([(x - nodes[m]) / (nodes[j] - nodes[m]) for m in range(len(nodes)) if m != j])
                     for j in range(len(nodes))])


def _dlag(nodes, x):
    n = len(nodes)
    out = np.zeros(n)
    for j in range(n):
        for m in range(n):
            if m != j:
                out[j] += np.prod([(x - nodes[r]) / (nodes[j] - nodes[r]) for r in range(n) if r not in (j, m)]) / (
                    nodes[j] - nodes[m])
    return out


@pytest.mark.parametrize("k", [1, 2, 3])
def test_independent_weak_form(k):
    n, nq = k + 1, k + 2
    nx, ny = 3, 2
    box = (-5.0, 1.0, -2.0, 3.0)
    cf = O.config(nx=nx, ny=ny, method="dg", k=k, box=box, dg_overintegrate=1)
    q = perturb(O.init_case(cf), 9, 5e-2)
    Q = q.reshape(4, ny, nx, n, n)
    xi, w = L.leggauss(n)
    z, W = L.leggauss(nq)
    dx, dy = (box[1] - box[0]) / nx, (box[3] - box[2]) / ny

    def qh(j, i, x, y):  # q_h of element (j, i) at reference point (x, y)
        return np.einsum("cba,b,a->c", Q[:, j % ny, i % nx], _lag(xi, y), _lag(xi, x))

    R = np.zeros_like(Q)
    for j, i in itertools.product(range(ny), range(nx)):
        for b, a in itertools.product(range(n), range(n)):
            vx = np.zeros(4)
            vy = np.zeros(4)
            for s, r in itertools.product(range(nq), range(nq)):
                qq = qh(j, i, z[r], z[s])
                vx += W[r] * W[s] * O.flux(cf, 0, qq) * _dlag(xi, z[r])[a] * _lag(xi, z[s])[b]
                vy += W[r] * W[s] * O.flux(cf, 1, qq) * _lag(xi, z[r])[a] * _dlag(xi, z[s])[b]
            sx = np.zeros(4)
            sy = np.zeros(4)
            for t in range(nq):
                FE = O.rusanov(cf, 0, qh(j, i, 1.0, z[t]), qh(j, i + 1, -1.0, z[t]))
                FW = O.rusanov(cf, 0, qh(j, i - 1, 1.0, z[t]), qh(j, i, -1.0, z[t]))
                FN = O.rusanov(cf, 1, qh(j, i, z[t], 1.0), qh(j + 1, i, z[t], -1.0))
                FS = O.rusanov(cf, 1, qh(j - 1, i, z[t], 1.0), qh(j, i, z[t], -1.0))
                sx += W[t] * (_lag(xi, 1.0)[a] * FE - _lag(xi, -1.0)[a] * FW) * _lag(xi, z[t])[b]
                sy += W[t] * (_lag(xi, 1.0)[b] * FN - _lag(xi, -1.0)[b] * FS) * _lag(xi, z[t])[a]
            R[:, j, i, b, a] = ((2 / dx) * (vx - sx) + (2 / dy) * (vy - sy)) / (w[a] * w[b])
    r_orc = O.residual(cf, q).reshape(R.shape)
    np.testing.assert_allclose(r_orc, R, rtol=0, atol=1e-11 * np.abs(R).max())


@pytest.mark.parametrize("k", [1, 3])
def test_conservation_and_free_stream(k):
    n = k + 1
    cf = O.config(nx=6, ny=5, method="dg", k=k, dg_overintegrate=1)
    q = perturb(O.init_case(cf), seed=2, amp=1e-2)
    r = O.residual(cf, q).reshape(4, -1, n, n)
    _, w = L.leggauss(n)
    tot = np.einsum("cmba,b,a->c", r, w, w)
    assert np.abs(tot).max() <= 1e-12 * np.abs(r).max() * r.shape[1]
    u = np.zeros((4, 30 * n * n))
    u[0], u[1], u[2], u[3] = 1.3, 0.4, -0.7, 4.0
    ru = O.residual(cf, u.ravel())
    assert np.abs(ru).max() <= 1e-12


@pytest.mark.parametrize("k,nx,cfl,l2", [(1, 20, 0.24, 1.65e-3), (2, 20, 0.14, 2.24e-4)])
def test_tables_dg_column_under_overintegration(k, nx, cfl, l2):
    """P:989-1039, DG column (tests/golden/paper_tables_2_3.txt): over-integration
    reproduces the printed 20x20 entries as well as collocation does."""
    errs = []
    for oi in (0, 1):
        cf = O.config(nx=nx, ny=nx, method="dg", k=k, cfl=cfl, dg_overintegrate=oi)
        q2, t, _ = O.run(cf, O.init_case(cf), 10 ** 6, 1.0)
        errs.append(O.error(cf, q2, t)[1])
    assert all(abs(e / l2 - 1) < 6e-3 for e in errs), errs
    assert abs(errs[1] / errs[0] - 1) < 2e-3
