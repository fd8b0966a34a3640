"""P16 brute force: the oracle's tensor-product residuals against dense 2-D
assemblies written from the paper's matrix definitions.

* NDG: M, S, D = M^{-1} S, face mass M^A and lift L = M^{-1} M^A of Eqs.
  (25)-(29), assembled over the full n^2-point nodal basis with
  exact (high-order Gauss) integration, no tensor-product factorisation.
* DG: Algorithm 4: dense volume loop over all n^2 points (stiffness
  S_x, S_y), surface loop over all 4n face points (integration matrix I), and
  M^{-1}, from the weak form Eq. (19).
* SD: Eqs. (30)-(34): the flux polynomial through ALL (n+1) x n flux
  points of each direction differentiated as a numpy polynomial.

Only pinned physics primitives (orc.flux, orc.rusanov: test_oracle_pins P1) and
numpy polynomials are used; the element operators here come from numpy, not the
oracle.
"""
import itertools

import numpy as np
import pytest
from numpy.polynomial import Polynomial as Poly
from numpy.polynomial import legendre as L


def gll(n):
    inner = np.sort(L.legroots(L.legder(np.eye(n)[n - 1]))) if n > 2 else np.array([])
    return np.concatenate([[-1.0], inner, [1.0]])


def cheb_lobatto(n1):
    return -np.cos(np.pi * np.arange(n1) / (n1 - 1))


def lagrange_polys(x):
    out = []
    for j in range(len(x)):
        others = np.delete(x, j)
        p = Poly.fromroots(others)
        out.append(p / p(x[j]))
    return out


GQ_X, GQ_W = L.leggauss(12)


def integ(f):
    return float(np.sum(GQ_W * f(GQ_X)))


def elem_traces_and_neighbours(orc, cfg, q, xi):
    n = len(xi)
    nx, ny = cfg.nx, cfg.ny
    Q = q.reshape(4, ny, nx, n, n)  # [c][j][i][b][a]
    ell = lagrange_polys(xi)
    eL = np.array([p(-1.0) for p in ell])
    eR = np.array([p(1.0) for p in ell])
    return Q, eL, eR


def face_fluxes(orc, cfg, Q, eL, eR):
    """F^W,F^E [j,i,b,c], G^S,G^N [j,i,a,c] from interpolated traces (exact at
    GLL edge nodes) and the pinned Rusanov flux, periodic."""
    _, ny, nx, n, _ = Q.shape
    W = np.einsum("cjiba,a->jibc", Q, eL)
    E = np.einsum("cjiba,a->jibc", Q, eR)
    S = np.einsum("cjiba,b->jiac", Q, eL)
    N = np.einsum("cjiba,b->jiac", Q, eR)
    FW, FE, GS, GN = (np.zeros((ny, nx, n, 4)) for _ in range(4))
    for j, i, t in itertools.product(range(ny), range(nx), range(n)):
        FW[j, i, t] = orc.rusanov(cfg, 0, E[j, (i - 1) % nx, t], W[j, i, t])
        FE[j, i, t] = orc.rusanov(cfg, 0, E[j, i, t], W[j, (i + 1) % nx, t])
        GS[j, i, t] = orc.rusanov(cfg, 1, N[(j - 1) % ny, i, t], S[j, i, t])
        GN[j, i, t] = orc.rusanov(cfg, 1, N[j, i, t], S[(j + 1) % ny, i, t])
    return FW, FE, GS, GN


def pointwise_flux(orc, cfg, Q, d):
    _, ny, nx, n, _ = Q.shape
    out = np.zeros_like(Q)
    for j, i, b, a in itertools.product(range(ny), range(nx), range(n), range(n)):
        out[:, j, i, b, a] = orc.flux(cfg, d, Q[:, j, i, b, a])
    return out


def basis2d(xi):
    """phi_p(xi, eta) = l_a(xi) l_b(eta), p = b*n + a; returns callables."""
    ell = lagrange_polys(xi)
    dell = [p.deriv() for p in ell]
    n = len(xi)
    idx = [(a, b) for b in range(n) for a in range(n)]
    return ell, dell, idx


def mass_stiffness(xi):
    ell, dell, idx = basis2d(xi)
    n2 = len(idx)
    M = np.zeros((n2, n2))
    Sx = np.zeros((n2, n2))   # Sx[i,j] = int phi_i d(phi_j)/dxi
    Sy = np.zeros((n2, n2))
    for p, (a, b) in enumerate(idx):
        for r, (c, d) in enumerate(idx):
            mx = integ(lambda x: ell[a](x) * ell[c](x))
            my = integ(lambda x: ell[b](x) * ell[d](x))
            M[p, r] = mx * my
            Sx[p, r] = integ(lambda x: ell[a](x) * dell[c](x)) * my
            Sy[p, r] = mx * integ(lambda x: ell[b](x) * dell[d](x))
    return M, Sx, Sy


@pytest.mark.parametrize("k", [1, 2])
def test_ndg_dense_matrices(orc, k):
    n = k + 1
    cfg = orc.config(nx=3, ny=2, method="ndg", k=k, box=(-5.0, 1.0, -2.0, 3.0))
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(cfg), 7, 5e-2)
    xi = gll(n)
    Q, eL, eR = elem_traces_and_neighbours(orc, cfg, q, xi)
    FW, FE, GS, GN = face_fluxes(orc, cfg, Q, eL, eR)
    f = pointwise_flux(orc, cfg, Q, 0)
    g = pointwise_flux(orc, cfg, Q, 1)
    M, Sx, Sy = mass_stiffness(xi)
    Dx, Dy = np.linalg.solve(M, Sx), np.linalg.solve(M, Sy)        # Eq. (27)
    ell, _, idx = basis2d(xi)
    # face mass M^A on each face: int_face phi_i phi_j dS over the face nodes j
    MA = {}
    for face in ("W", "E", "S", "N"):
        A = np.zeros((n * n, n))
        for p, (a, b) in enumerate(idx):
            for t in range(n):
                if face in ("W", "E"):
                    xe = -1.0 if face == "W" else 1.0
                    A[p, t] = ell[a](xe) * integ(lambda y: ell[b](y) * ell[t](y))
                else:
                    ye = -1.0 if face == "S" else 1.0
                    A[p, t] = ell[b](ye) * integ(lambda x: ell[a](x) * ell[t](x))
        MA[face] = np.linalg.solve(M, A)                               # L = M^{-1} M^A
    dx, dy = 6.0 / 3, 5.0 / 2
    R = np.zeros_like(Q)
    for j, i in itertools.product(range(2), range(3)):
        for c in range(4):
            fv = f[c, j, i].ravel()
            gv = g[c, j, i].ravel()
            res = -(2 / dx) * Dx @ fv - (2 / dy) * Dy @ gv
            # F.n - F_com on each face (outward normals), Eq. (29)
            res += (2 / dx) * MA["E"] @ (f[c, j, i][:, n - 1] - FE[j, i, :, c])
            res += (2 / dx) * MA["W"] @ (-f[c, j, i][:, 0] + FW[j, i, :, c])
            res += (2 / dy) * MA["N"] @ (g[c, j, i][n - 1, :] - GN[j, i, :, c])
            res += (2 / dy) * MA["S"] @ (-g[c, j, i][0, :] + GS[j, i, :, c])
            R[c, j, i] = res.reshape(n, n)
    r_orc = orc.residual(cfg, q).reshape(R.shape)
    np.testing.assert_allclose(r_orc, R, rtol=0, atol=1e-12 * np.abs(R).max())


@pytest.mark.parametrize("k", [1, 2])
def test_dg_dense_algorithm4(orc, k):
    n = k + 1
    cfg = orc.config(nx=3, ny=2, method="dg", k=k, box=(-5.0, 1.0, -2.0, 3.0))
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(cfg), 8, 5e-2)
    xi, w = L.leggauss(n)
    Q, eL, eR = elem_traces_and_neighbours(orc, cfg, q, xi)
    FW, FE, GS, GN = face_fluxes(orc, cfg, Q, eL, eR)
    f = pointwise_flux(orc, cfg, Q, 0)
    g = pointwise_flux(orc, cfg, Q, 1)
    M, Sx, Sy = mass_stiffness(xi)
    ell, _, idx = basis2d(xi)
    # weak form: stiffness acting on the flux interpolant = int d(phi_i) phi_j
    Kx, Ky = Sx.T, Sy.T
    # surface integration matrix I over the 4n face points (GL points on each face)
    I = np.zeros((n * n, 4 * n))
    for p, (a, b) in enumerate(idx):
        for t in range(n):
            I[p, 0 * n + t] = -ell[a](-1.0) * w[t] * (ell[b](xi[t]))   # W, n = -x
            I[p, 1 * n + t] = ell[a](1.0) * w[t] * (ell[b](xi[t]))     # E
            I[p, 2 * n + t] = -ell[b](-1.0) * w[t] * (ell[a](xi[t]))   # S
            I[p, 3 * n + t] = ell[b](1.0) * w[t] * (ell[a](xi[t]))     # N
    dx, dy = 6.0 / 3, 5.0 / 2
    Minv = np.linalg.inv(M)
    R = np.zeros_like(Q)
    for j, i in itertools.product(range(2), range(3)):
        for c in range(4):
            vol = (2 / dx) * Kx @ f[c, j, i].ravel() + (2 / dy) * Ky @ g[c, j, i].ravel()
            fn = np.concatenate([FW[j, i, :, c] * (2 / dx), FE[j, i, :, c] * (2 / dx),
                                 GS[j, i, :, c] * (2 / dy), GN[j, i, :, c] * (2 / dy)])
            R[c, j, i] = (Minv @ (vol - I @ fn)).reshape(n, n)
    r_orc = orc.residual(cfg, q).reshape(R.shape)
    np.testing.assert_allclose(r_orc, R, rtol=0, atol=1e-12 * np.abs(R).max())


@pytest.mark.parametrize("k", [1, 2, 3])
def test_sd_definition(orc, k):
    """Eqs. (30)-(34): per x-line, the flux polynomial of degree k+1 through the
    n+1 flux points (Chebyshev-Gauss-Lobatto, reading R9) -- interior values
    f(q interpolated), end values Rusanov with the neighbour -- differentiated
    exactly at the GL solution points."""
    n = k + 1
    cfg = orc.config(nx=3, ny=2, method="sd", k=k, box=(-5.0, 1.0, -2.0, 3.0))
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(cfg), 9, 5e-2)
    xi, _ = L.leggauss(n)
    xf = cheb_lobatto(n + 1)
    ell = lagrange_polys(xi)
    lam = lagrange_polys(xf)
    Q = q.reshape(4, 2, 3, n, n)
    dx, dy = 6.0 / 3, 5.0 / 2

    def line(j, i, d, t):   # solution values along line t in direction d, [c][pt]
        return Q[:, j, i, t, :] if d == 0 else Q[:, j, i, :, t]

    def qf(vals, x):
        return np.array([sum(vals[c, a] * ell[a](x) for a in range(n)) for c in range(4)])

    R = np.zeros_like(Q)
    for j, i in itertools.product(range(2), range(3)):
        for d in (0, 1):
            for t in range(n):
                own = line(j, i, d, t)
                lo = line(j, (i - 1) % 3, d, t) if d == 0 else line((j - 1) % 2, i, d, t)
                hi = line(j, (i + 1) % 3, d, t) if d == 0 else line((j + 1) % 2, i, d, t)
                phi = np.zeros((n + 1, 4))
                for r in range(1, n):
                    phi[r] = orc.flux(cfg, d, qf(own, xf[r]))
                phi[0] = orc.rusanov(cfg, d, qf(lo, 1.0), qf(own, -1.0))
                phi[n] = orc.rusanov(cfg, d, qf(own, 1.0), qf(hi, -1.0))
                for c in range(4):
                    poly = sum(phi[r, c] * lam[r] for r in range(n + 1)).deriv()
                    vals = -(2 / (dx if d == 0 else dy)) * poly(xi)
                    if d == 0:
                        R[c, j, i, t, :] += vals
                    else:
                        R[c, j, i, :, t] += vals
    r_orc = orc.residual(cfg, q).reshape(R.shape)
    np.testing.assert_allclose(r_orc, R, rtol=0, atol=1e-11 * np.abs(R).max())
