"""Pins of the oracle's method variants: the alternatives to the
readings Q10 (FV limiter), Q12 (limiter detection variables) and Q13 (when to
limit).  Expected values are closed forms, invariants or compositions of
already-pinned oracle parts -- never a retyped formula of the variant itself.
"""
import numpy as np
import pytest

HO = [(m, k) for m in ("cpr", "ndg", "dg", "sd") for k in (1, 2)]


# --------------------------------------------------------------------------- #
# Q10 alternative: unlimited kappa-schemes (MUSCL, P:346-351 without minmod)   #
# --------------------------------------------------------------------------- #
def test_unlimited_kappa_face_closed_forms(orc):
    ones = np.ones(4)
    q = [0.0, 3.0, 1.0, 5.0]  # an extremum at cell i = 1: the limited schemes fall back to q_i
    qs = [v * ones for v in q]
    # kappa = 0 (Fromm): q_{i+1/2}^- = q_i + (q_{i+1} - q_{i-1}) / 4, q_{i+1/2}^+ = q_{i+1} - (q_{i+2} - q_i) / 4
    qW, qE = orc.muscl_face(1, *qs, unlimited=True)
    np.testing.assert_allclose(qW, (3.0 + (1.0 - 0.0) / 4) * ones, rtol=1e-15)
    np.testing.assert_allclose(qE, (1.0 - (5.0 - 3.0) / 4) * ones, rtol=1e-15)
    # kappa = 1/3: (-q_{i-1} + 5 q_i + 2 q_{i+1}) / 6 and (2 q_i + 5 q_{i+1} - q_{i+2}) / 6
    qW, qE = orc.muscl_face(2, *qs, unlimited=True)
    np.testing.assert_allclose(qW, (-0.0 + 15.0 + 2.0) / 6 * ones, rtol=1e-15)
    np.testing.assert_allclose(qE, (6.0 + 5.0 - 5.0) / 6 * ones, rtol=1e-15)
    # the limited schemes on the same data: zero slope in cell i (first order)
    qW, _ = orc.muscl_face(1, *qs)
    np.testing.assert_allclose(qW, 3.0 * ones)


def test_unlimited_kappa_third_exact_on_quadratic_extremum(orc):
    """kappa = 1/3 reproduces the face value of any quadratic from its cell
    averages -- including at an extremum, where the limited scheme clips."""
    f = lambda x: 2.0 - 0.3 * (x - 0.6) ** 2  # noqa: E731  peak inside cell 0 / at face 0.5 region
    F = lambda x: 2.0 * x - 0.1 * (x - 0.6) ** 3  # noqa: E731  antiderivative
    avg = lambda i: F(i + 0.5) - F(i - 0.5)  # noqa: E731
    ones = np.ones(4)
    qs = [avg(i) * ones for i in range(-1, 3)]
    qW, qE = orc.muscl_face(2, *qs, unlimited=True)
    np.testing.assert_allclose(qW, f(0.5) * ones, rtol=1e-14)
    np.testing.assert_allclose(qE, f(0.5) * ones, rtol=1e-14)


@pytest.mark.parametrize("order", [1, 2])
def test_unlimited_fv_conservative_and_converges(orc, order):
    """The unlimited FV residual conserves every component on a periodic grid,
    and on the vortex its error falls under refinement at >= 2nd order."""
    cfg = orc.config(nx=12, ny=9, method="fv", k=order, fv_unlimited=1)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(cfg), seed=3, amp=1e-2)
    r = orc.residual(cfg, q).reshape(4, -1)
    for c in range(4):
        assert abs(r[c].sum()) <= 1e-12 * np.abs(r[c]).sum()
    errs = []
    for n in (32, 64):
        c2 = orc.config(nx=n, ny=n, method="fv", k=order, fv_unlimited=1, cfl=0.3)
        q, t, _ = orc.run(c2, orc.init_case(c2), 10 ** 6, t_end=1.0)
        errs.append(orc.error(c2, q, t)[1])
    assert np.log2(errs[0] / errs[1]) > 1.8


# --------------------------------------------------------------------------- #
# Q12 alternative: detection on all four conserved components                  #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("method,k", HO)
def test_all_vars_detection_sees_a_pressure_jump(orc, method, k):
    """rho constant, an O(1) energy jump inside element column 3: rho-only
    detection marks nothing; detection on every component marks that column
    (the constant neighbours are not marked), and the limited state keeps the
    averages."""
    cfg0 = orc.config(nx=8, ny=3, method=method, k=k, bc=1, box=(0.0, 8.0, 0.0, 3.0), limiter=1)
    cfg1 = orc.config(nx=8, ny=3, method=method, k=k, bc=1, box=(0.0, 8.0, 0.0, 3.0), limiter=1, limiter_all_vars=1)
    X, Y = orc.point_coords(cfg0)
    rho = np.ones_like(X)
    q = np.concatenate([rho, 0 * rho, 0 * rho, np.where(X < 3.3, 2.5, 0.25)])
    _, m0 = orc.limit(cfg0, q)
    ql, m1 = orc.limit(cfg1, q)
    assert m0.sum() == 0
    mk = m1.reshape(3, 8)
    assert mk[:, 3].all() and mk.sum() == 3
    np.testing.assert_allclose(orc.averages(cfg1, ql), orc.averages(cfg1, q), rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("method,k", HO)
def test_all_vars_marks_superset(orc, method, k):
    cfg0 = orc.config(nx=20, ny=20, method=method, k=k, bc=1, box=(-1.0, 1.0, -1.0, 1.0), limiter=1)
    cfg1 = orc.config(nx=20, ny=20, method=method, k=k, bc=1, box=(-1.0, 1.0, -1.0, 1.0), limiter=1,
                      limiter_all_vars=1)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(orc.config(nx=20, ny=20, method=method, k=k, bc=1, box=(-1.0, 1.0, -1.0, 1.0)),
                              orc.SHOCK), seed=7, amp=1e-2)
    _, m0 = orc.limit(cfg0, q)
    _, m1 = orc.limit(cfg1, q)
    assert m0.sum() > 0 and np.all(m1 >= m0) and m1.sum() >= m0.sum()


# --------------------------------------------------------------------------- #
# Q13 alternative: limit once per step (after stage 3) instead of every stage  #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("method,k", HO)
def test_limit_per_step_is_unlimited_step_then_limit(orc, method, k):
    """With a fixed dt, one per-step-limited SSP-RK3 step equals one unlimited
    step followed by one application of the (pinned) limiter; the per-stage
    variant differs on the shock tube."""
    box = (-1.0, 1.0, -1.0, 1.0)
    kw = dict(nx=16, ny=16, method=method, k=k, bc=1, box=box, dt_fixed=2e-3)
    c_step = orc.config(limiter=1, limiter_per_step=1, **kw)
    c_none = orc.config(limiter=0, **kw)
    c_stage = orc.config(limiter=1, **kw)
    q0 = orc.init_case(c_stage, orc.SHOCK)  # limited initial data
    q_step, _, _ = orc.run(c_step, q0, 1)
    q_free, _, _ = orc.run(c_none, q0, 1)
    q_ref, _ = orc.limit(c_step, q_free)
    np.testing.assert_array_equal(q_step, q_ref)
    q_stage, _, _ = orc.run(c_stage, q0, 1)
    assert np.abs(q_stage - q_step).max() > 1e-8


# --------------------------------------------------------------------------- #
# Q12 alternative: Eq. (35) slopes limited in characteristic fields           #
# --------------------------------------------------------------------------- #
def _random_states(n, seed=0):
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.2, 2.0, n)
    u, v = rng.uniform(-1.5, 1.5, n), rng.uniform(-1.5, 1.5, n)
    p = rng.uniform(0.1, 3.0, n)
    return [np.array([r, r * a, r * b, pp / 0.4 + 0.5 * r * (a * a + b * b)]) for r, a, b, pp in zip(rho, u, v, p)]


@pytest.mark.parametrize("dir", [0, 1])
def test_char_vectors_diagonalise_the_jacobian(orc, dir):
    """L R = I and L A R = diag(u_n - c, u_n, u_n, u_n + c), with A the pinned
    flux-Jacobian action."""
    cfg = orc.config()
    for q in _random_states(20, seed=dir):
        R, Lm = orc.char_vectors(cfg, dir, q)
        np.testing.assert_allclose(Lm @ R, np.eye(4), atol=1e-13)
        A = np.column_stack([orc.jacobian_apply(cfg, dir, q, e) for e in np.eye(4)])
        lam = Lm @ A @ R
        un = q[1 + dir] / q[0]
        c = np.sqrt(1.4 * orc.pressure(cfg, q) / q[0])
        np.testing.assert_allclose(lam, np.diag([un - c, un, un, un + c]), atol=1e-12 * (abs(un) + c))


@pytest.mark.parametrize("method,k", [("cpr", 1), ("dg", 2), ("sd", 1), ("ndg", 2)])
def test_characteristic_limiting_flattens_opposite_waves(orc, method, k):
    """Centre element average q0; its E neighbour differs by dx r_1 (the u-c
    acoustic wave at q0), its W neighbour by -dx r_4 (the u+c wave): every
    characteristic field has slopes of opposite sign or zero, so characteristic
    limiting rebuilds the marked element as the constant q0, while the
    componentwise limiter keeps a nonzero density slope."""
    kw = dict(nx=3, ny=3, method=method, k=k, bc=1, box=(0.0, 3.0, 0.0, 3.0), limiter=1)
    c_comp = orc.config(**kw)
    c_char = orc.config(limiter_characteristic=1, **kw)
    q0 = np.array([1.0, 0.3, -0.2, 2.6])
    R, _ = orc.char_vectors(c_char, 0, q0)
    X, Y = orc.point_coords(c_comp)
    npe = (k + 1) ** 2
    q = np.zeros((4, X.size))
    for m in range(9):
        i, j = m % 3, m // 3
        sl = slice(m * npe, (m + 1) * npe)
        st = q0.copy()
        if (i, j) == (2, 1):
            st = q0 + 1.0 * R[:, 0]
        elif (i, j) == (0, 1):
            st = q0 - 1.0 * R[:, 3]
        q[:, sl] = st[:, None]
        if (i, j) == (1, 1):  # zero-average density ramp inside the centre: it trips the detector
            xi = X[sl] - 1.5
            q[:, sl] = q0[:, None] + 0.4 * np.outer(np.array([1.0, 0.3, -0.2, 1.3]), xi)
    q = q.reshape(-1)
    qc, mc = orc.limit(c_char, q)
    qm, mm = orc.limit(c_comp, q)
    m = 4
    assert mc[m] == 1 and mm[m] == 1
    cen = qc.reshape(4, -1)[:, m * npe:(m + 1) * npe]
    np.testing.assert_allclose(cen, np.repeat(q0[:, None], npe, axis=1), rtol=1e-13, atol=1e-14)
    cen_comp = qm.reshape(4, -1)[:, m * npe:(m + 1) * npe]
    assert np.ptp(cen_comp[0]) > 0.1
