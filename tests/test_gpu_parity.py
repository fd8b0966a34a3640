"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same
seeded inputs (BASELINE.json north_star: relative L-inf <= 1e-10 per conserved
variable after 100 fp64 steps; branch decisions identical).

Tolerances ("parity bar"): one residual evaluation agrees to 1e-12
relative (a few hundred fp64 operations with different FMA contraction and
summation order); 100 SSP-RK3 steps (300 stages) to the north_star's 1e-10.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HO = [(m, k) for m in ("cpr", "ndg", "dg", "sd") for k in (1, 2, 3, 4)]
ALL = HO + [("fv", 1), ("fv", 2)]
CFL = {("cpr", 1): 0.24, ("ndg", 1): 0.24, ("dg", 1): 0.24, ("sd", 1): 0.3,
       ("cpr", 2): 0.13, ("ndg", 2): 0.13, ("dg", 2): 0.13, ("sd", 2): 0.2,
       ("cpr", 3): 0.08, ("ndg", 3): 0.08, ("dg", 3): 0.08, ("sd", 3): 0.1,
       ("cpr", 4): 0.05, ("ndg", 4): 0.05, ("dg", 4): 0.05, ("sd", 4): 0.06,
       ("fv", 1): 0.37, ("fv", 2): 0.37}


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1709_01619_b200 as P
    from paper_1709_01619_b200 import build
    build.build()
    P.load()
    return P


def pair(orc, P, nx, ny, method, k, bc=0, box=(-5.0, 5.0, -5.0, 5.0), cfl=None, limiter=0, record=0,
         cpr_chain_rule=1):
    cfl = CFL[(method, k)] if cfl is None else cfl
    oc = orc.config(nx=nx, ny=ny, method=method, k=k, bc=bc, box=box, cfl=cfl, limiter=limiter,
                    cpr_chain_rule=cpr_chain_rule)
    gc = P.make_config(nx, ny, method=method, k=k, bc=bc, box=box, cfl=cfl, limiter=limiter,
                       cpr_chain_rule=cpr_chain_rule, record_decisions=record)
    return oc, P.Solver(gc)


def rel_linf(a, b):
    """max over components of L-inf(a - b) / L-inf(b); an identically zero
    component of b (e.g. momenta of the quiescent shock-tube start) must match
    to 1e-300, i.e. exactly up to denormals."""
    a, b = a.reshape(4, -1), b.reshape(4, -1)
    return max(np.abs(a[c] - b[c]).max() / max(np.abs(b[c]).max(), 1e-300) for c in range(4))


def rel_linf_res(a, b):
    """residuals: per component, relative to the largest |R| of that component (or
    to the largest |R| overall where a component is identically ~0)."""
    a, b = a.reshape(4, -1), b.reshape(4, -1)
    big = np.abs(b).max()
    return max(np.abs(a[c] - b[c]).max() / max(np.abs(b[c]).max(), 1e-3 * big) for c in range(4))


@pytest.mark.parametrize("method,k", ALL)
@pytest.mark.parametrize("bc", [0, 1])
def test_residual_parity(orc, P, method, k, bc):
    import torch
    # 19 x 13: ragged against every tile shape, several tiles in each direction
    nx, ny = (19, 13) if method != "fv" else (45, 21)
    oc, s = pair(orc, P, nx, ny, method, k, bc=bc)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=11 + k, amp=1e-2)
    r_orc = orc.residual(oc, q)
    r_gpu = s.residual(torch.from_numpy(q).cuda()).cpu().numpy()
    assert rel_linf_res(r_gpu, r_orc) < 1e-12


@pytest.mark.parametrize("method,k", ALL)
def test_100_steps_parity(orc, P, method, k):
    """north_star gate: 100 SSP-RK3 steps, rel L-inf <= 1e-10 per variable."""
    nx, ny = (10, 10) if method != "fv" else (40, 40)
    oc, s = pair(orc, P, nx, ny, method, k)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=3, amp=1e-3)
    s.set_state(q)
    t_g, n_g = s.step(100)
    q_o, t_o, n_o = orc.run(oc, q, 100)
    assert n_g == n_o == 100
    assert abs(t_g - t_o) <= 1e-12 * t_o
    assert rel_linf(s.get_state(), q_o) <= 1e-10


def test_config1_cpr_p1_vortex(orc, P):
    """BASELINE config 1: CPR P1 vortex 10x10 periodic, 100 steps, from init_case."""
    oc, s = pair(orc, P, 10, 10, "cpr", 1)
    s.init_case(P.VORTEX)
    q0 = s.get_state()
    q0_o = orc.init_case(oc)
    assert rel_linf(q0, q0_o) <= 1e-14
    s.step(100)
    q_o, t_o, _ = orc.run(oc, q0_o, 100)
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    e_g = s.error(P.VORTEX, 0)
    e_o = orc.error(oc, q_o, t_o)
    np.testing.assert_allclose(e_g, e_o, rtol=1e-9)


@pytest.mark.parametrize("method,k", [("cpr", 1), ("dg", 2), ("sd", 1), ("ndg", 2), ("cpr", 3)])
def test_paper_table_point_on_gpu(orc, P, method, k):
    """The GPU reproduces a Table 2/3 entry end to end (init, march to t = 1, error)."""
    cfl = {1: 0.24, 2: 0.14}.get(k, 0.08) if method != "sd" else {1: 0.3, 2: 0.2}[k]
    oc, s = pair(orc, P, 20, 20, method, k, cfl=cfl)
    s.init_case(P.VORTEX)
    t, _ = s.step(10 ** 6, 1.0)
    assert t == 1.0
    q_o, t_o, _ = orc.run(oc, orc.init_case(oc), 10 ** 6, 1.0)
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    np.testing.assert_allclose(s.error(P.VORTEX, 0), orc.error(oc, q_o, t_o), rtol=1e-8)


@pytest.mark.parametrize("method,k", ALL)
def test_dt_parity(orc, P, method, k):
    oc, s = pair(orc, P, 12, 9, method, k)
    s.init_case(P.VORTEX)
    assert s.compute_dt() == pytest.approx(orc.dt(oc, orc.init_case(oc)), rel=1e-14)


@pytest.mark.parametrize("method,k,cfl", [("cpr", 1, 0.2), ("cpr", 2, 0.1), ("ndg", 1, 0.2), ("dg", 1, 0.2),
                                          ("dg", 2, 0.08), ("sd", 1, 0.27), ("sd", 2, 0.18), ("cpr", 3, 0.06),
                                          ("sd", 4, 0.05), ("dg", 4, 0.03)])
def test_shock_limiter_parity(orc, P, method, k, cfl):
    """Radial shock tube, transmissive, limiter after every stage: state parity and
    identical trouble-cell marks (decision counters)."""
    box = (-1.0, 1.0, -1.0, 1.0)
    oc, s = pair(orc, P, 24, 24, method, k, bc=1, box=box, cfl=cfl, limiter=1, record=1)
    s.init_case(P.SHOCK)
    q0 = orc.init_case(oc, orc.SHOCK)
    assert rel_linf(s.get_state(), q0) <= 1e-14
    cnt = np.zeros(8, dtype=np.int64)
    s.set_state(q0)
    t_g, n_g = s.step(40, 0.25)
    q_o, t_o, n_o = orc.run(oc, q0, 40, 0.25, counts=cnt)
    assert n_g == n_o
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    assert s.decisions()[0] == cnt[0] > 0


@pytest.mark.parametrize("k,cfl", [(1, 0.58), (2, 0.54)])
def test_fv_shock_decisions(orc, P, k, cfl):
    box = (-1.0, 1.0, -1.0, 1.0)
    oc, s = pair(orc, P, 48, 48, "fv", k, bc=1, box=box, cfl=cfl, record=1)
    q0 = orc.init_case(oc, orc.SHOCK)
    s.set_state(q0)
    t_g, n_g = s.step(30, 0.25)
    cnt = np.zeros(8, dtype=np.int64)
    q_o, t_o, n_o = orc.run(oc, q0, 30, 0.25, counts=cnt)
    assert n_g == n_o
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    d = s.decisions()
    # non-tie decisions identical; ties (within 1e-12 of the switch point) reported
    np.testing.assert_array_equal(d[1:4], cnt[1:4])
    assert d[4] == cnt[4]


@pytest.mark.parametrize("method,k", [("cpr", 2), ("dg", 3), ("sd", 2), ("ndg", 1)])
def test_limiter_single_application(orc, P, method, k):
    import torch  # noqa: F401
    box = (-1.0, 1.0, -1.0, 1.0)
    oc, s = pair(orc, P, 17, 15, method, k, bc=1, box=box, limiter=1, record=1)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc, orc.SHOCK), seed=5, amp=1e-2)
    s.set_state(q)
    s.limit()
    ql, marks = orc.limit(oc, q)
    assert rel_linf(s.get_state(), ql) <= 1e-14
    assert s.decisions()[0] == marks.sum()


def test_nonphysical_is_reported(orc, P):
    oc, s = pair(orc, P, 8, 8, "cpr", 1)
    q = orc.init_case(oc)
    n = q.size // 4
    q[3 * n + 5] = -1.0  # negative energy -> negative pressure
    s.set_state(q)
    with pytest.raises(P.NonPhysicalState):
        s.step(5)


def test_time_clipping(orc, P):
    oc, s = pair(orc, P, 10, 10, "cpr", 2)
    s.init_case(P.VORTEX)
    t, n = s.step(1000, 0.3)
    _, t_o, n_o = orc.run(oc, orc.init_case(oc), 1000, 0.3)
    assert t == t_o == pytest.approx(0.3, abs=1e-15) and n == n_o
    t2, n2 = s.step(5, 0.3)  # already there: no-op
    assert n2 == 0 and t2 == t


def test_determinism_bitwise(orc, P):
    oc, s = pair(orc, P, 33, 17, "dg", 2)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=9, amp=1e-2)
    out = []
    for _ in range(2):
        s.set_state(q)
        s.step(20)
        out.append(s.get_state())
    np.testing.assert_array_equal(out[0], out[1])


@pytest.mark.parametrize("method,k,n", [("cpr", 3, 4096), ("cpr", 2, 1024), ("fv", 1, 2048), ("ndg", 3, 2048),
                                          ("dg", 3, 2048), ("sd", 3, 2048), ("cpr", 1, 2048), ("cpr", 4, 1024),
                                          ("dg", 4, 1024), ("sd", 2, 1024), ("fv", 2, 2048), ("sd", 4, 1024),
                                          ("ndg", 4, 1024), ("ndg", 2, 1024), ("dg", 2, 1024)])
def test_full_size_tiled_patch(orc, P, method, k, n):
    """At BASELINE sizes, in the bench's launch configuration (CPR P3 at 4096^2 is
    the north-star bench launch itself): a state that repeats a seeded 16x16-element
    patch must give the oracle's residual of that patch on its own periodic 16x16
    grid, at every element of the big grid (a property that holds at any size; the
    oracle only ever sees the small patch).  Tiling and comparison on the device."""
    import torch
    pn = 16
    box_small = (-5.0, -5.0 + 10.0 * pn / n, -5.0, -5.0 + 10.0 * pn / n)  # same element size
    oc = orc.config(nx=pn, ny=pn, method=method, k=k, box=box_small)
    from paper_1709_01619_b200.inputs import perturb
    qp = perturb(orc.init_case(oc), seed=21, amp=1e-2)
    r_p = orc.residual(oc, qp)
    npe = 1 if method == "fv" else (k + 1) ** 2
    # tile the patch on the device: [c][J][I][p] -> [c][j][i][p]
    patch = torch.from_numpy(qp.reshape(4, pn, 1, pn, npe)).cuda()
    big = patch.repeat(1, n // pn, 1, n // pn, 1).reshape(4, n // pn, pn, n // pn, pn, npe)
    big = big.permute(0, 1, 2, 3, 4, 5).reshape(-1).contiguous()
    s = P.Solver(P.make_config(n, n, method=method, k=k, cfl=CFL[(method, k)]))
    r_big = s.residual(big).view(4, n // pn, pn, n // pn, pn, npe)
    del big
    ref = torch.from_numpy(r_p.reshape(4, 1, pn, 1, pn, npe)).cuda()
    scale = torch.maximum(ref.reshape(4, -1).abs().amax(1), 1e-3 * ref.abs().max())
    err = max(float((r_big[c] - ref[c]).abs().max() / scale[c]) for c in range(4))
    assert err < 1e-12
    s.close()


def test_full_size_free_stream_and_mass(orc, P):
    """4096^2 CPR P3 (north-star size): a uniform state stays uniform to round-off
    after 3 steps (free-stream preservation), in the bench's launch config."""
    import torch
    n = 4096
    s = P.Solver(P.make_config(n, n, method="cpr", k=3, cfl=0.08))
    npts = n * n * 16
    rho, u, v, p = 1.0, 1.0, 0.5, 1.0
    q = torch.empty(4 * npts, dtype=torch.float64, device="cuda")
    q[:npts] = rho
    q[npts:2 * npts] = rho * u
    q[2 * npts:3 * npts] = rho * v
    q[3 * npts:] = p / 0.4 + 0.5 * rho * (u * u + v * v)
    s.set_state(q)
    s.step(3)
    out = torch.empty_like(q)
    s.get_state(out)
    assert float((out - q).abs().max()) < 1e-12
    s.close()


@pytest.mark.parametrize("method,k,n,cfl", [("cpr", 1, 1024, 0.2), ("cpr", 2, 1024, 0.1), ("dg", 1, 1024, 0.2),
                                            ("sd", 1, 1024, 0.27), ("ndg", 3, 512, 0.06)])
def test_full_size_tiled_patch_limited_step(orc, P, method, k, n, cfl):
    """Limiter path at bench sizes (fused element averages in the stage kernels,
    k_limit, the lambda pass): one limited SSP-RK3 step of a periodic state that
    repeats a seeded 16x16 patch equals the oracle's step of the patch on its own
    periodic grid, tiled (dt agrees: same element size, same max wave speed)."""
    import torch
    pn = 16
    box_small = (-5.0, -5.0 + 10.0 * pn / n, -5.0, -5.0 + 10.0 * pn / n)
    oc = orc.config(nx=pn, ny=pn, method=method, k=k, box=box_small, cfl=cfl, limiter=1)
    from paper_1709_01619_b200.inputs import perturb
    X, Y = orc.point_coords(oc)
    inner = (X - box_small[0]) ** 2 + (Y - box_small[2]) ** 2 < (0.3 * (box_small[1] - box_small[0])) ** 2
    rho = np.where(inner, 1.0, 0.125)  # a shock-tube disc in the patch (and jumps at its tiled edges)
    qp = perturb(np.concatenate([rho, 0 * rho, 0 * rho, np.where(inner, 2.5, 0.25)]), seed=23, amp=1e-2)
    cnt = np.zeros(8, dtype=np.int64)
    q1, _, _ = orc.run(oc, qp, 1, counts=cnt)
    assert cnt[0] > 0
    npe = (k + 1) ** 2
    big = np.tile(qp.reshape(4, pn, pn, npe), (1, n // pn, n // pn, 1)).reshape(-1)
    s = P.Solver(P.make_config(n, n, method=method, k=k, cfl=cfl, limiter=1, record_decisions=1))
    s.set_state(torch.from_numpy(big).cuda())
    s.step(1)
    out = s.get_state().reshape(4, n // pn, pn, n // pn, pn, npe)
    ref = q1.reshape(4, 1, pn, 1, pn, npe)
    err = np.abs(out - ref).max(axis=(1, 2, 3, 4, 5)) / np.maximum(np.abs(ref).reshape(4, -1).max(1), 1e-300)
    assert err.max() < 1e-10
    assert s.decisions()[0] == cnt[0] * (n // pn) ** 2
    s.close()


@pytest.mark.parametrize("method,k,n", [("cpr", 3, 2048), ("dg", 3, 2048), ("sd", 4, 1024), ("ndg", 4, 1024),
                                          ("sd", 2, 1024), ("fv", 2, 2048)])
def test_full_size_tiled_patch_step(orc, P, method, k, n):
    """Every stage variant at bench sizes (stage 1 without q^n, stage 2 with it,
    stage 3 with the dt wave speed / non-physical epilogue; the fused dt): two
    SSP-RK3 steps of a periodic state that repeats a seeded 16x16 patch equal the
    oracle's two steps of the patch on its own periodic grid, tiled (dt agrees:
    same element size, same max wave speed)."""
    import torch
    pn = 16
    box_small = (-5.0, -5.0 + 10.0 * pn / n, -5.0, -5.0 + 10.0 * pn / n)
    cfl = CFL[(method, k)]
    oc = orc.config(nx=pn, ny=pn, method=method, k=k, box=box_small, cfl=cfl)
    from paper_1709_01619_b200.inputs import perturb
    qp = perturb(orc.init_case(oc), seed=29, amp=1e-3)
    q2, t2, n2 = orc.run(oc, qp, 2)
    npe = 1 if method == "fv" else (k + 1) ** 2
    patch = torch.from_numpy(qp.reshape(4, pn, 1, pn, npe)).cuda()
    big = patch.repeat(1, n // pn, 1, n // pn, 1).reshape(-1).contiguous()
    s = P.Solver(P.make_config(n, n, method=method, k=k, cfl=cfl, box=(-5.0, 5.0, -5.0, 5.0)))
    s.set_state(big)
    del big
    t, steps = s.step(2)
    assert steps == n2 == 2 and abs(t - t2) <= 1e-12 * t2
    out = torch.empty(4 * n * n * npe, dtype=torch.float64, device="cuda")
    s.get_state(out)
    out = out.view(4, n // pn, pn, n // pn, pn, npe)
    ref = torch.from_numpy(q2.reshape(4, 1, pn, 1, pn, npe)).cuda()
    err = max(float((out[c] - ref[c]).abs().max() / ref[c].abs().max().clamp_min(1e-300)) for c in range(4))
    assert err <= 1e-10
    s.close()


@pytest.mark.parametrize("method,k", [("cpr", 3), ("ndg", 3), ("dg", 3), ("sd", 3), ("sd", 4), ("ndg", 4),
                                      ("cpr", 2), ("fv", 2)])
def test_multi_row_march_transmissive(orc, P, method, k):
    """Transmissive x and y (the mirrored end faces, the missing ghost rows of the
    strip's first and last marches, the q^n ring's first and last rows) on grids
    where every CTA marches several element rows and strips are ragged: 10
    SSP-RK3 steps against the oracle on seeded perturbed input."""
    nx, ny = (200, 163) if method != "fv" else (700, 523)
    oc = orc.config(nx=nx, ny=ny, method=method, k=k, cfl=CFL[(method, k)], bc=1)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=43, amp=1e-3)
    s = P.Solver(P.make_config(nx, ny, method=method, k=k, cfl=CFL[(method, k)], bc=P.TRANSMISSIVE))
    s.set_state(q)
    _, n_g = s.step(10)
    q_o, _, n_o = orc.run(oc, q, 10)
    assert n_g == n_o == 10
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    s.close()


@pytest.mark.parametrize("method,k", [("cpr", 3), ("ndg", 3), ("dg", 2), ("sd", 3), ("fv", 2)])
def test_multi_row_march_parity(orc, P, method, k):
    """Grids big enough that each CTA marches several element rows (and strips are
    ragged): 10 SSP-RK3 steps against the oracle on seeded perturbed input."""
    nx, ny = (200, 163) if method != "fv" else (700, 523)
    oc = orc.config(nx=nx, ny=ny, method=method, k=k, cfl=CFL[(method, k)])
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=41, amp=1e-3)
    s = P.Solver(P.make_config(nx, ny, method=method, k=k, cfl=CFL[(method, k)]))
    s.set_state(q)
    _, n_g = s.step(10)
    q_o, _, n_o = orc.run(oc, q, 10)
    assert n_g == n_o == 10
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    s.close()


# --------------------------------------------------------------------------- #
# Round 2: the north_star gate as written -- 100 steps with the limiter on /   #
# 100 FV shock steps, decisions identical element by element      #
# --------------------------------------------------------------------------- #
LIMITED_GATE = [("cpr", 1, 0.2), ("cpr", 2, 0.1), ("ndg", 1, 0.2), ("ndg", 2, 0.1), ("dg", 1, 0.2),
                ("dg", 2, 0.08), ("sd", 1, 0.27), ("sd", 2, 0.18), ("cpr", 3, 0.06)]


@pytest.mark.parametrize("method,k,cfl", LIMITED_GATE)
def test_limiter_gate_100_steps(orc, P, method, k, cfl):
    """Radial shock tube on 32^2, transmissive, minmod detection +
    limiting after every stage: 100 SSP-RK3 steps (no t_end), the
    state within 1e-10 (north_star) and, after EVERY step, the per-element count
    of limiter passes that marked the element identical to the oracle's."""
    box = (-1.0, 1.0, -1.0, 1.0)
    n = 32
    oc, s = pair(orc, P, n, n, method, k, bc=1, box=box, cfl=cfl, limiter=1, record=1)
    q = orc.init_case(oc, orc.SHOCK)
    s.set_state(q)
    em = np.zeros(n * n, dtype=np.int64)
    t = 0.0
    for step in range(100):
        q, t, n_o = orc.run(oc, q, 1, t0=t, emap=em)
        t_g, n_g = s.step(1)
        assert n_o == n_g == 1
        assert abs(t_g - t) <= 1e-12 * t
        g = s.decision_map()
        bad = np.flatnonzero(g != em)
        assert bad.size == 0, (step, bad[:10], g[bad[:10]], em[bad[:10]])
    assert em.sum() > 0 and s.decisions()[0] == em.sum()
    assert rel_linf(s.get_state(), q) <= 1e-10
    s.close()


def _unpack(m):
    return np.stack([(m >> (16 * sl)) & 0xFFFF for sl in range(4)])


@pytest.mark.parametrize("k,cfl", [(1, 0.58), (2, 0.54)])
@pytest.mark.parametrize("bc", [0, 1])
def test_fv_decisions_100_steps(orc, P, k, cfl, bc):
    """FV MUSCL-2/3 + minmod on the shock tube, 100 steps: state within
    1e-10 and, per cell, the minmod outcomes of its own slopes (-> 0 / first /
    second argument) identical to the oracle's; ties (an argument or their
    difference within 1e-12 of the switch point) counted separately and equal."""
    box = (-1.0, 1.0, -1.0, 1.0)
    n = 48
    oc, s = pair(orc, P, n, n, "fv", k, bc=bc, box=box, cfl=cfl, record=1)
    q0 = orc.init_case(oc, orc.SHOCK)
    s.set_state(q0)
    em = np.zeros(n * n, dtype=np.int64)
    cnt = np.zeros(8, dtype=np.int64)
    q_o, t_o, n_o = orc.run(oc, q0, 100, counts=cnt, emap=em)
    t_g, n_g = s.step(100)
    assert n_g == n_o == 100
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    g = s.decision_map()
    ug, uo = _unpack(g), _unpack(em)
    bad = np.flatnonzero((ug != uo).any(axis=0))
    assert bad.size == 0, (bad[:10], ug[:, bad[:10]], uo[:, bad[:10]])
    np.testing.assert_array_equal(s.decisions()[1:5], cnt[1:5])
    assert uo[1:3].sum() > 0 and uo[0].sum() > 0  # every outcome occurs


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("bc", [0, 1])
def test_fv_rough_data_residual(orc, P, k, bc):
    """FV residual on strongly perturbed data (20 % cell-to-cell noise), where every
    minmod branch occurs, including MUSCL-3's beta-bounded arguments (|D+| > 4|D-|)."""
    import torch
    nx, ny = 45, 21
    oc, s = pair(orc, P, nx, ny, "fv", k, bc=bc, record=1)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=31 + k, amp=0.2)
    em = np.zeros(nx * ny, dtype=np.int64)
    cnt = np.zeros(8, dtype=np.int64)
    r_orc = orc.residual(oc, q, counts=cnt, emap=em)
    s.set_state(q)  # resets the map
    r_gpu = s.residual(torch.from_numpy(q).cuda()).cpu().numpy()
    assert rel_linf_res(r_gpu, r_orc) < 1e-12
    np.testing.assert_array_equal(_unpack(s.decision_map()), _unpack(em))
    np.testing.assert_array_equal(s.decisions()[1:5], cnt[1:5])


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("nx", [64, 65, 130, 131, 257])
def test_fv_strip_widths(orc, P, k, bc, nx):
    """FV stage kernel across its x-strip raggedness (64-cell warp strips, 4 per
    CTA): a full strip, odd / even ragged last strips, several CTAs, odd nx (the
    8-B path) and even nx (the 16-B pair path); residual and per-cell decision
    maps against the oracle on rough data, then 20 steps."""
    import torch
    ny = 9
    oc, s = pair(orc, P, nx, ny, "fv", k, bc=bc, record=1)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=5 + nx, amp=0.2)
    em = np.zeros(nx * ny, dtype=np.int64)
    cnt = np.zeros(8, dtype=np.int64)
    r_orc = orc.residual(oc, q, counts=cnt, emap=em)
    s.set_state(q)
    r_gpu = s.residual(torch.from_numpy(q).cuda()).cpu().numpy()
    assert rel_linf_res(r_gpu, r_orc) < 1e-12
    np.testing.assert_array_equal(_unpack(s.decision_map()), _unpack(em))
    np.testing.assert_array_equal(s.decisions()[1:5], cnt[1:5])
    q1 = perturb(orc.init_case(oc), seed=6 + nx, amp=1e-3)
    s.set_state(q1)
    s.step(20)
    q_o, _, _ = orc.run(oc, q1, 20)
    assert rel_linf(s.get_state(), q_o) <= 1e-10


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("case", [0, 1])
@pytest.mark.parametrize("bc", [0, 1])
def test_fv_init_case_parity(orc, P, k, case, bc):
    """FV initial data: 8x8 Gauss-Legendre cell averages of the closed-form case
    (vortex P:897-913 / shock tube P:1043-1047), GPU k_init vs the oracle."""
    box = (-5.0, 5.0, -5.0, 5.0) if case == 0 else (-1.0, 1.0, -1.0, 1.0)
    oc, s = pair(orc, P, 37, 23, "fv", k, bc=bc, box=box)
    s.init_case(case)
    np.testing.assert_allclose(s.get_state(), orc.init_case(oc, case), rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("method,k", [("cpr", 1), ("ndg", 2), ("dg", 3), ("sd", 4), ("cpr", 4), ("sd", 1),
                                      ("fv", 1), ("fv", 2)])
@pytest.mark.parametrize("var", [0, 1, 2, 3])
def test_error_parity_all_norms(orc, P, method, k, var):
    """hom2d_error: L1, L2 and Linf of every conserved component against the exact
    vortex at t != 0 (reading R8), GPU vs oracle on a seeded
    perturbed state."""
    nx, ny = (13, 11) if method != "fv" else (40, 30)
    oc, s = pair(orc, P, nx, ny, method, k)
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=7 + var, amp=1e-3)
    t0 = 0.37
    s.set_state(q, t0)
    np.testing.assert_allclose(s.error(P.VORTEX, var), orc.error(oc, q, t0, var=var), rtol=1e-12)


@pytest.mark.parametrize("k,unl", [(1, 0), (2, 0), (2, 1), (1, 1)])
@pytest.mark.parametrize("var", [0, 1, 2, 3])
@pytest.mark.parametrize("self_x", [0, 1, 2])
def test_fv_recon_error_parity(orc, P, monkeypatch, k, unl, var, self_x):
    """f4 (reading R22): hom2d_error with fv_error_recon -- the FV solution
    reconstructed from the scheme's MUSCL face states, compared with the exact
    vortex at the 3x3 Gauss points of every cell -- GPU vs oracle, all norms and
    variables, limited and unlimited; self_x = 1 reads the y-neighbour rows through
    the strip ghost buffers (HOM2D_SELF_EXCHANGE)."""
    if self_x:
        monkeypatch.setenv("HOM2D_SELF_EXCHANGE", str(self_x))
    nx, ny = 41, 30
    oc = orc.config(nx=nx, ny=ny, method="fv", k=k, cfl=0.37, fv_unlimited=unl, fv_error_recon=1)
    s = P.Solver(P.make_config(nx, ny, method="fv", k=k, cfl=0.37, fv_unlimited=unl, fv_error_recon=1))
    from paper_1709_01619_b200.inputs import perturb
    q = perturb(orc.init_case(oc), seed=17 + var, amp=1e-2)
    t0 = 0.61
    s.set_state(q, t0)
    np.testing.assert_allclose(s.error(P.VORTEX, var), orc.error(oc, q, t0, var=var), rtol=1e-12)
    s.close()
