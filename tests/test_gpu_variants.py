"""GPU parity of the method variants against the oracle: the
unlimited FV kappa-schemes (Q10), limiter detection on all components (Q12),
limiting once per step (Q13).  Same bars as tests/test_gpu_parity.py."""
import numpy as np
import pytest

from test_gpu_parity import rel_linf, rel_linf_res

pytestmark = pytest.mark.gpu


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


def pair(orc, P, nx, ny, method, k, cfl, bc=0, box=(-5.0, 5.0, -5.0, 5.0), **kw):
    oc = orc.config(nx=nx, ny=ny, method=method, k=k, bc=bc, box=box, cfl=cfl, **kw)
    gc = P.make_config(nx, ny, method=method, k=k, bc=bc, box=box, cfl=cfl, record_decisions=1, **kw)
    return oc, P.Solver(gc)


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("bc", [0, 1])
def test_fv_unlimited_residual(orc, P, k, bc):
    import torch
    from paper_1709_01619_b200.inputs import perturb
    oc, s = pair(orc, P, 45, 21, "fv", k, 0.3, bc=bc, fv_unlimited=1)
    q = perturb(orc.init_case(oc), seed=21 + k, amp=1e-2)
    r_gpu = s.residual(torch.from_numpy(q).cuda()).cpu().numpy()
    assert rel_linf_res(r_gpu, orc.residual(oc, q)) < 1e-12
    assert s.decisions()[1:5].sum() == 0  # no minmod on this path


@pytest.mark.parametrize("k", [1, 2])
def test_fv_unlimited_100_steps(orc, P, k):
    from paper_1709_01619_b200.inputs import perturb
    oc, s = pair(orc, P, 40, 40, "fv", k, 0.3, fv_unlimited=1)
    q = perturb(orc.init_case(oc), seed=4, amp=1e-3)
    s.set_state(q)
    _, n_g = s.step(100)
    q_o, _, n_o = orc.run(oc, q, 100)
    assert n_g == n_o == 100
    assert rel_linf(s.get_state(), q_o) <= 1e-10


SHOCK_CASES = [("cpr", 1, 0.2), ("cpr", 2, 0.1), ("ndg", 1, 0.2), ("dg", 1, 0.2), ("dg", 2, 0.08),
               ("sd", 1, 0.27), ("sd", 2, 0.18), ("cpr", 3, 0.06)]


@pytest.mark.parametrize("method,k,cfl", SHOCK_CASES)
@pytest.mark.parametrize("variant", ["limiter_per_step", "limiter_all_vars", "limiter_characteristic"])
def test_shock_limiter_variants(orc, P, method, k, cfl, variant):
    """Radial shock tube, transmissive, 40 steps: state parity and identical
    trouble-cell mark counts for each limiter variant."""
    box = (-1.0, 1.0, -1.0, 1.0)
    oc, s = pair(orc, P, 24, 24, method, k, cfl, bc=1, box=box, limiter=1, **{variant: 1})
    q0 = orc.init_case(oc, orc.SHOCK)
    cnt = np.zeros(8, dtype=np.int64)
    s.set_state(q0)
    try:
        q_o, _, n_o = orc.run(oc, q0, 40, 0.25, counts=cnt)
    except FloatingPointError:  # e.g. P3 limited only once per step: both sides must flag it
        with pytest.raises(P.NonPhysicalState):
            s.step(40, 0.25)
        return
    _, n_g = s.step(40, 0.25)
    assert n_g == n_o
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    assert s.decisions()[0] == cnt[0] > 0


@pytest.mark.parametrize("method,k,limiter", [("cpr", 3, 0), ("dg", 2, 0), ("fv", 1, 0), ("sd", 1, 1)])
@pytest.mark.parametrize("after,min_batch", [("256", "64"), ("0", "1")])
def test_graph_replay_bitwise_equals_eager(orc, P, monkeypatch, method, k, limiter, after, min_batch):
    """hom2d_step replays cached CUDA graphs of 2^i steps on long single-GPU runs
    (HOM2D_GRAPH_AFTER / HOM2D_GRAPH_MIN_BATCH move the switch-over: after 256
    eager steps in 64-step batches, or from the first step in any batch); the
    state, t and step count equal the eager launch sequence bitwise, including
    the t_end-clipped last batch."""
    monkeypatch.setenv("HOM2D_GRAPH_AFTER", after)
    monkeypatch.setenv("HOM2D_GRAPH_MIN_BATCH", min_batch)
    box, bc, case, cfl = ((-1.0, 1.0, -1.0, 1.0), 1, P.SHOCK, 0.2) if limiter else ((-5.0, 5.0, -5.0, 5.0), 0,
                                                                                   P.VORTEX, 0.08)
    out = []
    for no_graph in ("0", "1"):
        monkeypatch.setenv("HOM2D_NO_GRAPH", no_graph)
        s = P.Solver(P.make_config(20, 16, method=method, k=k, bc=bc, box=box, cfl=cfl, limiter=limiter))
        s.init_case(case)
        t1, n1 = s.step(400)                     # 256 eager steps, 2 graph batches, 16 eager
        t2, n2 = s.step(10 ** 6, t1 + 0.3)       # clipped at t_end
        out.append((s.get_state(), t1, n1, t2, n2, s.launch_count()))
        s.close()
    (qa, *ra), (qb, *rb) = out
    np.testing.assert_array_equal(qa, qb)
    assert ra == rb


@pytest.mark.parametrize("method,k,limiter", [("cpr", 3, 0), ("sd", 2, 0), ("fv", 2, 0), ("dg", 1, 1)])
def test_programmatic_launch_bitwise_equals_plain(orc, P, monkeypatch, method, k, limiter):
    """Programmatic dependent launches (each kernel waits on griddepcontrol.wait)
    give bitwise the state of ordinary stream-ordered launches."""
    box, bc, case, cfl = ((-1.0, 1.0, -1.0, 1.0), 1, P.SHOCK, 0.2) if limiter else ((-5.0, 5.0, -5.0, 5.0), 0,
                                                                                   P.VORTEX, 0.08)
    out = []
    for no_pdl in ("0", "1"):
        monkeypatch.setenv("HOM2D_NO_PDL", no_pdl)  # read at hom2d_create
        s = P.Solver(P.make_config(40, 32, method=method, k=k, bc=bc, box=box, cfl=cfl, limiter=limiter))
        s.init_case(case)
        s.step(60)
        out.append(s.get_state())
        s.close()
    monkeypatch.setenv("HOM2D_NO_PDL", "0")
    P.Solver(P.make_config(8, 8)).close()  # leave PDL on for the tests that follow
    np.testing.assert_array_equal(out[0], out[1])


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("bc", [0, 1])
def test_dg_overintegration_residual(orc, P, k, bc):
    """f3: DG with (k+2)-point over-integration of Eq. (19) (dgoi_stage.cu) against
    the oracle's residual_dg_quad on seeded data, ragged grid."""
    import torch
    from paper_1709_01619_b200.inputs import perturb
    oc, s = pair(orc, P, 19, 13, "dg", k, 0.08, bc=bc, dg_overintegrate=1)
    q = perturb(orc.init_case(oc), seed=41 + k, amp=1e-2)
    r_gpu = s.residual(torch.from_numpy(q).cuda()).cpu().numpy()
    assert rel_linf_res(r_gpu, orc.residual(oc, q)) < 1e-12


@pytest.mark.parametrize("k,cfl", [(1, 0.24), (2, 0.13), (3, 0.08), (4, 0.05)])
def test_dg_overintegration_100_steps(orc, P, k, cfl):
    from paper_1709_01619_b200.inputs import perturb
    oc, s = pair(orc, P, 10, 10, "dg", k, cfl, dg_overintegrate=1)
    q = perturb(orc.init_case(oc), seed=6, amp=1e-3)
    s.set_state(q)
    t_g, n_g = s.step(100)
    q_o, t_o, n_o = orc.run(oc, q, 100)
    assert n_g == n_o == 100 and abs(t_g - t_o) <= 1e-12 * t_o
    assert rel_linf(s.get_state(), q_o) <= 1e-10


@pytest.mark.parametrize("k,cfl", [(1, 0.2), (2, 0.08)])
def test_dg_overintegration_shock_limited(orc, P, k, cfl):
    """over-integrated DG with the limiter after every stage (the fused element
    averages of dgoi_stage_kernel feed k_limit): state and marks per element."""
    box = (-1.0, 1.0, -1.0, 1.0)
    oc, s = pair(orc, P, 24, 24, "dg", k, cfl, bc=1, box=box, limiter=1, dg_overintegrate=1)
    q0 = orc.init_case(oc, orc.SHOCK)
    s.set_state(q0)
    cnt = np.zeros(8, dtype=np.int64)
    em = np.zeros(24 * 24, dtype=np.int64)
    q_o, t_o, n_o = orc.run(oc, q0, 40, 0.25, counts=cnt, emap=em)
    _, n_g = s.step(40, 0.25)
    assert n_g == n_o
    assert rel_linf(s.get_state(), q_o) <= 1e-10
    np.testing.assert_array_equal(s.decision_map(), em)


def test_dg_overintegration_self_exchange_bitwise(orc, P, monkeypatch):
    """the strip path (interior rows, then the boundary bands after the ghost-row
    exchange) of the over-integrated kernel equals the single launch bitwise"""
    from paper_1709_01619_b200.inputs import perturb
    outs = []
    for sx in ("0", "1", "2"):
        monkeypatch.setenv("HOM2D_SELF_EXCHANGE", sx)
        oc, s = pair(orc, P, 12, 10, "dg", 2, 0.1, dg_overintegrate=1)
        s.set_state(perturb(orc.init_case(oc), seed=8, amp=1e-3))
        s.step(10)
        outs.append(s.get_state())
        s.close()
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])


@pytest.mark.parametrize("method,k,limiter,sx", [("cpr", 3, 0, "0"), ("fv", 2, 0, "0"), ("dg", 1, 1, "0"),
                                                 ("sd", 2, 0, "1"), ("cpr", 1, 1, "2"), ("fv", 1, 0, "1")])
def test_fused_dt_bitwise_equals_kdt(orc, P, monkeypatch, method, k, limiter, sx):
    """The step's dt computed by every CTA of stage 1 and committed by stage 2
    (no k_dt launch) gives bitwise the state, t and step count of the k_dt chain
    (HOM2D_NO_DTFUSE=1) -- over a t_end-clipped run, with the limiter, and on the
    split (interior + boundary-band) multi-GPU stage path (HOM2D_SELF_EXCHANGE)."""
    monkeypatch.setenv("HOM2D_SELF_EXCHANGE", sx)
    box, bc, case, cfl = ((-1.0, 1.0, -1.0, 1.0), 1, P.SHOCK, 0.2) if limiter else ((-5.0, 5.0, -5.0, 5.0), 0,
                                                                                   P.VORTEX, 0.08)
    out = []
    for nofuse in ("0", "1"):
        monkeypatch.setenv("HOM2D_NO_DTFUSE", nofuse)
        s = P.Solver(P.make_config(24, 18, method=method, k=k, bc=bc, box=box, cfl=cfl, limiter=limiter))
        s.init_case(case)
        t1, n1 = s.step(37)
        t2, n2 = s.step(10 ** 6, t1 + 0.05)  # clipped at t_end
        out.append((s.get_state(), t1, n1, t2, n2))
        s.close()
    (qa, *ra), (qb, *rb) = out
    np.testing.assert_array_equal(qa, qb)
    assert ra == rb
