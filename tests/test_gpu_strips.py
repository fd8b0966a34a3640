"""Multi-GPU strip decomposition on ONE GPU: G strip-only handles (rank r of G,
created without an NCCL id) each compute the residual of their y-strip from
caller-supplied neighbour rows -- the exact kernel path a multi-GPU stage takes
after its NCCL halo exchange.  The concatenated strip residuals must equal the
whole-grid residual BITWISE (per-element arithmetic is partition-independent,
SURVEY 8(e)); the gloo test (test_dist_host.py) covers the exchange plan."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [(m, k) for m in ("cpr", "ndg", "dg", "sd") for k in (1, 2, 3, 4)] + [("fv", 1), ("fv", 2)]


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


@pytest.mark.parametrize("method,k", CASES)
@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("thin", [False, True])
def test_strips_bitwise(orc, P, method, k, G, bc, thin):
    """thin=False: nrows > 2G, the stage runs as interior rows + two boundary
    bands (the overlapped multi-GPU launch split); thin=True: nrows <= 2G, one
    launch after the exchange."""
    import torch
    from paper_1709_01619_b200.inputs import perturb
    rows = (3 if thin else 8) if method == "fv" else (2 if thin else 5)
    nx, ny = 19, rows * G
    npe = 1 if method == "fv" else (k + 1) ** 2
    box = (-5.0, 5.0, -5.0, 5.0)
    oc = orc.config(nx=nx, ny=ny, method=method, k=k, bc=bc, box=box)
    q = perturb(orc.init_case(oc), seed=31 + k, amp=1e-2)
    cfg = P.make_config(nx, ny, method=method, k=k, bc=bc, box=box)
    whole = P.Solver(cfg)
    r_glob = whole.residual(torch.from_numpy(q).cuda()).cpu().numpy().reshape(4, ny, nx, npe)
    Q = q.reshape(4, ny, nx, npe)
    gr = 2 if method == "fv" else 1
    parts = []
    for r in range(G):
        s = P.Solver(cfg, rank=r, nranks=G)
        assert (s.row0, s.nrows) == (r * rows, rows)
        loc = torch.from_numpy(np.ascontiguousarray(Q[:, s.row0:s.row0 + rows]).reshape(-1)).cuda()
        lo_rows = [s.row0 - gr + g for g in range(gr)]
        hi_rows = [s.row0 + rows + g for g in range(gr)]
        lo = hi = None
        if bc == 0 or r > 0:
            lo = torch.from_numpy(np.ascontiguousarray(Q[:, [x % ny for x in lo_rows]]).reshape(-1)).cuda()
        if bc == 0 or r < G - 1:
            hi = torch.from_numpy(np.ascontiguousarray(Q[:, [x % ny for x in hi_rows]]).reshape(-1)).cuda()
        parts.append(s.residual_strip(loc, lo, hi).cpu().numpy().reshape(4, rows, nx, npe))
        s.close()
    np.testing.assert_array_equal(np.concatenate(parts, axis=1), r_glob)
    whole.close()


@pytest.mark.parametrize("method,k,limiter", [("cpr", 3, 0), ("ndg", 4, 0), ("dg", 2, 0), ("sd", 1, 0),
                                              ("fv", 1, 0), ("fv", 2, 0), ("cpr", 1, 1), ("dg", 1, 1)])
def test_overlapped_stage_path_bitwise(P, monkeypatch, method, k, limiter):
    """The multi-GPU stage path on one GPU (HOM2D_SELF_EXCHANGE=1): the periodic
    wrap rows go through the ghost buffers on the high-priority exchange stream
    while the interior rows run, the boundary bands wait on its event, and the
    limiter's average rows take the same route.  30 steps (90 stages) must equal
    the single-launch path bitwise; the exchange stream's copies racing a kernel
    that writes its source or the ghost buffers would break this.  =2: the same
    through NCCL itself -- a 1-rank communicator (ncclCommInitRank), the grouped
    ncclSend/ncclRecv of every stage with rank 0 as both neighbours, the lambda /
    non-physical-flag ncclAllReduce of every step.  =3: the peer-memory halo
    (peer.cu) with the handle's own workspace as both neighbours': the signal
    kernel, the flag-gated pull kernel on the exchange stream, the ghost rows."""
    out = []
    for sx in ("0", "1", "2", "3"):
        monkeypatch.setenv("HOM2D_SELF_EXCHANGE", sx)
        cfg = P.make_config(23, 14, method=method, k=k, cfl=0.05, limiter=limiter)
        s = P.Solver(cfg)
        s.init_case(P.VORTEX)
        s.step(30)
        out.append(s.get_state())
        s.close()
    np.testing.assert_array_equal(out[0], out[1])
    np.testing.assert_array_equal(out[0], out[2])
    np.testing.assert_array_equal(out[0], out[3])


@pytest.mark.parametrize("method,k,limiter", [("cpr", 3, 0), ("fv", 2, 0), ("dg", 1, 1)])
def test_peer_connect_self_bitwise(P, monkeypatch, method, k, limiter):
    """The public peer-memory API on one GPU: hom2d_peer_id exports the
    workspace allocation (cuMemGetAddressRange + cudaIpcGetMemHandle), and
    hom2d_peer_connect with the handle's own id as both neighbours' (recognised
    as this process's allocation: no IPC mapping) switches the overlapped strip
    path to the peer-memory halo; 20 steps equal the plain path bitwise, and the
    error query's exchange (FV reconstructed error) takes the same route."""
    out = []
    for mode in ("plain", "peer"):
        monkeypatch.setenv("HOM2D_SELF_EXCHANGE", "1" if mode == "peer" else "0")
        cfg = P.make_config(21, 12, method=method, k=k, cfl=0.05, limiter=limiter,
                            fv_error_recon=1 if method == "fv" else 0)
        s = P.Solver(cfg)
        if mode == "peer":
            pid = s.peer_id()
            assert len(pid) == 80 and pid[:64] != bytes(64)
            s.peer_connect(pid, pid)
            with pytest.raises(P.Hom2dError):
                s.peer_connect(pid, pid)  # already connected
        s.init_case(P.VORTEX)
        s.step(20)
        out.append((s.get_state(), s.error(P.VORTEX, 0)))
        s.close()
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def test_peer_id_needs_strip_handle(P):
    """hom2d_peer_id / hom2d_peer_connect on a plain one-GPU handle: HOM2D_ERR_STATE."""
    s = P.Solver(P.make_config(8, 8, method="cpr", k=1))
    with pytest.raises(P.Hom2dError):
        s.peer_id()
    s.close()


@pytest.mark.parametrize("method,k", [("cpr", 2), ("fv", 2)])
def test_nccl_self_collectives(P, monkeypatch, method, k):
    """HOM2D_SELF_EXCHANGE=2: hom2d_error's sum/max allreduces, hom2d_decisions'
    sum allreduce and the non-physical flag's min allreduce on a 1-rank NCCL
    communicator give the single-GPU results exactly."""
    res = []
    for sx in ("0", "2"):
        monkeypatch.setenv("HOM2D_SELF_EXCHANGE", sx)
        s = P.Solver(P.make_config(16, 12, method=method, k=k, cfl=0.05, record_decisions=1))
        s.init_case(P.VORTEX)
        s.step(7)
        res.append((s.error(P.VORTEX, 0), s.error(P.VORTEX, 3), tuple(s.decisions()), s.time()))
        q = s.get_state()
        q[3 * (q.size // 4) + 5] = -1.0
        s.set_state(q, s.time())
        with pytest.raises(P.NonPhysicalState):
            s.step(3)
        s.close()
    assert res[0] == res[1]
