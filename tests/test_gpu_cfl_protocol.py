"""The max-CFL protocol (reading R19) run twice at
Table 1's first DoF level (1600 DoF): through the GPU path
(tools/sweep.py max_cfl, the sweep that produced profiles/round1_cfl_protocol.md)
and through the CPU oracle (the search written out again below), on the same
0.01 candidate grid.  Both must pick the same CFL: the protocol's output then
depends on the method, not on the implementation that ran it.

Protocol: from c_hi downwards in steps of 0.01, the first CFL whose run to t = 1
is stable and whose L2(rho) error (R8) differs by < 0.1 % from the run at half
that CFL."""
import math
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def oracle_max_cfl(orc, method, k, n, c_hi):
    def metric(cfl):
        cf = orc.config(nx=n, ny=n, method=method, k=k, cfl=cfl)
        try:
            q, t, _ = orc.run(cf, orc.init_case(cf), 10 ** 7, 1.0)
        except FloatingPointError:  # non-physical
            return None
        e = orc.error(cf, q, t)[1]
        return e if math.isfinite(e) else None

    for c100 in range(int(round(c_hi * 100)), 0, -1):
        e1 = metric(c100 / 100.0)
        if e1 is None:
            continue
        e2 = metric(c100 / 200.0)
        if e2 is None or e2 == 0.0:
            continue
        if abs(e1 - e2) / abs(e2) < 1e-3:
            return c100 / 100.0, e1, e2
    return None, None, None


@pytest.mark.parametrize("method,k,n,c_hi", [("cpr", 1, 20, 0.5), ("sd", 1, 20, 0.6), ("dg", 2, 20, 0.3),
                                             ("fv", 1, 40, 0.8)])
def test_protocol_same_cfl_gpu_and_oracle(orc, P, method, k, n, c_hi):
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sweep
    g = sweep.max_cfl(P, torch, method, k, n, "vortex", c_hi)
    c_o, e1, e2 = oracle_max_cfl(orc, method, k, n, c_hi)
    assert g["cfl"] is not None and g["cfl"] == c_o, (g, c_o)
    assert abs(g["metric"] / e1 - 1) < 1e-8 and abs(g["metric_half"] / e2 - 1) < 1e-8
