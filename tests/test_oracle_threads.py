"""The oracle's OpenMP option (timing only, SURVEY 8(d) "Oracle timing": 1 thread
and nproc threads, results bitwise equal): every residual and a short march with
4 threads equal the single-thread results bit for bit."""
import numpy as np
import pytest

import oracle as O
from paper_1709_01619_b200.inputs import perturb


@pytest.mark.parametrize("method,k", [("cpr", 2), ("ndg", 3), ("dg", 1), ("sd", 4), ("fv", 1), ("fv", 2)])
def test_threads_bitwise(method, k):
    n = 23 if method != "fv" else 57
    kw = dict(dg_overintegrate=1) if method == "dg" else {}
    cf = O.config(nx=n, ny=n - 4, method=method, k=k, cfl=0.1, **kw)
    q = perturb(O.init_case(cf), seed=12, amp=1e-2)
    out = []
    for th in (1, 4):
        O.set_threads(th)
        try:
            assert O.get_threads() == th
            r = O.residual(cf, q)
            qq, t, _ = O.run(cf, q, 3)
        finally:
            O.set_threads(1)
        out.append((r, qq, t))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]
