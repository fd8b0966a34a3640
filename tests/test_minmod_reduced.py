"""The troubled-cell detector's reduced minmod3 (aux.cu `MM3`, DESIGN §6 limiter
notes) against the three-way form of SURVEY C9 / reading R13.

The kernel reduces the element's neighbour-difference pair (b, c) once -- the
common sign (sign BITS of the high words) and the smaller magnitude -- and per
edge point returns the smaller magnitude of (a, that one) when the sign bits of
a and the pair agree, else a zero made by masking.  This host emulation of that
logic (sign bits via np.signbit, the same selects) checks the claim the kernel
relies on: the value equals minmod3 whenever no argument is zero, is a signed
zero otherwise, and every detector decision |q - (qbar -+ r)| > eps is the
same.  The GPU parity tests check the kernel's decisions against the oracle.
"""
import numpy as np


def minmod3(a, b, c):
    if a > 0.0 and b > 0.0 and c > 0.0:
        return min(a, b, c)
    if a < 0.0 and b < 0.0 and c < 0.0:
        return max(a, b, c)
    return 0.0


def mm3_reduced(a, b, c):
    same = np.signbit(b) == np.signbit(c)
    B = b if abs(b) <= abs(c) else c
    ok = same and (np.signbit(a) == np.signbit(B))
    m = a if abs(a) <= abs(B) else B
    return m if ok else 0.0


def _cases(rng, n):
    vals = [0.0, -0.0, 1e-3, -1e-3, 0.5, -0.5, 2.0, -2.0, 1e-300, -1e-300]
    for a in vals:
        for b in vals:
            for c in vals:
                yield a, b, c
    for _ in range(n):
        a, b, c = rng.normal(size=3) * 10.0 ** rng.integers(-4, 2, size=3)
        if rng.random() < 0.2:  # equal magnitudes
            b = np.copysign(abs(a), b)
        yield float(a), float(b), float(c)


def test_reduced_minmod3_value_and_decisions():
    rng = np.random.default_rng(11)
    eps = 1e-3
    for a, b, c in _cases(rng, 20000):
        r3, rr = minmod3(a, b, c), mm3_reduced(a, b, c)
        if a != 0.0 and b != 0.0 and c != 0.0:
            assert rr == r3 and np.signbit(rr) == np.signbit(r3)
        else:
            assert rr == 0.0
        # both detector sides (left/bottom: qbar - mm(qbar - q, ...), right/top: qbar + mm(q - qbar, ...))
        for cb in (1.0, 0.0, -0.0, 0.37):
            q_left, q_right = cb - a, cb + a
            d3 = abs(q_left - (cb - r3)) > eps, abs(q_right - (cb + r3)) > eps
            dr = abs(q_left - (cb - rr)) > eps, abs(q_right - (cb + rr)) > eps
            assert d3 == dr, (a, b, c, cb)
