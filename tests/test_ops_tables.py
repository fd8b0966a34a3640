"""The CUDA path's generated operator tables (csrc/ops_tables.h, written by
tools/gen_ops.py) against numpy and closed forms -- CPU only, no oracle."""
import math
import os
import re

import numpy as np
import pytest
from numpy.polynomial import legendre as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1709_01619_b200", "csrc", "ops_tables.h")


def parse():
    txt = open(HDR).read()
    out = {}
    for m in re.finditer(r"struct (Ops<(\d)>|GL8) \{(.*?)\n\};", txt, re.S):
        key = int(m.group(2)) if m.group(2) else "GL8"
        tabs = {}
        for a in re.finditer(r"static constexpr double (\w+)((?:\[\d+\])+) = (\{.*?\});", m.group(3)):
            dims = [int(d) for d in re.findall(r"\[(\d+)\]", a.group(2))]
            vals = [float(v) for v in re.findall(r"[-+]?\d[\d.eE+-]*", a.group(3))]
            tabs[a.group(1)] = np.array(vals).reshape(dims)
        out[key] = tabs
    return out


T = parse()


def lagrange_eval(nodes, x):
    n = len(nodes)
    return np.array([np.prod([(x - nodes[m]) / (nodes[j] - nodes[m]) for m in range(n) if m != j]) for j in range(n)])


def test_gl8():
    x, w = L.leggauss(8)
    np.testing.assert_allclose(T["GL8"]["x"], x, atol=1e-15)
    np.testing.assert_allclose(T["GL8"]["w"], w, atol=1e-15)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_nodes_and_weights(k):
    n = k + 1
    t = T[k]
    x, w = L.leggauss(n)
    np.testing.assert_allclose(t["xi_gl"], x, atol=2e-16)
    np.testing.assert_allclose(t["w_gl"], w, atol=1e-15)
    inner = np.sort(L.legroots(L.legder(np.eye(n)[n - 1]))) if n > 2 else np.array([])
    gll = np.concatenate([[-1.0], inner, [1.0]])
    np.testing.assert_allclose(t["xi_gll"], gll, atol=1e-15)
    wg = 2.0 / (n * (n - 1) * L.legval(gll, np.eye(n)[n - 1]) ** 2)
    np.testing.assert_allclose(t["w_gll"], wg, atol=1e-15)
    np.testing.assert_allclose(t["xf_sd"], -np.cos(np.pi * np.arange(n + 1) / n), atol=1e-15)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_derivative_and_interpolation(k):
    n = k + 1
    t = T[k]
    for xs, D in ((t["xi_gll"], t["D_gll"]), (t["xi_gl"], t["D_gl"])):
        for d in range(n):
            np.testing.assert_allclose(D @ xs ** d, d * xs ** max(d - 1, 0) * (d > 0), atol=1e-13)
    np.testing.assert_allclose(t["eL_gl"], lagrange_eval(t["xi_gl"], -1.0), atol=1e-14)
    np.testing.assert_allclose(t["eR_gl"], lagrange_eval(t["xi_gl"], 1.0), atol=1e-14)
    c = np.zeros(k + 2)
    c[k] = c[k + 1] = 0.5
    dc = L.legder(c)
    np.testing.assert_allclose(t["gRp_gll"], L.legval(t["xi_gll"], dc), atol=1e-13)
    np.testing.assert_allclose(t["gRp_gl"], L.legval(t["xi_gl"], dc), atol=1e-13)
    np.testing.assert_allclose(t["gLp_gll"], -L.legval(-t["xi_gll"], dc), atol=1e-13)
    np.testing.assert_allclose(t["gLp_gl"], -L.legval(-t["xi_gl"], dc), atol=1e-13)
    w = t["w_gl"]
    np.testing.assert_allclose(t["dg_vol"], (w[None, :] * t["D_gl"].T) / w[:, None], atol=1e-13)
    np.testing.assert_allclose(t["dg_sR"], t["eR_gl"] / w, atol=1e-14)
    np.testing.assert_allclose(t["dg_sL"], t["eL_gl"] / w, atol=1e-14)
    # SD: interpolation to the flux points is exact on degree <= k, derivative on degree <= k+1
    xf, xs = t["xf_sd"], t["xi_gl"]
    for d in range(n):
        np.testing.assert_allclose(t["sd_I"] @ xs ** d, xf ** d, atol=1e-13)
    for d in range(n + 1):
        np.testing.assert_allclose(t["sd_D"] @ xf ** d, d * xs ** max(d - 1, 0) * (d > 0), atol=1e-12)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_overintegration_tables(k):
    """DG (k+2)-point over-integration (f3): the Gauss rule and the GL-basis values
    and derivatives at its points (exact on polynomials of degree <= k)."""
    n = k + 1
    t = T[k]
    z, W = L.leggauss(n + 1)
    np.testing.assert_allclose(t["oi_z"], z, atol=2e-16)
    np.testing.assert_allclose(t["oi_W"], W, atol=1e-15)
    xs = t["xi_gl"]
    for d in range(n):
        np.testing.assert_allclose(t["oi_L"] @ xs ** d, z ** d, atol=1e-14)
        np.testing.assert_allclose(t["oi_dL"] @ xs ** d, d * z ** max(d - 1, 0) * (d > 0), atol=1e-13)
