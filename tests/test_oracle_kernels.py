"""Pins for oracle/kernels.py against the paper's closed forms (not gpu)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import kernels as K

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_fixed_points.json")))


def test_G_d_self_term_matches_paper():
    # eq:Hdmm P:331: G_d(k0, 0) = -j k0 / (4 pi)
    for case in GOLD["G_d_self"]["cases"]:
        v = K.G_d(case["k0"], np.array([0.0]))[0]
        assert v.real == 0.0
        assert v.imag == pytest.approx(case["im"], rel=1e-15)


def test_taylor_coefficients_match_paper():
    # eq:hgftaylor P:217: coefficient of r^(l-1) is (-j k0)^l / (4 pi l!)
    g = GOLD["taylor_coefficients"]
    k0 = g["k0"]
    for c in g["coef"]:
        l = c["l"]
        # difference of consecutive partial sums at r = 1 isolates the term
        t = K.taylor_G(k0, 1.0, l + 1) - K.taylor_G(k0, 1.0, l)
        assert t.real == pytest.approx(c["re"], abs=1e-15)
        assert t.imag == pytest.approx(c["im"], abs=1e-15)


def test_decomposition_identity_G_equals_Gs_plus_Gd():
    # eq:hgfdecomp0 P:222 over k0 r in [1e-12, 1e2]
    rng = np.random.default_rng(7)
    kr = 10.0 ** rng.uniform(-12, 2, 20000)
    k0 = 10.0 ** rng.uniform(-3, 3, 20000)
    r = kr / k0
    lhs = K.G(k0, r)
    rhs = K.G_s(r) + K.G_d(k0, r)
    assert np.max(np.abs(lhs - rhs) / np.abs(lhs)) < 1e-13


def test_G_d_small_argument_against_series():
    # eq:hgfdtaylor P:326: G_d = (-jk0)/(4pi) + (-jk0)^2 r/(8 pi) + O(r^2)
    k0 = 5.0
    for kr in (1e-9, 1e-7, 1e-5):
        r = kr / k0
        ser = (-1j * k0) / (4 * math.pi) + (-1j * k0) ** 2 * r / (8 * math.pi) \
            + (-1j * k0) ** 3 * r * r / (24 * math.pi)
        v = K.G_d(k0, np.array([r]))[0]
        assert abs(v - ser) <= 1e-14 * abs(ser)


def test_G_d_bounded_and_vanishes_at_zero_frequency():
    # |e^{-jx} - 1| <= |x|  =>  |G_d| <= k0/(4 pi); G_d -> 0 as k0 -> 0
    rng = np.random.default_rng(3)
    r = 10.0 ** rng.uniform(-6, 2, 5000)
    for k0 in (1e-6, 0.3, 40.0):
        v = K.G_d(k0, r)
        assert np.all(np.abs(v) <= k0 / (4 * math.pi) * (1 + 1e-14))
    assert np.all(K.G_d(0.0, r) == 0.0)


def test_taylor_partial_sums_converge_to_G():
    k0, r = 3.0, 0.05
    err = [abs(K.taylor_G(k0, r, t) - K.G(k0, r)) for t in (2, 4, 8, 14)]
    assert err[-1] < 1e-15 * abs(K.G(k0, r)) * 10
    assert all(a > b for a, b in zip(err, err[1:]))
