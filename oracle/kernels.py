"""Green's-function kernels (oracle, fp64).  TEST INFRASTRUCTURE ONLY.

P:151   time convention e^{j w t}
P:172   eq:hgf    G(k0, r) = e^{-j k0 r} / (4 pi r)
P:217   eq:hgftaylor   G = 1/(4 pi r) + (-j k0)/(4 pi) + (-j k0)^2 r/(4 pi 2!) + ...
P:226   eq:hgfs   G_s(r) = 1/(4 pi r)
P:230   eq:hgfd   G_d(k0, r) = (e^{-j k0 r} - 1)/(4 pi r)
P:331   eq:Hdmm   G_d(k0, r=0) = (-j k0)/(4 pi)

Constants (AMB-1, paper silent): c0 exact SI value, mu0 CODATA 2018.
"""
from __future__ import annotations

import math

import numpy as np

C0 = 299792458.0
MU0 = 1.25663706212e-6
EPS0 = 1.0 / (MU0 * C0 * C0)
ETA0 = math.sqrt(MU0 / EPS0)
FOUR_PI = 4.0 * math.pi


def wavenumber(f_hz: float) -> float:
    """k0 = omega / c0 with omega = 2 pi f."""
    return 2.0 * math.pi * f_hz / C0


def G(k0, r):
    """eq:hgf P:172-175."""
    r = np.asarray(r, dtype=np.float64)
    return np.exp(-1j * k0 * r) / (FOUR_PI * r)


def G_s(r):
    """eq:hgfs P:226-228 (static, frequency independent)."""
    r = np.asarray(r, dtype=np.float64)
    return 1.0 / (FOUR_PI * r)


def G_d(k0, r):
    """eq:hgfd P:230-232, evaluated without cancellation (AMB-11):
    e^{-jx} - 1 = -2 sin^2(x/2) - j sin(x), x = k0 r.
    At r = 0 the limit (-j k0)/(4 pi) of eq:hgfdtaylor / eq:Hdmm."""
    r = np.asarray(r, dtype=np.float64)
    k0 = np.asarray(k0, dtype=np.float64)
    r, k0 = np.broadcast_arrays(r, k0)
    out = np.empty(r.shape, dtype=np.complex128)
    z = r == 0.0
    rr = np.where(z, 1.0, r)
    x = k0 * rr
    s = np.sin(0.5 * x)
    re = -2.0 * s * s / (FOUR_PI * rr)
    im = -np.sin(x) / (FOUR_PI * rr)
    out.real = re
    out.imag = im
    out[z] = -1j * k0[z] / FOUR_PI
    return out


def taylor_G(k0, r, terms: int):
    """Partial sum of eq:hgftaylor: 1/(4 pi r) + sum_{l=1}^{terms-1}
    (-j k0)^l r^{l-1} / (4 pi l!)."""
    r = np.asarray(r, dtype=np.float64)
    acc = 1.0 / (FOUR_PI * r) + 0j
    for l in range(1, terms):
        acc = acc + (-1j * k0) ** l * r ** (l - 1) / (FOUR_PI * math.factorial(l))
    return acc
