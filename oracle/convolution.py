"""Toeplitz convolution H(k0) on the AIM grid via zero-padded FFTs (oracle).
TEST INFRASTRUCTURE ONLY.

P:303-309  eq:Hmn  H^(m,n) = G(k0, r_m, r_n); H is three-level Toeplitz and
           only its first row is unique
P:199-200  products with W H P "are accelerated with FFTs" and "operate on the
           entire AIM grid, including both the near and far regions"
P:281      H_s + H_d(k0) = H(k0)
P:320-337  self terms: eq:Hsmm H_s^(m,m) = 0, eq:Hdmm H_d^(m,m) = -j k0/(4 pi),
           eq:Hmm H^(m,m) = -j k0/(4 pi)

Readings (AMB-10, AMB-12; R10): circulant embedding of size 2N_a per
axis; the kernel sample at offset o (o = i for i < N_a, i - 2N_a for i > N_a)
is K(h |o|); the wrap slot i = N_a is 0 (it never reaches the cropped output).
The spectrum is split as the north star mandates: H_hat_s = DFT3(K_s) built
once, H_hat(k0) = H_hat_s + DFT3(K_d(k0)) per frequency.  Arrays are indexed
[z, y, x] so that ravel() gives the grid's linear index i + N_x (j + N_y k).
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft as sfft

from .kernels import FOUR_PI, G_d

WORKERS = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def padded_distances(n: tuple, h: float) -> tuple:
    """r = h sqrt(o_x^2 + o_y^2 + o_z^2) on the padded grid [2Nz, 2Ny, 2Nx];
    returns (r, wrap_mask)."""
    offs = []
    wrap = []
    for N in (n[2], n[1], n[0]):
        i = np.arange(2 * N)
        o = np.where(i < N, i, i - 2 * N)
        offs.append(o)
        wrap.append(i == N)
    oz, oy, ox = np.meshgrid(*offs, indexing="ij")
    q = ox * ox + oy * oy + oz * oz
    r = h * np.sqrt(q.astype(np.float64))
    wz, wy, wx = np.meshgrid(*wrap, indexing="ij")
    return r, (wz | wy | wx)


def kernel_static(n: tuple, h: float) -> np.ndarray:
    r, wrap = padded_distances(n, h)
    K = np.zeros(r.shape, dtype=np.complex128)
    nz = (r > 0) & ~wrap
    K[nz] = 1.0 / (FOUR_PI * r[nz])
    return K                      # K_s(0) = 0  (eq:Hsmm)


def kernel_dynamic(n: tuple, h: float, k0: float) -> np.ndarray:
    r, wrap = padded_distances(n, h)
    K = G_d(k0, r)                # includes G_d(0) = -j k0/(4 pi)  (eq:Hdmm)
    K[wrap] = 0.0
    return K


def spectrum_static(n: tuple, h: float) -> np.ndarray:
    return sfft.fftn(kernel_static(n, h), workers=WORKERS)


def spectrum(n: tuple, h: float, k0: float, Hs_hat: np.ndarray | None = None) -> np.ndarray:
    if Hs_hat is None:
        Hs_hat = spectrum_static(n, h)
    return Hs_hat + sfft.fftn(kernel_dynamic(n, h, k0), workers=WORKERS)


def convolve(H_hat: np.ndarray, g: np.ndarray) -> np.ndarray:
    """phi = IDFT3(H_hat * DFT3(pad(g)))[:Nz, :Ny, :Nx]; g is [..., Nz, Ny, Nx]."""
    Nz, Ny, Nx = g.shape[-3:]
    G = sfft.fftn(g, s=(2 * Nz, 2 * Ny, 2 * Nx), axes=(-3, -2, -1), workers=WORKERS)
    phi = sfft.ifftn(G * H_hat, axes=(-3, -2, -1), workers=WORKERS)
    return phi[..., :Nz, :Ny, :Nx]


def convolve_bruteforce(g: np.ndarray, h: float, kernel, self_value) -> np.ndarray:
    """Definition: phi(l) = sum_{l'} K(h |l - l'|) g(l'), K(0) = self_value.
    O(N_g^2), tiny grids only."""
    Nz, Ny, Nx = g.shape
    z, y, x = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    P = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
    d = P[:, None, :] - P[None, :, :]
    r = h * np.sqrt((d * d).sum(-1).astype(np.float64))
    H = np.empty(r.shape, dtype=np.complex128)
    nz = r > 0
    H[nz] = kernel(r[nz])
    H[~nz] = self_value
    return (H @ g.ravel()).reshape(g.shape)
