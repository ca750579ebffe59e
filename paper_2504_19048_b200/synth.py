"""Deterministic synthetic particle workloads (host numpy, input synthesis only).

The same arrays are handed to the CPU oracle, the reference (when generating
golden fixtures) and the CUDA path, so every comparison is on identical
inputs.  Conventions follow SURVEY.md §8(d):

* seed ``numpy.random.default_rng(20261017)``;
* isotropic directions ``mu = 2u-1, phi = 2*pi*u'``;
* flight length ``-ln(u'')/sigma_t`` with ``u''`` in (0, 1];
* the generic point source ``S`` (never the cube centre, which lies on a mesh
  vertex and on the plane x - 2y + z = 0 where the reference's centroid-0
  localization walk loses particles).
"""

from __future__ import annotations

import numpy as np

SEED = 20261017
POINT_SOURCE = (0.5123456789, 0.4876543211, 0.5031415926)


def rng(seed: int = SEED) -> np.random.Generator:
    return np.random.default_rng(seed)


def isotropic_directions(gen: np.random.Generator, n: int) -> np.ndarray:
    mu = 2.0 * gen.random(n) - 1.0
    phi = 2.0 * np.pi * gen.random(n)
    s = np.sqrt(np.maximum(0.0, 1.0 - mu * mu))
    return np.stack([s * np.cos(phi), s * np.sin(phi), mu], axis=1)


def flight_lengths(gen: np.random.Generator, n: int, sigma_t: float) -> np.ndarray:
    u = 1.0 - gen.random(n)  # (0, 1]
    return -np.log(u) / sigma_t


def point_source(n: int, src=POINT_SOURCE) -> np.ndarray:
    return np.tile(np.asarray(src, dtype=np.float64), (n, 1))


def uniform_box(gen: np.random.Generator, n: int, lo=0.05, hi=0.95) -> np.ndarray:
    lo = np.broadcast_to(np.asarray(lo, dtype=np.float64), (3,))
    hi = np.broadcast_to(np.asarray(hi, dtype=np.float64), (3,))
    return lo + (hi - lo) * gen.random((n, 3))


def flight_destinations(gen: np.random.Generator, positions: np.ndarray,
                        sigma_t: float) -> np.ndarray:
    """dest = pos + l * dir with isotropic dir and exponential l."""
    n = positions.shape[0]
    d = isotropic_directions(gen, n)
    ell = flight_lengths(gen, n, sigma_t)
    return positions + ell[:, None] * d


def torus_shell_points(gen: np.random.Generator, n: int, R: float, a_in: float,
                       a_out: float, theta_max: float = 2.0 * np.pi,
                       phi_max: float = 2.0 * np.pi) -> np.ndarray:
    """Generic points inside the toroidal shell a_in < r < a_out, in the
    sector 0 < theta < theta_max, 0 < phi < phi_max (a fixed-source sector)."""
    r = a_in + (a_out - a_in) * (0.1 + 0.8 * gen.random(n))
    th = theta_max * (0.05 + 0.9 * gen.random(n))
    ph = phi_max * (0.05 + 0.9 * gen.random(n))
    rr = R + r * np.cos(th)
    return np.stack([rr * np.cos(ph), rr * np.sin(ph), r * np.sin(th)], axis=1)


def points_in_elements(gen: np.random.Generator, vertices: np.ndarray,
                       elements: np.ndarray, elem_ids: np.ndarray) -> np.ndarray:
    """One generic point strictly inside each listed element (barycentric
    weights from a flat Dirichlet, kept away from the faces)."""
    k = elem_ids.shape[0]
    lam = -np.log(1.0 - gen.random((k, 4)))
    lam = 0.02 + 0.92 * lam / lam.sum(axis=1, keepdims=True)
    lam /= lam.sum(axis=1, keepdims=True)
    corners = vertices[elements[elem_ids]]          # (k, 4, 3)
    return np.einsum("kv,kvc->kc", lam, corners)
