"""Independent numpy pipelines for the device suites -- test infrastructure, not product code.

The reference's tests do not compare the library with itself: tests/oracles.hpp re-derives every result from first
principles (dense skew matrix, a generic linear solve, a from-scratch hash, a dense matrix product).  This module is the
same idea in numpy, written from the published algorithm and NOT from oracle/sxen_oracle.c, so that agreement between the
device path, the C oracle and this file is evidence rather than tautology (tests/oracles.hpp:1-8).

  skew_matrix / unskew_matrix   tests/oracles.hpp:25-33   (I + f 1 1^T, I - g 1 1^T)
  spatial_hash                  tests/oracles.hpp:56-66   (64-bit products reduced mod 2^32, XOR)
  encode_simplex_level          tests/oracles.hpp:81-133  (clamp, scale, dense skew, floor, stable sort, chain, blend in fp64)
  encode_grid_level             tests/oracles.hpp:135-170 (2^n corners, product weights)
  mlp_forward                   tests/oracles.hpp:175-201 (dense W v + b, ReLU between layers, fp64)
"""
import numpy as np

PRIMES = np.array([1, 2654435761, 805459861, 3674653429, 2097192037, 1434869437, 2165219737, 4294967291], dtype=np.uint64)
ONE_BELOW = np.nextafter(1.0, 0.0)
MASK32 = np.uint64(0xFFFFFFFF)


def skew_matrix(n: int) -> np.ndarray:
    f = (np.sqrt(n + 1.0) - 1.0) / n
    return np.eye(n) + np.full((n, n), f)


def unskew_matrix(n: int) -> np.ndarray:
    g = (1.0 - 1.0 / np.sqrt(n + 1.0)) / n
    return np.eye(n) - np.full((n, n), g)


def spatial_hash(vertices: np.ndarray) -> np.ndarray:
    """vertices [..., n] int64 -> uint32 hash of every vertex."""
    v = np.asarray(vertices, dtype=np.int64)
    acc = np.zeros(v.shape[:-1], dtype=np.uint64)
    for i in range(v.shape[-1]):
        c = v[..., i].astype(np.uint64) & MASK32      # two's complement low word
        acc ^= (c * PRIMES[i]) & MASK32               # c, prime < 2^32: the 64-bit product cannot wrap
    return acc.astype(np.uint32)


def _rows(table, T, F):
    return np.asarray(table, dtype=np.float64).reshape(T, F)


def simplex_vertices(n: int, resolution: int, x: np.ndarray):
    """(vertices [N, n+1, n] int64, weights [N, n+1] float64) of the simplex containing each point of x [N, n]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    scale = float(resolution) / np.sqrt(n + 1.0)
    y = (np.minimum(x, ONE_BELOW) * scale) @ skew_matrix(n).T
    base = np.clip(np.floor(y).astype(np.int64), 0, resolution - 1)
    frac = np.clip(y - base, 0.0, ONE_BELOW)
    order = np.argsort(-frac, axis=1, kind="stable")          # descending, ties keep axis order
    fs = np.take_along_axis(frac, order, axis=1)
    w = np.empty((x.shape[0], n + 1))
    w[:, 0] = 1.0 - fs[:, 0]
    w[:, 1:n] = fs[:, :-1] - fs[:, 1:]
    w[:, n] = fs[:, n - 1]
    verts = np.empty((x.shape[0], n + 1, n), dtype=np.int64)
    cur = base.copy()
    verts[:, 0] = cur
    rows = np.arange(x.shape[0])
    for k in range(1, n + 1):
        cur[rows, order[:, k - 1]] += 1
        verts[:, k] = cur
    return verts, w


def grid_vertices(n: int, resolution: int, x: np.ndarray):
    """(corners [N, 2^n, n] int64, weights [N, 2^n] float64) of the grid cell containing each point."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    y = np.minimum(x, ONE_BELOW) * float(resolution)
    base = np.clip(np.floor(y).astype(np.int64), 0, resolution - 1)
    frac = np.clip(y - base, 0.0, ONE_BELOW)
    m = np.arange(1 << n)
    bits = (m[:, None] >> np.arange(n)[None, :]) & 1                         # [2^n, n]
    corners = base[:, None, :] + bits[None, :, :]
    # product in axis order, starting from 1.0, like the scalar loop (same roundings)
    w = np.ones((x.shape[0], 1 << n))
    for d in range(n):
        w = w * np.where(bits[None, :, d] == 1, frac[:, None, d], 1.0 - frac[:, None, d])
    return corners, w


def _blend(verts, w, table, T, F):
    idx = spatial_hash(verts) & np.uint32(T - 1)
    rows = _rows(table, T, F)[idx]                                           # [N, V, F]
    out = np.zeros((verts.shape[0], F))
    for k in range(verts.shape[1]):                                          # vertex order, like the scalar loop
        out += w[:, k, None] * rows[:, k, :]
    return out


def encode_simplex_level(n, resolution, T, F, table, x):
    v, w = simplex_vertices(n, resolution, x)
    return _blend(v, w, table, T, F)


def encode_grid_level(n, resolution, T, F, table, x):
    v, w = grid_vertices(n, resolution, x)
    return _blend(v, w, table, T, F)


def mlp_forward(cfg, weights, biases, inputs):
    """Dense fp64 forward: weights[l] is [out, in] row-major, ReLU after every layer but the last."""
    v = np.asarray(inputs, dtype=np.float64)
    L = len(weights)
    for l in range(L):
        W = np.asarray(weights[l], dtype=np.float64)
        v = v @ W.T + np.asarray(biases[l], dtype=np.float64)
        if l + 1 < L:
            v = np.maximum(v, 0.0)
    return v
