"""GPU (-m gpu): the reference's `lattice` test suite (/root/reference/proj/tests/test_lattice.cpp) as far as it is visible
through the device's lattice walk.  The reference tests host functions (skew, subdivide, barycentric_weights,
unit_vertices, cell_vertices); on the device they exist only fused inside the encode kernels (csrc/sxen_device.cuh), and
`encode_debug` returns what they produce per (sample, level): the hashed index of every chain vertex and its weight.  So
each case places a point whose skewed cell coordinates are the reference's frozen fractions and checks the chain the
kernels walk; the random-point cases compare with tests/independent.py (dense-matrix skew, stable sort, from-scratch
hash)."""
import itertools

import numpy as np
import pytest

from independent import grid_vertices, simplex_vertices, skew_matrix, spatial_hash, unskew_matrix

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

T = 1 << 19
RES = 4


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def encoder(sx, n, backend=None, res=RES):
    return sx.HashEncoder(sx.EncoderConfig(dim=n, levels=1, table_size=T, features=2, base_resolution=res, growth=2.0,
                                           backend=sx.Backend.simplex if backend is None else backend))


def point_with_cell_coordinates(n, y, res=RES):
    """The point of the unit cube whose skewed, scaled coordinates are y (base + fractions)."""
    return (unskew_matrix(n) @ np.asarray(y, dtype=np.float64)) / (res / np.sqrt(n + 1.0))


def hashed(vertices):
    return spatial_hash(np.asarray(vertices, dtype=np.int64)) & np.uint32(T - 1)


def test_skew_constants_satisfy_the_exact_inverse_identity(sx):             # :39-45, 87-115
    for n in range(1, 9):
        f, g, s = sx.skew_constants(n)
        assert abs((1.0 + n * f) * (1.0 - n * g) - 1.0) < 1e-15
        assert np.allclose(np.eye(n) + f, skew_matrix(n), rtol=0, atol=1e-16)
        assert np.allclose(np.eye(n) - g, unskew_matrix(n), rtol=0, atol=1e-16)
    with pytest.raises(ValueError):                                          # :117-125
        sx.skew_constants(0)
    with pytest.raises(ValueError):
        sx.skew_constants(9)


def test_subdivide_and_barycentric_frozen_examples(sx):                     # :127-150, :169-184
    # fractions (0.3, 0.6): perm (1, 0), chain (0,0) (0,1) (1,1), weights (0.4, 0.3, 0.3)
    idx, w = encoder(sx, 2).encode_debug(point_with_cell_coordinates(2, [0.3, 0.6])[None, :])
    assert np.array_equal(idx[0, 0], hashed([[0, 0], [0, 1], [1, 1]]))
    assert np.abs(w[0, 0] - [0.4, 0.3, 0.3]).max() < 1e-12
    # fractions (0.7, 0.5, 0.2): identity perm, chain 000 100 110 111, weights (0.3, 0.2, 0.3, 0.2) -- in the cell with
    # base (1, 1, 1), because the base-0 cell's point with these fractions lies outside the unit cube
    idx, w = encoder(sx, 3).encode_debug(point_with_cell_coordinates(3, [1.7, 1.5, 1.2])[None, :])
    assert np.array_equal(idx[0, 0], hashed(1 + np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [1, 1, 1]])))
    assert np.abs(w[0, 0] - [0.3, 0.2, 0.3, 0.2]).max() < 1e-12
    # the same fractions in another cell: the chain is offset by the cell base (cell_vertices, :342-356)
    idx, w = encoder(sx, 3, res=16).encode_debug(point_with_cell_coordinates(3, [5.7, 4.5, 6.2], res=16)[None, :])
    base = np.array([5, 4, 6])
    assert np.array_equal(idx[0, 0], hashed(base + np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [1, 1, 1]])))
    assert np.abs(w[0, 0] - [0.3, 0.2, 0.3, 0.2]).max() < 1e-12


def test_ties_resolve_to_a_containing_simplex_that_reconstructs_the_point(sx):   # :152-167
    idx, w = encoder(sx, 2).encode_debug(point_with_cell_coordinates(2, [1.5, 2.5])[None, :])
    assert idx[0, 0, 0] == hashed([[1, 2]])[0] and idx[0, 0, 2] == hashed([[2, 3]])[0]
    assert idx[0, 0, 1] in (hashed([[2, 2]])[0], hashed([[1, 3]])[0])       # either simplex contains the diagonal
    # the tied middle vertex carries (next to) no weight, so either choice reconstructs the point
    assert abs(w[0, 0, 0] - 0.5) < 1e-12 and abs(w[0, 0, 1]) < 1e-12 and abs(w[0, 0, 2] - 0.5) < 1e-12


def test_every_permutations_chain_increments_one_axis_at_a_time(sx):        # :299-340
    for n in range(1, 5):                                # full n! enumeration while it stays small
        enc = encoder(sx, n)
        for perm in itertools.permutations(range(n)):
            fr = np.empty(n)
            fr[list(perm)] = np.linspace(0.9, 0.1, n)    # perm[0] has the largest fraction, and so on
            idx, w = enc.encode_debug(point_with_cell_coordinates(n, 1.0 + fr)[None, :])
            v = np.ones(n, dtype=np.int64)
            chain = [v.copy()]
            for k in range(n):
                v[perm[k]] += 1
                chain.append(v.copy())
            assert np.array_equal(idx[0, 0], hashed(chain)), (n, perm)
            assert abs(w[0, 0].sum() - 1.0) < 1e-12 and (w[0, 0] >= 0).all()


@pytest.mark.parametrize("n", range(1, 9))
def test_random_points_walk_the_independent_pipelines_chain(sx, n):         # :186-225, :237-260 (partition: one simplex)
    res = 16 if n <= 4 else 4
    x = torch.empty((500, n), dtype=torch.float64, device="cuda:0")
    sx.CounterRng(15, n).fill_device(x)
    xh = x.cpu().numpy()
    idx, w = encoder(sx, n, res=res).encode_debug(x)
    verts, want_w = simplex_vertices(n, res, xh)
    assert np.array_equal(idx[:, 0, :], hashed(verts))
    assert np.abs(w[:, 0, :] - want_w).max() < 1e-12
    # barycentric: the weights reconstruct the skewed point (the closed form against the geometry)
    y = (xh * (res / np.sqrt(n + 1.0))) @ skew_matrix(n).T
    assert np.abs((w[:, 0, :, None] * verts).sum(1) - y).max() < 1e-11
    if n <= 6:
        cidx, cw = encoder(sx, n, backend=sx.Backend.grid, res=res).encode_debug(x)
        corners, want_cw = grid_vertices(n, res, xh)
        assert np.array_equal(cidx[:, 0, :], hashed(corners))
        assert np.abs(cw[:, 0, :] - want_cw).max() < 1e-12
