"""GPU (-m gpu): the reference's `noise` test suite (/root/reference/proj/tests/test_noise.cpp) on the device path, for
the cases that go through the boundary this library exposes -- `noise_field_value` (the targets of fit_field).  A
one-octave field of frequency 1 is one noise evaluation (src/noise.cpp:167-188: octave 0 has weight 1 and the seed
hash_combine(seed, 0)), which is how the per-kind cases below reach `perlin_value` / `simplex_noise_value`.
`smoother_step`, `lattice_gradient` and `perlin_value_with` are internal to the device code (csrc/sxen_noise.cu) and have
no entry point; their values are pinned through tests/golden/field_cases.npz (test_gpu_tasks.py)."""
import numpy as np
import pytest

from independent import unskew_matrix

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def one(sx, kind, x, seed):
    """One noise evaluation at the points x [N, dim]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    spec = sx.NoiseFieldSpec(dim=x.shape[1], seed=seed, kind=kind, octaves=1, frequency=1.0)
    return sx.noise_field_value(spec, x)


def test_grid_noise_vanishes_at_every_integer_lattice_point(sx):            # :76-83
    for p in ([0.0, 0.0], [1.0, 2.0], [-3.0, 5.0], [4.0, 0.0, 2.0], [1.0]):
        assert abs(one(sx, sx.NoiseKind.perlin, [p], 7)[0]) < 1e-15


def test_grid_noise_is_deterministic_and_varies_with_the_seed(sx):          # :85-89
    x = [[0.37, 0.82]]
    assert one(sx, sx.NoiseKind.perlin, x, 5)[0] == one(sx, sx.NoiseKind.perlin, x, 5)[0]
    assert one(sx, sx.NoiseKind.perlin, x, 5)[0] != one(sx, sx.NoiseKind.perlin, x, 6)[0]


def test_simplex_noise_vanishes_at_shared_lattice_vertices(sx):             # :101-110
    assert abs(one(sx, sx.NoiseKind.simplex, [[0.0, 0.0]], 7)[0]) < 1e-12
    assert abs(one(sx, sx.NoiseKind.simplex, [[0.0, 0.0, 0.0]], 9)[0]) < 1e-12
    x = unskew_matrix(2) @ np.array([3.0, 1.0])          # a nonzero vertex: skewed integers mapped back
    assert abs(one(sx, sx.NoiseKind.simplex, [x], 7)[0]) < 1e-11


def test_simplex_noise_is_deterministic(sx):                                # :112-116
    x = [[0.21, 0.64, 0.93]]
    assert one(sx, sx.NoiseKind.simplex, x, 3)[0] == one(sx, sx.NoiseKind.simplex, x, 3)[0]
    assert one(sx, sx.NoiseKind.simplex, x, 3)[0] != one(sx, sx.NoiseKind.simplex, x, 4)[0]


def test_simplex_noise_census_is_bounded_and_symmetric(sx):                 # :118-138
    samples = 1000000
    x = torch.empty((samples, 2), dtype=torch.float64, device="cuda:0")
    sx.CounterRng(52).fill_device(x, 0.0, 64.0)          # the reference's draws, in its order
    spec = sx.NoiseFieldSpec(dim=2, seed=11, kind=sx.NoiseKind.simplex, octaves=1, frequency=1.0)
    v = sx.noise_field_value(spec, x).cpu().numpy()
    lo, hi = min(0.0, v.min()), max(0.0, v.max())
    assert 0.1 < hi < 2.0 and -2.0 < lo < -0.1           # unit gradients over cell-bounded displacements
    assert abs(hi + lo) <= 0.02 * max(hi, -lo)           # symmetric within 2 % of the extreme
    assert abs(v.sum() / samples) < 0.01


def test_octave_composition_is_the_normalized_weighted_sum(sx):             # :140-160
    x = np.array([[0.33, 0.71]])
    for kind in (sx.NoiseKind.perlin, sx.NoiseKind.simplex):
        two = sx.noise_field_value(sx.NoiseFieldSpec(dim=2, seed=21, kind=kind, octaves=2, frequency=4.0), x)[0]
        o0 = sx.noise_field_value(sx.NoiseFieldSpec(dim=2, seed=21, kind=kind, octaves=1, frequency=4.0), x)[0]
        # value = (o0 + 0.5 o1) / 1.5 with o1 one evaluation under another seed: recover it and hold it to the range
        # of a single evaluation; the exact two-octave values are in the reference-generated fixture
        o1 = (1.5 * two - o0) / 0.5
        assert abs(o1) < 2.0 and two != o0
        three = sx.noise_field_value(sx.NoiseFieldSpec(dim=2, seed=21, kind=kind, octaves=3, frequency=4.0), x)[0]
        o2 = (1.75 * three - o0 - 0.5 * o1) / 0.25
        assert abs(o2) < 2.0


def test_noise_field_validation(sx):                                        # :162-178
    spec = sx.NoiseFieldSpec(dim=0)
    with pytest.raises(ValueError):
        spec.validate()
    spec = sx.NoiseFieldSpec(dim=2, octaves=0)
    with pytest.raises(ValueError):
        spec.validate()
    spec = sx.NoiseFieldSpec(dim=2, octaves=1, frequency=0.0)
    with pytest.raises(ValueError):
        spec.validate()
    spec.frequency = 4.0
    spec.validate()
    assert sx.NoiseKind.perlin.name == "perlin" and sx.NoiseKind.simplex.name == "simplex"
    with pytest.raises(ValueError):
        sx.noise_field_value(spec, np.array([[0.5, 0.5, 0.5]]))   # spec.dim == 2
