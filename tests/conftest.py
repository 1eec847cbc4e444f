"""pytest configuration: markers, shared fixtures, repo root on sys.path."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build(ref=False)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref_lib():
    """The unmodified reference (oracle/_ref). Built here when /root/reference exists; prebuilt .so otherwise."""
    import oracle
    if not oracle.Ref.available():
        if os.path.isdir(os.path.join(oracle.REF_ROOT, "src")):
            oracle.build(ref=True)
        else:
            pytest.skip("reference library not built and /root/reference absent")
    return oracle.Ref()


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def golden_scalar():
    return _load("scalar_cases.npz")


@pytest.fixture(scope="session")
def golden_encode():
    return _load("encode_cases.npz")


@pytest.fixture(scope="session")
def golden_neural():
    return _load("neural_cases.npz")


def case_config(g, name):
    """Rebuild an oracle.Config from a golden encode case."""
    import oracle
    c = g[f"{name}/cfg"]
    return oracle.Config(dim=int(c[0]), levels=int(c[1]), table_size=int(c[2]), features=int(c[3]),
                         base_resolution=int(c[4]), growth=float(g[f"{name}/growth"]), backend=int(c[5]),
                         level_scale=int(c[6]))


def merge_chain(idx, w):
    """Merge duplicate rows of one (sample, level) vertex chain in first-touch order, summing weights the way
    EncoderGradient::add does (reference src/encoding.cpp:110-120)."""
    out_i, out_w = [], []
    for i, wi in zip(idx.tolist(), w.tolist()):
        if i in out_i:
            out_w[out_i.index(i)] += wi
        else:
            out_i.append(i)
            out_w.append(0.0 + wi)
    return out_i, out_w


@pytest.fixture(scope="session")
def golden_fields():
    """noise_field_value / fit_field outputs of the unmodified reference (tests/golden/make_golden.py fields)."""
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "field_cases.npz"), allow_pickle=False)
