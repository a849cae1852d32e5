"""Shared fixtures.  Markers: ``gpu`` = needs a B200 (run with -m gpu on the GPU box)."""
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run with -m gpu)")


@pytest.fixture(scope="session")
def golden_taps():
    return np.load(os.path.join(GOLDEN, "taps.npz"))


@pytest.fixture(scope="session")
def golden_cwth():
    return np.load(os.path.join(GOLDEN, "cwth.npz"))


def golden_cases(g):
    names = sorted({k.split("__")[0] for k in g.files if "__" in k})
    out = []
    for n in names:
        meta = g[f"{n}__meta"]
        out.append(dict(name=n, x=g[f"{n}__x"], scales=g[f"{n}__scales"], hop=int(meta[0]),
                        C=float(meta[1]), B=float(meta[2]), R=float(meta[3]),
                        kind=[str(v) for v in g[f"{n}__kind"]], ref=g[f"{n}__ref"]))
    return out


def row_rel_err(got, ref):
    """max over rows of max_k |got - ref| / max_k |ref_row| (SURVEY.md App. B metric)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    if ref.size == 0:
        return 0.0
    ref2 = ref.reshape(-1, ref.shape[-1])
    got2 = got.reshape(-1, got.shape[-1])
    scale = np.abs(ref2).max(axis=1)
    diff = np.abs(got2 - ref2).max(axis=1)
    ok = scale > 0
    err = np.where(ok, diff / np.where(ok, scale, 1.0), diff)
    return float(err.max())


def max_rel_err(actual, reference):
    """testutil.py:8-15 of the reference: max|a - r| / max|r| over the whole array."""
    actual = np.asarray(actual)
    reference = np.asarray(reference)
    scale = np.max(np.abs(reference)) if reference.size else 0.0
    if scale == 0:
        return float(np.max(np.abs(actual))) if actual.size else 0.0
    return float(np.max(np.abs(actual - reference)) / scale)


@pytest.fixture(scope="session")
def built_lib():
    """Build libwavehop_b200.so (nvcc cross-compiles without a GPU) if it is missing."""
    from paper_2408_14302_b200 import build

    return build.build()


@pytest.fixture(scope="session")
def golden_formats():
    return np.load(os.path.join(GOLDEN, "formats.npz"))


def decimate_cases(g, prefix):
    names = sorted({k.split("__")[0] for k in g.files if k.startswith(prefix) and "__" in k})
    return [(n, {k.split("__")[1]: g[k] for k in g.files if k.startswith(n + "__")}) for n in names]
