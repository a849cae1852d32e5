"""Non-finite input samples (NaN / +inf / -inf) against the reference's own outputs
(tests/golden/nonfinite.npz, oracle/gen_golden_nonfinite.py): a non-finite sample reaches
exactly the coefficients whose support [k*hop - L_s, k*hop + L_s] contains it, with the
reference's IEEE value there (NaN, or +-inf components; |W| = inf when a component is
infinite, as np.abs / hypot gives), and leaves every other coefficient -- of the same clip
and of the other clips in the batch -- at its finite value within the usual tolerance.
Per-clip min-max follows numpy's (v - lo) / (hi - lo): a NaN anywhere makes the clip NaN, an
infinite maximum maps the finite values to 0 and the infinite ones to NaN."""
import os

import numpy as np
import pytest

import paper_2408_14302_b200 as wh
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
ROW_TOL = 1e-5


def cases():
    g = np.load(os.path.join(GOLDEN, "nonfinite.npz"))
    names = sorted({k.split("__")[0] for k in g.files})
    return [(n, g[f"{n}__x"], g[f"{n}__scales"], int(g[f"{n}__hop"]), g[f"{n}__ref"]) for n in names]


CASES = cases()


def same_class(got, ref):
    """identical NaN / +inf / -inf pattern"""
    for f in (np.isnan, np.isposinf, np.isneginf):
        np.testing.assert_array_equal(f(got), f(ref))


def finite_rows_close(got, ref, tol=ROW_TOL):
    """per-row relative error over the entries the reference has finite; a
    complex array is compared as complex values (an imaginary part of ~1e-16, the a = 1 quirk,
    is judged against the row's |W|, as the golden tests do)"""
    fin = np.isfinite(ref) if not np.iscomplexobj(ref) else (np.isfinite(ref.real) & np.isfinite(ref.imag))
    scale = np.where(fin, np.abs(ref), 0.0).max(axis=-1, keepdims=True)
    d = np.where(fin, np.abs(got - np.where(fin, ref, 0.0)), 0.0)
    err = (d / np.where(scale > 0, scale, 1.0)).max()
    assert err <= tol, err


def batch(x, clean):
    """the bad clip between two clean ones"""
    return np.stack([clean, x, clean[::-1].copy()])


@pytest.mark.parametrize("engine", ["umma", "simt"])
@pytest.mark.parametrize("name,x,scales,hop,ref", CASES, ids=[c[0] for c in CASES])
def test_complex_output_propagates_like_the_reference(engine, name, x, scales, hop, ref):
    clean = np.random.default_rng(9).uniform(-1, 1, x.size).astype(np.float32)
    got = wh.cwth_batch(batch(x, clean), scales, None, hop, wavelet="cmor", output="complex", engine=engine)
    g = got[1]
    same_class(g.real, ref.real)
    same_class(g.imag, ref.imag)
    finite_rows_close(g, ref)
    # the clean clips are untouched by the bad one
    alone = wh.cwth_batch(np.stack([clean, clean[::-1].copy()]), scales, None, hop, wavelet="cmor",
                          output="complex", engine=engine)
    np.testing.assert_array_equal(got[[0, 2]], alone)


@pytest.mark.parametrize("engine", ["umma", "simt"])
@pytest.mark.parametrize("name,x,scales,hop,ref", CASES, ids=[c[0] for c in CASES])
def test_magnitude_outputs(engine, name, x, scales, hop, ref):
    clean = np.random.default_rng(9).uniform(-1, 1, x.size).astype(np.float32)
    xb = batch(x, clean)
    with np.errstate(invalid="ignore"):
        want = {("cmor", "abs"): np.abs(ref), ("rmor", "abs"): np.abs(ref.real),
                ("rmor", "log1p"): np.log1p(np.abs(ref.real))}
    for (wavelet, output), w in want.items():
        g = wh.cwth_batch(xb, scales, None, hop, wavelet=wavelet, output=output, engine=engine)[1]
        same_class(g, w)
        if output == "log1p":
            fin = np.isfinite(w)
            assert np.abs(np.where(fin, g - np.where(fin, w, 0), 0)).max() <= 1e-5
        else:
            finite_rows_close(g, w)


@pytest.mark.parametrize("engine", ["umma", "simt"])
@pytest.mark.parametrize("name,x,scales,hop,ref", CASES, ids=[c[0] for c in CASES])
def test_minmax_normalisation(engine, name, x, scales, hop, ref):
    clean = np.random.default_rng(9).uniform(-1, 1, x.size).astype(np.float32)
    got = wh.cwth_batch(batch(x, clean), scales, None, hop, wavelet="cmor", output="abs", norm="minmax",
                        engine=engine)
    m = np.abs(ref)
    with np.errstate(invalid="ignore"):
        lo, hi = m.min(), m.max()
        want = (m - lo) / (hi - lo)
    same_class(got[1], want)
    fin = np.isfinite(want)
    assert np.abs(np.where(fin, got[1] - np.where(fin, want, 0), 0)).max() <= 1e-5
    for c in (0, 2):  # clean clips: a proper [0, 1] range
        assert np.isfinite(got[c]).all() and got[c].min() == 0.0 and abs(got[c].max() - 1.0) <= 1e-6


def test_device_path_and_repeated_launches():
    """The records are reset by every launch: a clean launch after a bad one is clean, and the
    device (stream-ordered) path gives the host path's bytes."""
    import torch

    name, x, scales, hop, ref = CASES[0]
    plan = wh.CwthPlan(scales, None, hop, x.size, wavelet="cmor", output="abs", max_clips=2)
    clean = np.random.default_rng(3).uniform(-1, 1, x.size).astype(np.float32)
    bad = plan.execute_host(np.stack([x, clean])).copy()
    ok = plan.execute_host(np.stack([clean, clean])).copy()
    assert np.isfinite(ok).all()
    np.testing.assert_array_equal(ok[0], bad[1])
    dev = plan.execute(torch.from_numpy(np.stack([x, clean])).cuda()).cpu().numpy()
    np.testing.assert_array_equal(dev, bad)
    plan.close()
