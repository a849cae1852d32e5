"""Randomised parity sweep on the GPU (tools/fuzz.py): random hops (dividing 64 / 192, multiples
of 64 / 256, and hops only the SIMT engine takes), lengths from 1 sample, scale grids, both
wavelets, every output and min-max, AUTO and forced engines -- each case against the oracle;
"big" cases use full-length clips (160,000+ samples)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed,cases,mode", [(11, 80, ""), (12, 80, ""), (13, 20, "big")])
def test_random_cases_match_oracle(seed, cases, mode):
    args = [sys.executable, os.path.join(REPO, "tools", "fuzz.py"), str(cases), str(seed)] + ([mode] if mode else [])
    p = subprocess.run(args, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert p.returncode == 0 and "fuzz ok" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("seed,cases,env", [(63, 120, {"WH_UMMA_PSTREAM": "1"}),
                                             (64, 80, {"WH_UMMA_PSTREAM": "1", "WH_UMMA_NO_TMA": "1"}),
                                             (68, 80, {"WH_UMMA_PSTREAM": "1", "WH_UMMA_TF32": "1"})])
def test_random_cases_on_the_panel_streaming_paths(seed, cases, env):
    """The same sweep with panel streaming forced wherever it applies (TMA-fed fp16 panels,
    their cp.async fallback, the tf32 form).  Seed 63 holds the case that found fp16 panels
    straddling two rows of the batch tensor (hop 640, short filters: K origin not a multiple
    of 64)."""
    args = [sys.executable, os.path.join(REPO, "tools", "fuzz.py"), str(cases), str(seed)]
    p = subprocess.run(args, capture_output=True, text=True, timeout=600, cwd=REPO, env={**os.environ, **env})
    assert p.returncode == 0 and "fuzz ok" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]
