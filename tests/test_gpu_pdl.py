"""Programmatic dependent launch must not change results: every kernel waits
(griddepcontrol.wait) before touching its predecessor's outputs.  The same back-to-back
small-n sequences with PDL on and off (AA_NO_PDL=1, read once per process) must give
bitwise identical iterates for every variant."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_pdl_on_off_bitwise_identical(tmp_path):
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"pdl{flag}.npz"
        env = dict(os.environ, AA_NO_PDL=flag)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_pdl_worker.py"), str(out)],
                           capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        outs.append(np.load(out))
    a, b = outs
    assert set(a.files) == set(b.files) and len(a.files) == 15
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
        assert np.all(np.isfinite(a[k])), k
