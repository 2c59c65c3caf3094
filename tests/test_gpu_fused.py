"""GPU checks of the fused probe (probe_fused.cu: fp16 tcgen05 GEMM whose
epilogue keeps only the centroids below a sampled threshold, K3a from fp16
centroid rows).  It is the default from K = 2^17 up (test_gpu_parity_scale
runs it at K = 2^20); here GIVF_PROBE=fused forces it on the small golden
indexes, in subprocesses because the probe mode is read once per process.

* the fp16 GEMM's own scores stay inside probe_f16_eps on inputs built to
  maximise fp16 rounding and accumulation error;
* the whole golden parity suite (test_gpu_parity.py: probe lists vs the
  oracle, full results vs the reference's own outputs) passes in fused mode;
* results are identical to the D-matrix path under every GEMM tile shape."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_BOUND_CODE = r"""
import sys, json, numpy as np
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
from test_gpu_kernels import _arrays
from paper_1802_02422_b200.query import probe_scores
fam, d = %(fam)r, %(d)d
rng = np.random.default_rng(11)
if fam == "gauss":
    c = rng.standard_normal((3000, d)) * 37.0
elif fam == "aligned":
    c = rng.uniform(0.5, 1.0, (3000, d))
elif fam == "boundary":   # mantissas just below an fp16 rounding boundary
    c = 1.0 + (2.0**-11 - 2.0**-20) * (2 * rng.integers(1, 500, (3000, d)) + 1)
else:                     # 2^+-6 exponent spread across the columns
    c = rng.uniform(0.5, 1.0, (3000, d)) * 2.0 ** rng.integers(-6, 6, (1, d))
c = c.astype(np.float32)
q = c[:200].copy()
s, eps_scale = probe_scores(_arrays(c), q)
c64, q64 = c.astype(np.float64), q.astype(np.float64)
exact = (c64 * c64).sum(1)[None, :] - 2.0 * q64 @ c64.T
cmax = np.sqrt((c64 * c64).sum(1).max())
unit = cmax**2 + 2.0 * np.linalg.norm(q64, axis=1)[:, None] * cmax
print(json.dumps([float(np.nanmax(np.abs(s - exact) / (eps_scale * unit))), int(np.isnan(s).sum())]))
"""


@pytest.mark.parametrize("family", ["gauss", "aligned", "boundary", "wide"])
@pytest.mark.parametrize("d", [24, 96, 128])
def test_fused_scores_within_bound(family, d):
    code = _BOUND_CODE % dict(root=ROOT, tests=os.path.join(ROOT, "tests"), fam=family, d=d)
    env = dict(os.environ, GIVF_PROBE="fused")
    out = subprocess.check_output([sys.executable, "-c", code], env=env, cwd=ROOT)
    ratio, nans = json.loads(out.decode().strip().splitlines()[-1])
    print(f"{family} d={d}: max |err| / bound = {ratio:.3e}")
    assert nans == 0          # the filter at thr = +inf returned every centroid
    assert ratio < 1.0        # the certified paths rely on this bound


def test_golden_parity_suite_in_fused_mode():
    """test_gpu_parity.py (probe lists vs the oracle, full results vs the
    reference fixtures, top-k vs the oracle) with the fused probe forced."""
    env = dict(os.environ, GIVF_PROBE="fused")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                       env=env, cwd=ROOT, capture_output=True, text=True)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0
