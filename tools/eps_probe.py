"""Adversarial accuracy check of the tensor-core probe scores: max
|s~ - s| / (cmax^2 + 2 |q| cmax) over input families that maximise the
bf16-split residual and the fp32 accumulation error (aligned, all-positive
vectors; mantissas just below a bf16 rounding boundary; wide exponent range).
usage: python tools/eps_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_kernels import _arrays  # noqa: E402

from paper_1802_02422_b200.query import probe_scores  # noqa: E402


def run(name, c, q):
    s, eps_scale = probe_scores(_arrays(c), q)
    c64, q64 = c.astype(np.float64), q.astype(np.float64)
    exact = (c64 * c64).sum(1)[None, :] - 2.0 * q64 @ c64.T
    cmax = np.sqrt((c64 * c64).sum(1).max())
    unit = cmax**2 + 2.0 * np.linalg.norm(q64, axis=1)[:, None] * cmax
    r = np.abs(s.astype(np.float64) - exact) / unit
    print(f"{name:28s} max err/unit = {r.max():.3e}   (eps_scale {eps_scale:.2e})", flush=True)
    return r.max()


rng = np.random.default_rng(0)
worst = 0.0
for d in (96, 128, 64, 32):
    g = rng.standard_normal((4096, d)).astype(np.float32)
    worst = max(worst, run(f"gaussian d={d}", g, g[:256].copy()))
    u = rng.uniform(0.5, 1.0, (4096, d)).astype(np.float32)
    worst = max(worst, run(f"positive aligned d={d}", u, u[:256].copy()))
    # mantissas just below a bf16 half-ulp boundary: 1 + (2^-8 - 2^-17) style
    base = 1.0 + (np.float32(2.0**-8) - np.float32(2.0**-17)) * rng.integers(1, 127, (4096, d))
    b = (base * rng.choice([1.0, 1.0], (4096, d))).astype(np.float32)
    worst = max(worst, run(f"bf16 boundary d={d}", b, b[:256].copy()))
    w = (rng.uniform(0.5, 1.0, (4096, d)) * 2.0 ** rng.integers(-6, 6, (1, d))).astype(np.float32)
    worst = max(worst, run(f"wide exponents d={d}", w, w[:256].copy()))
    big = (u * 1e3).astype(np.float32)
    worst = max(worst, run(f"offset positive x1e3 d={d}", big + 7.0, big[:256] + 7.0))
print(f"WORST {worst:.3e}")
