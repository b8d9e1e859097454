"""NEXT-4: the paper's §5.1 slope study (Table 1 / Fig. 1a) on the GPU path:
the fast solver's transport plan equals the dense Sinkhorn's (the fp64 oracle O1) to the paper's
magnitude (||P_O - P_S||_F ~ 1e-16..1e-17), the dense solver scales like N^3 (paper
3.01) and the GPU path like N (paper 1.01) once it is bandwidth-bound."""
import os
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "examples"))

import slope_study  # noqa: E402


def test_slope_study_table1():
    """Large-N slope fitted on 3e7 .. 3e8 points: the bandwidth-bound regime (smaller N still carries
    fixed per-update latencies)."""
    res = slope_study.run(paper_n=[10, 20, 40, 80, 160], large_n=[1_000_000, 30_000_000, 100_000_000, 300_000_000])
    out = os.environ.get("SLOPE_OUT")
    if out:
        import json
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
    for r in res["rows"]:
        assert r["plan_diff_F"] <= 1e-14, r
    assert 2.5 <= res["dense_slope"] <= 3.5, res["dense_slope"]
    assert 0.9 <= res["gpu_slope_large_n"] <= 1.1, res["large_n"]
