"""Profiling aid: worst row error of the direct cascade cases with the default dense pass and the
CTA-pair variant (IL_DENSE2=1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import tests.test_parity_attn_direct as T  # noqa: E402

T.TOL = 1.0
reqs = [(1600, 33), (1840, 1), (2048, 200), (1600, 64), (1760, 130), (1600, 1), (1616, 97)]
for v in ("0", "1"):
    os.environ["IL_DENSE2"] = v
    errs = [T.run_case(32, 8, 128, reqs, shared_blocks=100, seed=s) for s in (17, 18, 19, 23)]
    errs2 = [T.run_case(32, 8, 128, reqs, shared_blocks=100, seed=s, big_rows=False) for s in (17, 18)]
    print("IL_DENSE2", v, "big rows", [round(e, 5) for e in errs], "plain", [round(e, 5) for e in errs2], flush=True)
