"""Profiling aid: worst row-normalised attention error vs the fp64 oracle (tests/test_parity_attn
cases) for the library selected by IL_LIB_VARIANT (default build if unset)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests import test_parity_attn as T  # noqa: E402
from tests.parity_util import StreamSpec  # noqa: E402

cases = {
    "llama": lambda: T.run(StreamSpec(B=16, k=5, Hq=32, Hkv=8, d=128, max_prompt_tokens=1024), n_batches=3),
    "peaky": lambda: T.run(StreamSpec(B=16, k=5, Hq=32, Hkv=8, d=128, max_prompt_tokens=1024), n_batches=2, q_scale=8.0),
    "qwen": lambda: T.run(StreamSpec(B=12, k=8, Hq=40, Hkv=8, d=128, max_prompt_tokens=1536), n_batches=2),
    "long64": lambda: T.run(T._long(64), n_batches=2, sample=10, max_rows=48),
}
T.TOL = 1.0          # report, do not assert
for name, f in cases.items():
    print(f"{os.environ.get('IL_LIB_VARIANT', 'default'):10s} {name:8s} worst err {f():.3e}", flush=True)
