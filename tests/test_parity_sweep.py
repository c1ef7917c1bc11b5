"""Randomised shape sweep of the whole path with attention (GPU vs oracle): GQA group sizes
1 / 2 / 4 / 8, head dims 64 / 128, ragged batch sizes, small page pools (LRU pressure and
uneven hits inside a batch), cascade on and off.  Integer outputs are compared bit for bit on
every batch inside run(); attention on sampled requests against fp64 (Z27)."""
import pytest

import oracle as O
from tests.parity_util import StreamSpec
from tests.test_parity_attn import run

pytestmark = pytest.mark.gpu

CASES = [
    # (Hq, Hkv, d, B, C, k, seed, ramp); C ~1.3x the smallest page pool the stream fits, so most
    # batches evict
    (8, 8, 128, 40, 200, 3, 11, (3,)),
    (16, 8, 64, 33, 450, 5, 12, (5, 17)),
    (32, 4, 128, 24, 650, 5, 13, ()),
    (64, 8, 128, 16, 200, 3, 14, (1,)),
    (4, 4, 64, 57, 450, 4, 15, (2, 9)),
    (12, 4, 128, 20, 330, 8, 16, (4,)),
]


@pytest.mark.parametrize("Hq,Hkv,d,B,C,k,seed,ramp", CASES)
def test_shape_sweep(Hq, Hkv, d, B, C, k, seed, ramp):
    sp = StreamSpec(n_logs=1500, n_templates=40, zipf=1.2, seed=seed, pool_seed=seed + 1000, k=k, B=B, C=C,
                    Hq=Hq, Hkv=Hkv, d=d, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=ramp, max_prompt_tokens=768)
    run(sp, n_batches=10, sample=6)


def test_shape_sweep_no_cascade(monkeypatch):
    monkeypatch.setenv("IL_CASCADE", "0")
    sp = StreamSpec(n_logs=1500, n_templates=40, zipf=1.2, seed=21, pool_seed=1021, k=5, B=30, C=700,
                    Hq=16, Hkv=4, d=128, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(2,))
    run(sp, n_batches=8, sample=6)
