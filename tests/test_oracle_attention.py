"""Pins of the fp64 attention oracle (SURVEY §8(c) c.4 closed forms)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from workload import gen


ATTN = [O.attention, O.attention_np]          # the C++ loops and the numpy-matmul form, same pins


@pytest.mark.parametrize("attn", ATTN)
def test_single_key_returns_v0(attn):
    rng = np.random.default_rng(0)
    q = rng.normal(size=(1, 2, 8)); k = rng.normal(size=(1, 1, 8)); v = rng.normal(size=(1, 1, 8))
    o = attn(q, k, v, P=0, scale=0.3)
    assert np.allclose(o[0, 0], v[0, 0], atol=1e-15) and np.allclose(o[0, 1], v[0, 0], atol=1e-15)


@pytest.mark.parametrize("attn", ATTN)
def test_equal_logits_mean_of_visible(attn):
    rng = np.random.default_rng(1)
    L, P = 7, 3
    q = np.zeros((L - P, 1, 4)); k = rng.normal(size=(L, 1, 4)); v = rng.normal(size=(L, 1, 4))
    o = attn(q, k, v, P=P, scale=1.0)
    for s in range(L - P):
        assert np.allclose(o[s, 0], v[:P + s + 1, 0].mean(0), atol=1e-14)   # causal: j <= p


@pytest.mark.parametrize("attn", ATTN)
def test_two_keys_sigmoid(attn):
    d, delta = 4, 1.7
    k = np.zeros((2, 1, d)); k[0, 0, 0] = delta; v = np.zeros((2, 1, d)); v[0, 0, 1] = 1; v[1, 0, 2] = 1
    q = np.zeros((1, 1, d)); q[0, 0, 0] = 1.0
    o = attn(q, k, v, P=1, scale=1.0)
    sig = 1 / (1 + math.exp(-delta))
    assert o[0, 0, 1] == pytest.approx(sig, abs=1e-15) and o[0, 0, 2] == pytest.approx(1 - sig, abs=1e-15)


@pytest.mark.parametrize("attn", ATTN)
def test_first_token_sees_itself_and_peaky_argmax(attn):
    rng = np.random.default_rng(2)
    L = 5
    k = rng.normal(size=(L, 1, 8)); v = rng.normal(size=(L, 1, 8))
    q = rng.normal(size=(L, 1, 8))
    o = attn(q, k, v, P=0, scale=1.0)
    assert np.allclose(o[0, 0], v[0, 0], atol=1e-15)
    qb = q * 1e4
    ob = attn(qb, k, v, P=0, scale=1.0)
    for s in range(L):
        j = int(np.argmax((k[:s + 1, 0] @ qb[s, 0])))
        assert np.allclose(ob[s, 0], v[j, 0], atol=1e-9)


@pytest.mark.parametrize("attn", ATTN)
def test_matches_torch_sdpa_fp64_gqa(attn):
    """Special case reducing to a library routine: torch SDPA (fp64, explicit causal mask)."""
    rng = np.random.default_rng(3)
    Hq, Hkv, d, L, P = 8, 2, 16, 37, 20
    q = rng.normal(size=(L - P, Hq, d)); k = rng.normal(size=(L, Hkv, d)); v = rng.normal(size=(L, Hkv, d))
    o, lse = attn(q, k, v, P=P, scale=d ** -0.5, want_lse=True)
    g = Hq // Hkv
    tq = torch.tensor(q).permute(1, 0, 2)
    tk = torch.tensor(k).repeat_interleave(g, dim=1).permute(1, 0, 2)
    tv = torch.tensor(v).repeat_interleave(g, dim=1).permute(1, 0, 2)
    mask = torch.arange(L)[None, :] <= (torch.arange(L - P)[:, None] + P)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask, scale=d ** -0.5)
    assert np.allclose(o, ref.permute(1, 0, 2).numpy(), atol=1e-12)
    logits = torch.einsum("hsd,hld->hsl", tq, tk) * d ** -0.5
    logits = logits.masked_fill(~mask, -math.inf)
    assert np.allclose(lse, torch.logsumexp(logits, -1).T.numpy(), atol=1e-12)


def test_cache_transparency_generator():
    """Z28: K/V of a token depend only on (seed, token, position, head, dim), so a prefix
    cached by one request equals recomputation by another; cached prefill == recompute."""
    tok = np.arange(40, dtype=np.uint32) + 100
    pos = np.arange(40)
    a = gen.synth_bf16_bits(3000, "k", tok, pos, 2, 16)
    b = gen.synth_bf16_bits(3000, "k", tok[:25], pos[:25], 2, 16)
    assert (a[:25] == b).all()
    x = gen.bf16_bits_to_f64(a)
    assert np.abs(x).max() <= 1.0 and len(np.unique(x)) > 100
    q = gen.bf16_bits_to_f64(gen.synth_bf16_bits(3000, "q", tok, pos, 4, 16))
    v = gen.bf16_bits_to_f64(gen.synth_bf16_bits(3000, "v", tok, pos, 2, 16))
    full = O.attention(q, x, v, P=0, scale=0.25)
    part = O.attention(q[30:], x, v, P=30, scale=0.25)
    assert np.array_equal(full[30:], part)


def test_numpy_form_equals_loop_form_on_random_gqa():
    """attention_np (matmul steps) == attention (plain loops) to rounding, several shapes."""
    rng = np.random.default_rng(9)
    for Hq, Hkv, d, L, P in [(4, 4, 8, 1, 0), (8, 2, 16, 40, 23), (40, 8, 32, 70, 64), (6, 3, 8, 17, 0)]:
        q = rng.normal(size=(L - P, Hq, d)) * 3; k = rng.normal(size=(L, Hkv, d)); v = rng.normal(size=(L, Hkv, d))
        a, la = O.attention(q, k, v, P=P, scale=d ** -0.5, want_lse=True)
        b, lb = O.attention_np(q, k, v, P=P, scale=d ** -0.5, want_lse=True)
        assert np.allclose(a, b, atol=1e-12, rtol=0) and np.allclose(la, lb, atol=1e-12, rtol=0)
