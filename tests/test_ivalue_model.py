"""CPU model of the integer value product's fixed point (kv_mma.cu, IV): p is
carried as W = rn(p * vscale * (2^22 - 16) / Sb) with p <= 2 (the reference
max moves only past +1 in log2) and Sb = 1.0625 x the largest V scale, and
sum_j W_j * code_j is exact in integers. The model checks that this meets
the attention bar (2e-5 abs for |v| <= 1, test_attention.cpp:142-163) on the
parity tests' distributions, and that a 16-bit P would not: the reason for
three byte limbs."""
import numpy as np


def _attend(L, qscale, bits, rng, headroom_p=2.0, headroom_s=1.0625, hd=128):
    k = rng.uniform(-1, 1, (L, hd))
    v = rng.uniform(-1, 1, (L, hd))
    q = rng.uniform(-1, 1, hd) * qscale
    sv = np.abs(v).max(1) / 127
    c = np.rint(v / sv[:, None]).clip(-127, 127)          # quantize_int8's codes
    sk = np.abs(k).max(1) / 127
    s = (np.rint(k / sk[:, None]) * sk[:, None]) @ q / np.sqrt(hd)
    p = np.exp(s - s.max())                                # p <= 1 <= headroom_p
    w = p * sv
    exact = (w[:, None] * c).sum(0) / p.sum()
    sb = sv.max() * headroom_s
    scale = (2.0 ** (bits - 1) - 16) / (headroom_p * sb) if bits == 23 else (2.0 ** bits - 1) / (headroom_p * sb)
    W = np.rint(w * scale)
    assert W.max() < 2.0 ** bits
    approx = (W[:, None] * c).sum(0) / scale / p.sum()
    return float(np.abs(approx - exact).max())


def test_23_bit_p_meets_the_attention_bar():
    rng = np.random.default_rng(0)
    worst = max(_attend(L, qs, 23, rng) for qs in (3, 30, 90) for L in (17, 700, 2048) for _ in range(3))
    assert worst < 2e-5 / 4, worst  # with a 4x margin


def test_16_bit_p_would_not():
    rng = np.random.default_rng(0)
    worst = max(_attend(L, 30, 16, rng) for L in (700, 2048) for _ in range(5))
    assert worst > 2e-5, worst
