"""R-Part parity on the GPU: the B200 KvShard (paged HBM store + split-K
decode-attention kernel) against the CPU oracle restatement of
KvShard::append_request / attend (attention.cpp:139-305).

Tolerances: KV layout, int8 codes/scales and fp16 bits are bit-exact; the
attention output is fp32 with a different (parallel, online-softmax)
reduction order, so it must satisfy the reference's own bound of 1e-5 abs
for |values| <= 1 (test_attention.cpp:142-163, acceptance.cpp:303-357),
scaled by max|o| for larger values."""
import math

import numpy as np
import pytest

from conftest import rnd_stream

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sd():
    import paper_2403_11421_b200 as m
    return m


def _specs(sd, oracle, L, D, H, F, V, Hkv=0):
    return sd.make_model_spec(L, D, H, F, V, Hkv), oracle.make_spec(L, D, H, F, V, Hkv)


def _rng(seed):
    return np.random.default_rng(seed)


def test_single_token_returns_v_exactly(sd):
    # proj/tests/test_attention.cpp:73-82
    vec = rnd_stream(7)
    s = sd.make_model_spec(1, 16, 2, 8, 8)
    kv = sd.KvShard(s, 0, 2, 64)
    q, k, v = vec(16), vec(16), vec(16)
    o = kv.append_attend(0, [7], [0], q[None], k[None], v[None])
    assert np.array_equal(o[0], v)


def test_orthogonal_query_averages_values(sd):
    # proj/tests/test_attention.cpp:84-98 (hd = 4: generic kernel)
    vec = rnd_stream(9)
    s = sd.make_model_spec(1, 4, 1, 8, 8)
    kv = sd.KvShard(s, 0, 1, 64)
    k1, k2, q = np.zeros(4, np.float32), np.zeros(4, np.float32), np.zeros(4, np.float32)
    k1[0] = k2[1] = 1.0
    q[3] = 5.0
    v1, v2 = vec(4), vec(4)
    kv.append_request(0, [1], [0], k1[None], v1[None])
    kv.append_request(0, [1], [1], k2[None], v2[None])
    o = kv.attend(0, [1], q[None])[0]
    assert np.abs(o - (0.5 * v1 + 0.5 * v2)).max() < 1e-6


def test_softmax_weights_sum_to_one(sd):
    # proj/tests/test_attention.cpp:118-140 (hd = 12: generic kernel)
    vec = rnd_stream(5)
    n = 12
    s = sd.make_model_spec(1, n, 1, 8, 8)
    kv = sd.KvShard(s, 0, 1, 64)
    for pos in range(n):
        v = np.zeros(n, np.float32)
        v[pos] = 1.0
        kv.append_request(0, [1], [pos], vec(n)[None], v[None])
    w = kv.attend(0, [1], vec(n)[None])[0]
    assert (w >= 0).all() and abs(float(w.astype(np.float64).sum()) - 1.0) < 1e-6


def _double_attention(q, ks, vs, H, G, hd):
    out = np.zeros(H * hd)
    for h in range(H):
        kh = h // G
        qs = q[h * hd:(h + 1) * hd].astype(np.float64)
        sc = np.array([qs @ k[kh * hd:(kh + 1) * hd].astype(np.float64) for k in ks]) / math.sqrt(hd)
        e = np.exp(sc - sc.max())
        a = e / e.sum()
        out[h * hd:(h + 1) * hd] = sum(a[j] * vs[j][kh * hd:(kh + 1) * hd].astype(np.float64)
                                       for j in range(len(ks)))
    return out


@pytest.mark.parametrize("D,H", [(32, 4), (64, 4), (256, 2)])
def test_incremental_cache_matches_double_oracle(sd, D, H):
    # proj/tests/test_attention.cpp:142-163 and acceptance.cpp:303-357
    vec = rnd_stream(11 + D)
    s = sd.make_model_spec(1, D, H, 8, 8)
    hd = D // H
    for trial in range(6):
        kv = sd.KvShard(s, 0, H, 256)
        ks, vs = [], []
        worst = 0.0
        n = 1 + (trial * 37) % 64
        for pos in range(n):
            q = vec(D)
            ks.append(vec(D))
            vs.append(vec(D))
            o = kv.append_attend(0, [1], [pos], q[None], ks[-1][None], vs[-1][None])[0]
            worst = max(worst, float(np.abs(o - _double_attention(q, ks, vs, H, 1, hd)).max()))
        assert worst < 1e-5, (trial, worst)


CASES = [
    # (L, D, H, Hkv, fmt, batch, max_len)
    (2, 64, 4, 0, "single", 5, 40),        # reference toy geometry, hd 16
    (2, 64, 4, 0, "half", 5, 40),
    (2, 64, 4, 0, "int8", 5, 40),
    (1, 256, 2, 0, "single", 16, 130),     # C1 geometry, hd 128
    (1, 256, 2, 0, "half", 16, 130),
    (1, 512, 8, 2, "half", 7, 200),        # GQA (extension), hd 64
    (1, 1024, 8, 0, "single", 9, 300),     # hd 128, 8 heads
    (1, 2048, 16, 4, "int8", 6, 150),      # GQA + int8
    (1, 1024, 32, 0, "half", 4, 60),       # hd 32, 32 heads (2 heads per row group)
    (1, 4096, 32, 0, "half", 3, 90),       # Llama-2-7B head geometry
    (1, 5120, 40, 0, "half", 3, 70),       # Llama-2-13B head geometry (3 heads per row group)
    (1, 4096, 32, 8, "half", 3, 90),       # Llama-3-8B GQA geometry
    # int4 KV (extension: the paper's 4-bit hook)
    (2, 64, 4, 0, "int4", 5, 40),          # hd 16, CUDA-core K2
    (1, 48, 4, 0, "int4", 4, 30),          # hd 12: rows not 16-B multiples, generic path
    (1, 4096, 32, 0, "int4", 3, 90),       # Llama-2-7B heads, K2
    (1, 2048, 16, 4, "int4", 6, 150),      # GQA hd 128, tensor-core K2m
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[1]}x{c[2]}kv{c[3]}-{c[4]}" for c in CASES])
def test_ragged_batch_parity_vs_oracle(sd, oracle, case):
    L, D, H, Hkv, fmt, B, max_len = case
    s, os_ = _specs(sd, oracle, L, D, H, 8, 8, Hkv)
    hkv = s.num_kv_heads
    kvw = hkv * s.head_dim
    cap = B * max_len + 8
    gpu = sd.KvShard(s, 0, hkv, cap, fmt)
    cpu = oracle.KvShard(os_, 0, hkv, cap, fmt)
    rng = _rng(hash(case) & 0xffff)
    lens = rng.integers(1, max_len, B)
    seqs = [int(x) for x in rng.permutation(1000)[:B] + 1]
    # prefill through append_request, several positions at a time, all layers
    for pos in range(int(lens.max())):
        act = [i for i in range(B) if lens[i] > pos]
        ids = [seqs[i] for i in act]
        for layer in range(L):
            k = rng.uniform(-1, 1, (len(act), kvw)).astype(np.float32)
            v = rng.uniform(-1, 1, (len(act), kvw)).astype(np.float32)
            gpu.append_request(layer, ids, [pos] * len(act), k, v)
            cpu.append_request(layer, ids, [pos] * len(act), k, v)
    assert gpu.token_count() == cpu.token_count()
    for layer in range(L):
        q = rng.uniform(-1, 1, (B, D)).astype(np.float32) * 2.0
        og = gpu.attend(layer, seqs, q)
        oc = cpu.attend(layer, seqs, q)
        err = float(np.abs(og - oc).max())
        tol = 1e-5 if fmt == "single" else 2e-5
        assert err < tol, err
    # bit-exact KV layout / codecs against the oracle's storage
    for i in (0, B - 1):
        for which in (0, 1):
            bg, sg = gpu.export_lane(seqs[i], 0, which)
            bc, sc = cpu.export_lane(seqs[i], 0, which)
            assert np.array_equal(bg, bc)
            if fmt in ("int8", "int4"):
                assert np.array_equal(sg.view(np.uint32), sc.view(np.uint32))


def test_many_sequences_split_and_combine(sd, oracle):
    """Enough work to split items across CTAs (balanced split-K + combine)."""
    s, os_ = _specs(sd, oracle, 1, 1024, 8, 8, 8)
    B, Lmax = 300, 700
    gpu = sd.KvShard(s, 0, 8, B * Lmax, "half")
    cpu = oracle.KvShard(os_, 0, 8, B * Lmax, "half")
    rng = _rng(3)
    lens = rng.integers(1, Lmax, B)
    seqs = list(range(1, B + 1))
    for pos in range(int(lens.max())):
        act = [i for i in range(B) if lens[i] > pos]
        k = rng.uniform(-1, 1, (len(act), 1024)).astype(np.float32)
        v = rng.uniform(-1, 1, (len(act), 1024)).astype(np.float32)
        ids = [seqs[i] for i in act]
        gpu.append_request(0, ids, [pos] * len(act), k, v)
        cpu.append_request(0, ids, [pos] * len(act), k, v)
    q = rng.uniform(-2, 2, (B, 1024)).astype(np.float32)
    err = float(np.abs(gpu.attend(0, seqs, q) - cpu.attend(0, seqs, q)).max())
    assert err < 2e-5, err


@pytest.mark.parametrize("stages,rps", [(0, 1), (2, 1), (3, 1), (0, 0)],
                         ids=["default", "ring2", "ring3", "quad-copies"])
@pytest.mark.parametrize("iv", [0, 1], ids=["fp16-values", "int-values"])
@pytest.mark.parametrize("fmt", ["half", "int8", "int4"])
@pytest.mark.parametrize("h0,hc", [(4, 4), (2, 2), (7, 1)])
def test_gqa_tensor_core_head_slices(sd, oracle, fmt, h0, hc, stages, rps, iv):
    """Shards holding 4 / 2 / 1 of 8 kv heads (by-head / hybrid ShardMap):
    the tensor-core kernel splits each head's stages over 8/hc warps and
    merges their softmax states per piece. Any requested ring depth (0 =
    default) is rounded to a multiple of those 8/hc position classes: with
    fewer ring slots than classes a class's parity wait could pass on a
    slot's previous fill (a stage not yet landed) and the kernel hung.
    Shards of 1-2 heads copy 8 positions at a time (attn_rps8 = 1) or 4
    (0), in every format. Ring depth and slot layout are fixed when the
    store is built."""
    if rps != 1 and hc > 2:
        pytest.skip("copy width variants apply to shards of 1-2 kv heads")
    if iv and fmt == "half":
        pytest.skip("the integer value product: quantized KV")
    G = 4
    H, D = 8 * G, 8 * G * 128
    s, os_ = _specs(sd, oracle, 1, D, H, 8, 8, 8)
    B, Lmax = 24, 500
    with sd.tuned(attn_max_stages=stages, attn_rps8=rps):
        gpu = sd.KvShard(s, h0, hc, B * Lmax, fmt)
    cpu = oracle.KvShard(os_, h0, hc, B * Lmax, fmt)
    rng = _rng(100 + hc)
    lens = rng.integers(1, Lmax, B)
    lens[0], lens[1], lens[2] = 1, 17, 33
    seqs = list(range(1, B + 1))
    w = hc * 128
    for pos in range(int(lens.max())):
        act = [i for i in range(B) if lens[i] > pos]
        k = rng.uniform(-1, 1, (len(act), w)).astype(np.float32)
        v = rng.uniform(-1, 1, (len(act), w)).astype(np.float32)
        ids = [seqs[i] for i in act]
        gpu.append_request(0, ids, [pos] * len(act), k, v)
        cpu.append_request(0, ids, [pos] * len(act), k, v)
    q = rng.uniform(-3, 3, (B, w * G)).astype(np.float32)
    with sd.tuned(attn_ivalue=iv):
        got = gpu.attend(0, seqs, q)
    err = float(np.abs(got - cpu.attend(0, seqs, q)).max())
    assert err < 2e-5, err


@pytest.mark.parametrize("iv", [0, 1, 3], ids=["fp16-values", "int-values", "int-values-flush3"])
@pytest.mark.parametrize("imma", [1, 0], ids=["int-scores", "fp16-scores"])
@pytest.mark.parametrize("fmt", ["half", "int8", "int4"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_gqa_tensor_core_path_parity(sd, oracle, G, fmt, imma, iv):
    """fp16 / int8 KV, hd 128, 8 kv heads: the mma.sync attention path
    (kv_mma.cu), with ragged lengths (tails of 16-position stages) and split
    pieces. int8 keys enter the MMA as exact fp16 integers with the K scale
    applied to the scores and the V scale folded into p; same bar as fp16.
    iv: int8 values on integer tensor cores too (p as 23-bit fixed point in
    byte limbs, int32 sums flushed to fp32 when the reference max or the
    scale bound moves; flush3 forces a flush every 3 stages; int4 splits a
    byte column's nibbles into two head dims)."""
    if fmt == "half" and not imma:
        pytest.skip("fp16 KV has one score path")
    if iv and (fmt == "half" or not imma or G > 4):
        pytest.skip("the integer value product: quantized KV, integer scores, G <= 4")
    H = 8 * G
    D = H * 128
    s, os_ = _specs(sd, oracle, 1, D, H, 8, 8, 8)
    B, Lmax = 40, 700
    gpu = sd.KvShard(s, 0, 8, B * Lmax, fmt)
    cpu = oracle.KvShard(os_, 0, 8, B * Lmax, fmt)
    rng = _rng(G)
    lens = rng.integers(1, Lmax, B)
    lens[0], lens[1] = 1, 17
    seqs = list(range(1, B + 1))
    for pos in range(int(lens.max())):
        act = [i for i in range(B) if lens[i] > pos]
        k = rng.uniform(-1, 1, (len(act), 1024)).astype(np.float32)
        v = rng.uniform(-1, 1, (len(act), 1024)).astype(np.float32)
        ids = [seqs[i] for i in act]
        gpu.append_request(0, ids, [pos] * len(act), k, v)
        cpu.append_request(0, ids, [pos] * len(act), k, v)
    q = rng.uniform(-3, 3, (B, D)).astype(np.float32)
    with sd.tuned(attn_imma=imma, attn_ivalue=iv):
        og = gpu.attend(0, seqs, q)
    oc = cpu.attend(0, seqs, q)
    err = float(np.abs(og - oc).max())
    assert err < 2e-5, err


def test_capacity_positions_atomicity_drop(sd):
    # proj/tests/test_attention.cpp:205-284, reference error types
    vec = rnd_stream(17)
    s = sd.make_model_spec(2, 8, 2, 8, 8)
    kv = sd.KvShard(s, 0, 2, 4)
    k, v = vec(8), vec(8)
    kv.append(1, 0, 0, k, v)
    assert kv.stored_length(1, 0) == 1
    kv.append(1, 1, 0, k, v)
    assert kv.token_count() == 1
    for pos in range(1, 4):
        for layer in range(2):
            kv.append(1, layer, pos, k, v)
    assert kv.token_count() == 4
    with pytest.raises(sd.CapacityError, match="capacity exceeded"):
        kv.append(1, 0, 4, k, v)

    s1 = sd.make_model_spec(1, 8, 2, 8, 8)
    kv = sd.KvShard(s1, 0, 2, 64)
    with pytest.raises(sd.UnknownSequenceError):
        kv.append(9, 0, 3, k, v)
    kv.append(9, 0, 0, k, v)
    with pytest.raises(sd.ProtocolError) as e:
        kv.append(9, 0, 2, k, v)
    assert not isinstance(e.value, sd.UnknownSequenceError)

    kv = sd.KvShard(s1, 0, 2, 2)
    ks = np.stack([vec(8) for _ in range(3)])
    with pytest.raises(sd.CapacityError):
        kv.append_request(0, [1, 2, 3], [0, 0, 0], ks, ks)
    assert kv.token_count() == 0 and not kv.has_sequence(1)

    kv = sd.KvShard(s, 0, 2, 16)
    for pos in range(3):
        for layer in range(2):
            kv.append(4, layer, pos, k, v)
    assert kv.token_count() == 3
    kv.drop_sequence(4)
    assert kv.token_count() == 0 and not kv.has_sequence(4) and kv.warning_count() == 0
    kv.drop_sequence(4)
    assert kv.warning_count() == 1
    with pytest.raises(sd.UnknownSequenceError):
        kv.attend(0, [4], vec(8)[None])


def test_duplicate_item_partial_commit_matches_oracle(sd, oracle):
    """append_request validates against the pre-call state, then appends
    sequentially; a duplicated new sequence fails on its second item with the
    first already stored (attention.cpp:172-202)."""
    s, os_ = _specs(sd, oracle, 1, 32, 2, 8, 8)
    g, c = sd.KvShard(s, 0, 2, 64), oracle.KvShard(os_, 0, 2, 64)
    rows = np.ones((3, 32), np.float32)
    with pytest.raises(sd.ProtocolError):
        g.append_request(0, [5, 6, 5], [0, 0, 0], rows, rows)
    with pytest.raises(oracle.OracleError):
        c.append_request(0, [5, 6, 5], [0, 0, 0], rows, rows)
    for q in (5, 6):
        assert g.stored_length(q, 0) == c.stored_length(q, 0)
    assert g.token_count() == c.token_count()


def test_empty_layer_is_logic_error(sd):
    s = sd.make_model_spec(2, 32, 2, 8, 8)
    kv = sd.KvShard(s, 0, 2, 64)
    kv.append(3, 0, 0, np.ones(32), np.ones(32))
    with pytest.raises(sd.LogicError):
        kv.attend(1, [3], np.ones((1, 32)))


def test_slot_and_page_reuse_after_drop(sd, oracle):
    s, os_ = _specs(sd, oracle, 1, 128, 1, 8, 8)
    g = sd.KvShard(s, 0, 1, 200, "half", max_sequences=4)
    c = oracle.KvShard(os_, 0, 1, 200, "half")
    rng = _rng(5)
    live = {}
    nxt = 1
    for it in range(60):
        if len(live) == 4 or (live and rng.random() < 0.3):
            q = int(rng.choice(list(live)))
            g.drop_sequence(q)
            c.drop_sequence(q)
            del live[q]
        else:
            live[nxt] = 0
            nxt += 1
        ids = list(live)
        if not ids:
            continue
        k = rng.uniform(-1, 1, (len(ids), 128)).astype(np.float32)
        v = rng.uniform(-1, 1, (len(ids), 128)).astype(np.float32)
        q = rng.uniform(-1, 1, (len(ids), 128)).astype(np.float32)
        pos = [live[i] for i in ids]
        og = g.append_attend(0, ids, pos, q, k, v)
        c.append_request(0, ids, pos, k, v)
        oc = c.attend(0, ids, q)
        assert np.abs(og - oc).max() < 2e-5
        for i in ids:
            live[i] += 1
    assert g.token_count() == c.token_count()


@pytest.mark.parametrize("fmt,iv", [("int8", 0), ("int4", 0), ("int8", 1), ("int8", 2), ("int4", 1), ("int4", 2)])
def test_integer_scores_extreme_query_scales(sd, oracle, fmt, iv):
    """The integer-score path carries q per head as a 22-bit fixed-point
    integer scaled by the head's max: a zero head, a ~1e-20 head and a
    sharply peaked (x30) head must match the oracle like an ordinary one."""
    G = 4
    H, D = 8 * G, 8 * G * 128
    s, os_ = _specs(sd, oracle, 1, D, H, 8, 8, 8)
    B, L = 6, 90
    gpu = sd.KvShard(s, 0, 8, B * L, fmt)
    cpu = oracle.KvShard(os_, 0, 8, B * L, fmt)
    rng = _rng(77)
    seqs = list(range(1, B + 1))
    for pos in range(L):
        k = rng.uniform(-1, 1, (B, 1024)).astype(np.float32)
        v = rng.uniform(-1, 1, (B, 1024)).astype(np.float32)
        gpu.append_request(0, seqs, [pos] * B, k, v)
        cpu.append_request(0, seqs, [pos] * B, k, v)
    q = rng.uniform(-1, 1, (B, H, 128)).astype(np.float32)
    q[:, 0::4] = 0.0
    q[:, 1::4] *= 1e-20
    q[:, 2::4] *= 30.0
    q = q.reshape(B, D)
    with sd.tuned(attn_imma=1, attn_ivalue=iv):
        og = gpu.attend(0, seqs, q)
    oc = cpu.attend(0, seqs, q)
    err = float(np.abs(og - oc).max())
    assert err < 2e-5, err


@pytest.mark.parametrize("iv", [1, 0], ids=["int-values", "fp16-values"])
@pytest.mark.parametrize("imma", [1, 0])
def test_int8_pair_slot_variant(sd, oracle, imma, iv):
    """int8 with two positions per bulk copy (attn_i8_quad = 0; the default
    is four, the layout int4 always uses) under both score and value paths:
    same results as the oracle."""
    G = 4
    H, D = 8 * G, 8 * G * 128
    s, os_ = _specs(sd, oracle, 1, D, H, 8, 8, 8)
    B, Lmax = 12, 300
    with sd.tuned(attn_i8_quad=0):  # the slot layout is fixed when the store is built
        gpu = sd.KvShard(s, 0, 8, B * Lmax, "int8")
    cpu = oracle.KvShard(os_, 0, 8, B * Lmax, "int8")
    rng = _rng(31)
    lens = rng.integers(1, Lmax, B)
    lens[0] = 5
    seqs = list(range(1, B + 1))
    for pos in range(int(lens.max())):
        act = [i for i in range(B) if lens[i] > pos]
        k = rng.uniform(-1, 1, (len(act), 1024)).astype(np.float32)
        v = rng.uniform(-1, 1, (len(act), 1024)).astype(np.float32)
        ids = [seqs[i] for i in act]
        gpu.append_request(0, ids, [pos] * len(act), k, v)
        cpu.append_request(0, ids, [pos] * len(act), k, v)
    q = rng.uniform(-3, 3, (B, D)).astype(np.float32)
    with sd.tuned(attn_imma=imma, attn_ivalue=iv):
        og = gpu.attend(0, seqs, q)
    err = float(np.abs(og - cpu.attend(0, seqs, q)).max())
    assert err < 2e-5, err
