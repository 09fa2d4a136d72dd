"""Pins the CPU oracle (oracle/sd_oracle.cpp) against the reference's own
golden vectors and known-answer tests. CPU only."""
import collections
import math
import os

import numpy as np
import pytest

from conftest import rnd_stream

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_golden_weight_checksum(oracle):
    # proj/tests/test_core.cpp:55-63
    s = oracle.make_spec(2, 64, 4, 256, 128)
    w = oracle.Weights(s, 0)
    assert w.checksum() == 0x138062486C631272
    assert w.tensor("w_q")[0, 0] == pytest.approx(-0.0454264432, rel=1e-6)
    assert w.tensor("embedding")[0, 0] == pytest.approx(0.0976269245, rel=1e-6)
    assert w.tensor("head")[0, 0] == pytest.approx(0.100667059, rel=1e-6)
    assert oracle.Weights(s, 1).checksum() != w.checksum()


def test_weight_shapes(oracle):
    # proj/tests/test_core.cpp:65-79
    w = oracle.Weights(oracle.make_spec(3, 32, 2, 48, 50), 5)
    assert w.tensor("w_q", 1).shape == (32, 32)
    assert w.tensor("w_mlp_in", 1).shape == (48, 32)
    assert w.tensor("w_mlp_out", 1).shape == (32, 48)
    assert w.tensor("head").shape == (50, 32)
    assert w.tensor("embedding").shape == (32, 50)


def test_spec_validation(oracle):
    # proj/tests/test_core.cpp:11-24
    assert oracle.make_spec(2, 64, 4, 256, 128).head_dim == 16
    assert oracle.make_spec(32, 4096, 32, 11008, 32000).head_dim == 128
    with pytest.raises(oracle.OracleError, match="not divisible"):
        oracle.make_spec(2, 63, 4, 256, 128)
    with pytest.raises(oracle.OracleError):
        oracle.make_spec(0, 64, 4, 256, 128)


def test_golden_transcript_bytes(oracle):
    # proj/tests/test_dense.cpp:173-190
    w = oracle.Weights(oracle.make_spec(2, 64, 4, 256, 128), 0)
    recs, _ = oracle.run_monolithic(w, batch=3, target_len=20, interval=20, steps=20, seed=0)
    with open(os.path.join(GOLDEN, "golden_transcript_2x64_3seq_20.csv")) as f:
        assert oracle.transcript_csv(recs) == f.read()


def test_prompt_tokens(oracle):
    # proj/tests/test_core.cpp:129-136
    for i in range(1, 200):
        t = oracle.prompt_token(42, i, 97)
        assert 0 <= t < 97 and t == oracle.prompt_token(42, i, 97)


def test_int8_known_answer(oracle):
    # proj/tests/test_attention.cpp:286-308
    q, s = oracle.quantize_int8([1.27, 0.635, -1.27])
    assert s == pytest.approx(0.01, rel=1e-6)
    assert list(q) == [127, 64, -127]  # 63.5 ties to even
    q0, s0 = oracle.quantize_int8(np.zeros(8))
    assert s0 == 0.0 and not q0.any()


def test_int8_half_step_bound(oracle):
    # proj/tests/test_attention.cpp:310-334 (1000 of the 10k trials)
    vec = rnd_stream(7)
    worst = 0.0
    for _ in range(1000):
        x = vec(16)
        q, s = oracle.quantize_int8(x)
        exact = np.abs(x.astype(np.float64) - q.astype(np.float64) * s)
        worst = max(worst, float((exact - s / 2).max()))
    assert worst <= 1e-12


def test_half_rne(oracle):
    # proj/tests/test_attention.cpp:336-344
    h = oracle.float_to_half_bits
    f = oracle.half_bits_to_float
    assert h(0.0) == 0
    assert f(h(1.0)) == 1.0
    assert f(h(1.0 + 2.0**-11)) == 1.0
    assert f(h(1.0 + 3 * 2.0**-11)) == 1.0 + 2.0**-9
    # agrees with numpy's IEEE RNE on random + edge values
    vals = np.concatenate([np.random.default_rng(0).standard_normal(20000).astype(np.float32) * 10,
                           np.array([65504, 65519, 65520, 1e-8, 6e-5, 6.1e-5, -0.0, 1e30],
                                    dtype=np.float32)])
    ours = np.array([h(float(v)) for v in vals], dtype=np.uint16)
    assert np.array_equal(ours, vals.astype(np.float16).view(np.uint16))


def _double_oracle(q, ks, vs, heads, hd):
    # proj/tests/test_attention.cpp:26-61 — scalar double-precision attention
    out = np.zeros(heads * hd)
    for h in range(heads):
        sl = slice(h * hd, (h + 1) * hd)
        sc = np.array([np.dot(q[sl].astype(np.float64), k[sl].astype(np.float64)) for k in ks])
        sc = sc / math.sqrt(hd)
        e = np.exp(sc - sc.max())
        a = e / e.sum()
        out[sl] = sum(a[j] * vs[j][sl].astype(np.float64) for j in range(len(ks)))
    return out


def test_attention_single_token_returns_v(oracle):
    # proj/tests/test_attention.cpp:73-82
    vec = rnd_stream(7)
    s = oracle.make_spec(1, 16, 2, 8, 8)
    kv = oracle.KvShard(s, 0, 2, 64)
    q, k, v = vec(16), vec(16), vec(16)
    kv.append_request(0, [7], [0], k[None], v[None])
    assert np.array_equal(kv.attend(0, [7], q[None])[0], v)


def test_attention_incremental_matches_double_oracle(oracle):
    # proj/tests/test_attention.cpp:142-163 (10 of 50 trials)
    vec = rnd_stream(11)
    s = oracle.make_spec(1, 32, 4, 8, 8)
    for trial in range(10):
        kv = oracle.KvShard(s, 0, 4, 256)
        ks, vs = [], []
        n = 1 + oracle.mix64(trial) % 64
        worst = 0.0
        for pos in range(n):
            q = vec(32)
            ks.append(vec(32))
            vs.append(vec(32))
            kv.append_request(0, [1], [pos], ks[-1][None], vs[-1][None])
            o = kv.attend(0, [1], q[None])[0]
            worst = max(worst, float(np.abs(o - _double_oracle(q, ks, vs, 4, 8)).max()))
        assert worst < 1e-5


def test_storage_formats_within_bounds(oracle):
    # proj/tests/test_attention.cpp:165-203
    vec = rnd_stream(13)
    s = oracle.make_spec(1, 32, 4, 8, 8)
    wh = wi = 0.0
    for trial in range(60):
        sh = {f: oracle.KvShard(s, 0, 4, 256, f) for f in ("single", "half", "int8")}
        n = 1 + oracle.mix64(1000 + trial) % 32
        for pos in range(n):
            q, k, v = vec(32), vec(32), vec(32)
            for kv in sh.values():
                kv.append_request(0, [1], [pos], k[None], v[None])
        base = sh["single"].attend(0, [1], q[None])
        wh = max(wh, float(np.abs(sh["half"].attend(0, [1], q[None]) - base).max()))
        wi = max(wi, float(np.abs(sh["int8"].attend(0, [1], q[None]) - base).max()))
    assert wh < 2e-3 and wi < 5e-2


def test_kvshard_capacity_positions_atomicity_drop(oracle):
    # proj/tests/test_attention.cpp:205-284
    vec = rnd_stream(17)
    s = oracle.make_spec(2, 8, 2, 8, 8)
    kv = oracle.KvShard(s, 0, 2, 4)
    k, v = vec(8), vec(8)
    kv.append(1, 0, 0, k, v)
    assert kv.stored_length(1, 0) == 1
    kv.append(1, 1, 0, k, v)
    assert kv.token_count() == 1
    for pos in range(1, 4):
        for layer in range(2):
            kv.append(1, layer, pos, k, v)
    assert kv.token_count() == 4
    with pytest.raises(oracle.OracleError, match="capacity exceeded") as e:
        kv.append(1, 0, 4, k, v)
    assert e.value.kind == "CapacityError"

    s1 = oracle.make_spec(1, 8, 2, 8, 8)
    kv = oracle.KvShard(s1, 0, 2, 64)
    with pytest.raises(oracle.OracleError) as e:
        kv.append(9, 0, 3, k, v)
    assert e.value.kind == "UnknownSequenceError"
    kv.append(9, 0, 0, k, v)
    with pytest.raises(oracle.OracleError) as e:
        kv.append(9, 0, 2, k, v)
    assert e.value.kind == "ProtocolError"

    kv = oracle.KvShard(s1, 0, 2, 2)
    ks = np.stack([vec(8) for _ in range(3)])
    with pytest.raises(oracle.OracleError) as e:
        kv.append_request(0, [1, 2, 3], [0, 0, 0], ks, ks)
    assert e.value.kind == "CapacityError"
    assert kv.token_count() == 0 and not kv.has_sequence(1)

    kv = oracle.KvShard(s, 0, 2, 16)
    for pos in range(3):
        for layer in range(2):
            kv.append(4, layer, pos, k, v)
    assert kv.token_count() == 3
    kv.drop_sequence(4)
    assert kv.token_count() == 0 and not kv.has_sequence(4) and kv.warning_count() == 0
    kv.drop_sequence(4)
    assert kv.warning_count() == 1
    with pytest.raises(oracle.OracleError) as e:
        kv.attend(0, [4], vec(8)[None])
    assert e.value.kind == "UnknownSequenceError"


def test_bytes_per_token(oracle):
    # attention.cpp:296-305
    s = oracle.make_spec(1, 32, 4, 8, 8)
    assert oracle.KvShard(s, 0, 4, 8, "single").bytes_per_token() == 2 * 32 * 4
    assert oracle.KvShard(s, 0, 4, 8, "half").bytes_per_token() == 2 * 32 * 2
    assert oracle.KvShard(s, 0, 4, 8, "int8").bytes_per_token() == 2 * (32 + 4 * 4)
    assert oracle.KvShard(s, 0, 4, 8, "int4").bytes_per_token() == 2 * (16 + 4 * 4)


def test_int4_codec_follows_the_int8_rules(oracle):
    """The 4-bit extension restated independently in
    numpy: scale = fp32(max|x| / 7), q = clamp(round-half-even(x * (1 / scale)
    in double), +-7), element 2i in the low nibble; zeros give scale 0."""
    rng = np.random.default_rng(4)
    cases = [rng.uniform(-1, 1, 128).astype(np.float32), np.zeros(16, np.float32),
             np.array([7, -7, 3.5, -3.5, 0.5, -0.5, 1e-30, 6.999], np.float32)]
    for x in cases:
        packed, sc = oracle.quantize_int4(x)
        mx = np.float32(np.abs(x).max())
        want_sc = np.float32(mx / np.float32(7.0)) if mx else np.float32(0)
        assert np.float32(sc) == want_sc
        inv = 1.0 / float(want_sc) if want_sc else 0.0
        want = np.clip(np.rint(x.astype(np.float64) * inv), -7, 7).astype(np.int8)
        assert np.array_equal(oracle.unpack_int4(packed, x.size), want)
        nib = (want & 0xF).astype(np.uint8)
        assert np.array_equal(packed, nib[0::2] | (nib[1::2] << 4))


def test_int4_storage_within_bounds(oracle):
    """int4 attention against fp32 storage on the reference's bounds test
    inputs (test_attention.cpp:165-203): 4 bits of mantissa per element."""
    vec = rnd_stream(13)
    s = oracle.make_spec(1, 32, 4, 8, 8)
    w4 = 0.0
    for trial in range(30):
        sh = {f: oracle.KvShard(s, 0, 4, 256, f) for f in ("single", "int4")}
        n = 1 + oracle.mix64(1000 + trial) % 32
        for pos in range(n):
            q, k, v = vec(32), vec(32), vec(32)
            for kv in sh.values():
                kv.append_request(0, [1], [pos], k[None], v[None])
        base = sh["single"].attend(0, [1], q[None])
        w4 = max(w4, float(np.abs(sh["int4"].attend(0, [1], q[None]) - base).max()))
    assert 1e-3 < w4 < 0.5
    with pytest.raises(oracle.OracleError, match="even head_dim"):
        oracle.KvShard(oracle.make_spec(1, 12, 4, 8, 8), 0, 4, 8, "int4")


def test_shardmap_cases(oracle):
    # proj/tests/test_transport.cpp:333-387
    for seq in range(50):
        for h in range(8):
            assert oracle.shardmap_worker_for("by-sequence", 8, 1, seq, h) == 0
    assert oracle.shardmap_head_range("by-head", 8, 2, 0) == (0, 4)
    assert oracle.shardmap_head_range("by-head", 8, 2, 1) == (4, 4)
    assert [oracle.shardmap_head_range("by-head", 7, 3, w)[1] for w in range(3)] == [3, 2, 2]
    c = collections.Counter(oracle.shardmap_worker_for("by-sequence", 8, 4, q, 0)
                            for q in range(1, 1001))
    assert [c[i] for i in range(4)] == [261, 241, 244, 254]  # within [230, 270]
    for mode in ("by-sequence", "by-head", "hybrid"):
        for workers in (1, 2, 4):
            for seq in range(1, 65):
                for h in range(8):
                    w = oracle.shardmap_worker_for(mode, 8, workers, seq, h)
                    h0, hc = oracle.shardmap_head_range(mode, 8, workers, w)
                    assert 0 <= w < workers and h0 <= h < h0 + hc


def test_scheduler_worked_examples(oracle):
    # proj/tests/test_scheduler.cpp:40-105, 148-200
    assert oracle.micro_batch_size(6, 2, 6) == 2
    assert oracle.micro_batch_size(7, 3, 10) == 2
    with pytest.raises(oracle.OracleError, match="interval too short"):
        oracle.micro_batch_size(4, 2, 16)
    t = oracle.LoadTracker(24)
    assert t.earliest_start(2, 6) == 0
    t.add_micro_batch(0, 2, 6)
    t.add_micro_batch(2, 2, 6)
    assert [w for _, w in t.batches()] == [20, 12]
    with pytest.raises(oracle.OracleError, match="admission rejected"):
        t.add_micro_batch(3, 2, 6)
    assert [w for _, w in t.batches()] == [20, 12]
    t = oracle.LoadTracker(100)
    t.add_micro_batch(0, 2, 3)
    t.add_micro_batch(1, 1, 3)
    loads = [t.step()["total_load"] for _ in range(5)]
    assert loads == [2, 5, 8, 3, 0]
    adm = oracle.cold_start_schedule(6, 6, 2, "fixed-interval", 8)
    assert adm == [(2 * k, 2, 6) for k in range(5)]
    adm = oracle.cold_start_schedule(6, 6, 2, "fixed-interval", 40)
    plans = oracle.run_schedule(adm, 24, 40)
    steady = [int(p[2]) for p in plans if p[0] > 6]
    assert max(int(p[2]) for p in plans) == 24
    assert steady == [18 if i % 2 == 0 else 24 for i in range(len(steady))]


def test_earliest_start_vs_exhaustive(oracle):
    # proj/tests/test_scheduler.cpp:14-36, 107-146 (2000 of 10k trials)
    state = [2024]

    def rnd(mod):
        state[0] = oracle.mix64(state[0])
        return state[0] % mod

    def feasible(limit):
        m = 1 + rnd(4)
        s = 1 + rnd(12)
        if m * s > limit:
            s = limit // m
        return m, max(1, s)

    for _ in range(2000):
        limit = 8 + rnd(60)
        t = oracle.LoadTracker(limit)
        for _ in range(rnd(7)):
            m, s = feasible(limit)
            start = t.earliest_start(m, s) + rnd(3)
            try:
                t.add_micro_batch(start, m, s)
            except oracle.OracleError:
                pass
        for _ in range(rnd(4)):
            t.step()
        m, s = feasible(limit)
        got = t.earliest_start(m, s)
        r = t.current_step()
        while True:
            if all(not (e > r) or w + (e - r) * m <= limit for e, w in t.batches()):
                break
            r += 1
        assert got == r


def test_every_sequence_completes_in_s_steps(oracle):
    # proj/tests/test_workers.cpp:334-344 (monolithic part)
    w = oracle.Weights(oracle.make_spec(2, 64, 4, 256, 128), 0)
    recs, _ = oracle.run_monolithic(w, batch=12, target_len=16, interval=4, steps=0)
    c = collections.Counter(q for _, q, _ in recs)
    assert len(c) == 12 and set(c.values()) == {16}


def test_batch_of_one_equals_batched_bitwise(oracle):
    # proj/tests/test_dense.cpp:145-171
    s = oracle.make_spec(2, 64, 4, 256, 128)
    w = oracle.Weights(s, 0)
    emb = w.tensor("embedding")
    x = np.stack([emb[:, b + 5] for b in range(3)]).astype(np.float32)
    a = oracle.KvShard(s, 0, 4, 1 << 12)
    b = oracle.KvShard(s, 0, 4, 1 << 12)
    for _ in range(4):
        ta, fa, _ = oracle.decode_step_monolithic(w, a, [1, 2, 3], x)
        tb, fb, _ = oracle.decode_step_monolithic(w, b, [2], x[1:2])
        assert ta[1] == tb[0] and np.array_equal(fa[1], fb[0])
        x = np.stack([emb[:, t] for t in ta]).astype(np.float32)


def test_gqa_extension_reduces_to_mha(oracle):
    """GQA is a repo extension (unpinned by the reference). With Hkv == H the
    extended oracle is the reference; with Hkv < H it equals MHA over
    repeated K/V heads."""
    vec = rnd_stream(19)
    H, Hkv, hd = 8, 2, 16
    s_gqa = oracle.make_spec(1, H * hd, H, 32, 8, Hkv)
    s_mha = oracle.make_spec(1, H * hd, H, 32, 8)
    g = oracle.KvShard(s_gqa, 0, Hkv, 64)
    m = oracle.KvShard(s_mha, 0, H, 64)
    G = H // Hkv
    for pos in range(9):
        k, v, q = vec(Hkv * hd), vec(Hkv * hd), vec(H * hd)
        rep = lambda t: np.repeat(t.reshape(Hkv, hd), G, axis=0).reshape(-1)
        g.append_request(0, [3], [pos], k[None], v[None])
        m.append_request(0, [3], [pos], rep(k)[None], rep(v)[None])
        assert np.array_equal(g.attend(0, [3], q[None]), m.attend(0, [3], q[None]))
