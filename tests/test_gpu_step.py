"""GPU StepComputation parity: the engine (S-Part + R-Part on one B200)
against the oracle's decode_step_monolithic / run_monolithic and the
reference's golden transcript."""
import collections
import os

import numpy as np
import pytest

from conftest import upload_oracle_weights

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sd():
    import paper_2403_11421_b200 as m
    return m


def _engine(sd, oracle, spec_args, seed=0, mode="exact", fmt="single", cap=1 << 16):
    W = oracle.Weights(oracle.make_spec(*spec_args), seed)
    dw = upload_oracle_weights(W, mode)
    kv = sd.KvShard(dw.spec, 0, dw.spec.num_kv_heads, cap, fmt)
    return W, dw, kv, sd.Engine(dw, kv)


def test_golden_transcript_on_gpu(sd, oracle):
    # proj/tests/test_dense.cpp:173-190: byte-exact against the fixture
    W, dw, kv, eng = _engine(sd, oracle, (2, 64, 4, 256, 128))
    recs, _, _ = sd.run_generation(eng, batch=3, target_len=20, interval=20, steps=20, seed=0)
    with open(os.path.join(GOLDEN, "golden_transcript_2x64_3seq_20.csv")) as f:
        assert sd.transcript_csv(recs) == f.read()


def test_exact_dense_path_is_bitwise(sd, oracle):
    """K7 reproduces apply_linear / project_qkv bit for bit (dense.cpp:16-43)."""
    W = oracle.Weights(oracle.make_spec(1, 64, 4, 96, 50), 9)
    dw = upload_oracle_weights(W, "exact")
    x = np.random.default_rng(0).uniform(-1, 1, (7, 64)).astype(np.float32)
    q, k, v = sd.project_qkv(dw, 0, x)
    qo, ko, vo = oracle.project_qkv(W, 0, list(range(1, 8)), x)
    assert np.array_equal(q, qo) and np.array_equal(k, ko) and np.array_equal(v, vo)
    lg, tk = sd.output_logits_argmax(dw, x)
    assert np.array_equal(lg, oracle.output_logits(W, x))
    assert list(tk) == [oracle.argmax_token(r) for r in lg]
    # finish_block differs only through device expf in silu: <= a few ulp
    o = np.random.default_rng(1).uniform(-1, 1, (7, 64)).astype(np.float32)
    fb = sd.finish_block(dw, 0, o, x)
    assert np.abs(fb - oracle.finish_block(W, 0, o, x)).max() < 1e-5


def test_monolithic_generation_matches_oracle(sd, oracle):
    # proj/tests/test_workers.cpp:280-321: identical tokens, activations <= 1e-5
    W, dw, kv, eng = _engine(sd, oracle, (2, 64, 4, 256, 128))
    recs, acts, _ = sd.run_generation(eng, 8, 32, 32, 32, seed=0, record_activations=True)
    orecs, oacts = oracle.run_monolithic(W, 8, 32, 32, 32, seed=0, record=True)
    assert recs == orecs
    assert np.abs(acts - oacts).max() <= 1e-5


def test_stabilized_schedule_with_retirement(sd, oracle):
    # proj/tests/test_workers.cpp:323-344
    W, dw, kv, eng = _engine(sd, oracle, (2, 64, 4, 256, 128))
    recs, acts, _ = sd.run_generation(eng, 8, 16, 4, 48, seed=0, record_activations=True)
    orecs, oacts = oracle.run_monolithic(W, 8, 16, 4, 48, seed=0, record=True)
    assert recs == orecs
    assert np.abs(acts - oacts).max() <= 1e-5
    recs, _, _ = sd.run_generation(eng, 12, 16, 4, 0, seed=0)
    c = collections.Counter(q for _, q, _ in recs)
    assert set(c.values()) == {16}


@pytest.mark.parametrize("mode", ["exact", "bf16"])
def test_two_minibatch_pipeline_matches_oracle(sd, oracle, mode):
    """The S/R-overlapped two-mini-batch step (seq % 2 groups on two streams,
    workers.cpp:405-452) computes the same decode as the monolithic oracle."""
    W, dw, kv, eng = _engine(sd, oracle, (2, 64, 4, 256, 128), mode=mode)
    eng.pipeline(True, 100)
    recs, acts, _ = sd.run_generation(eng, 8, 16, 4, 48, seed=0, record_activations=True)
    orecs, oacts = oracle.run_monolithic(W, 8, 16, 4, 48, seed=0, record=True)
    assert recs == orecs
    if mode == "exact":
        assert np.abs(acts - oacts).max() <= 1e-5
    with open(os.path.join(GOLDEN, "golden_transcript_2x64_3seq_20.csv")) as f:
        golden = f.read()
    W2, dw2, kv2, eng2 = _engine(sd, oracle, (2, 64, 4, 256, 128), mode=mode)
    eng2.pipeline(True, 64)
    recs2, _, _ = sd.run_generation(eng2, 3, 20, 20, 20, seed=0)
    assert sd.transcript_csv(recs2) == golden


def test_c1_tiny_config_matches_oracle(sd, oracle):
    """BASELINE config 1: 2 layers, d=256 (hd 128), batch 16, context 128, fp32."""
    W, dw, kv, eng = _engine(sd, oracle, (2, 256, 2, 1024, 256))
    recs, acts, _ = sd.run_generation(eng, 16, 128, 128, 128, seed=0, record_activations=True)
    orecs, oacts = oracle.run_monolithic(W, 16, 128, 128, 128, seed=0, record=True, threads=8)
    assert recs == orecs
    assert np.abs(acts - oacts).max() <= 1e-4


def test_engine_capacity_error_is_typed(sd, oracle):
    W, dw, kv, eng = _engine(sd, oracle, (2, 64, 4, 256, 128), cap=4)
    toks = [1, 2, 3]
    eng.compute([1, 2, 3], tokens=toks)
    with pytest.raises(sd.CapacityError):
        eng.compute([1, 2, 3], tokens=toks)
    with pytest.raises(sd.ConfigError):
        eng.compute([1, 1], tokens=[0, 0])


@pytest.mark.parametrize("B", [256, 320, 512])
def test_chained_s_part_is_bitwise_equal_to_separate_gemms(B, monkeypatch):
    """The chained S-Part launch (W_o, MLP-in, MLP-out, next QKV / head as one
    persistent kernel with per-row-block dependencies) computes every tile
    exactly as the separate GEMM launches: tokens (through the chained head
    GEMM) and final activations are bitwise equal over several steps
    (ragged M, GQA)."""
    import numpy as np
    import paper_2403_11421_b200 as sd
    spec = sd.make_model_spec(3, 512, 8, 1024, 2048, 2)
    seqs = list(range(1, B + 1))

    def run(chain):
        if chain:
            monkeypatch.setenv("SD_CHAIN", "1")
        else:
            monkeypatch.delenv("SD_CHAIN", raising=False)
        w = sd.DeviceWeights(spec, None, "bf16", 0, seed=3)
        kv = sd.KvShard(spec, 0, 2, B * 80, "half", max_sequences=B, max_seq_len=80)
        kv.prefill_synthetic(seqs, 40)
        eng = sd.Engine(w, kv)
        tok = np.array([sd.prompt_token(0, s, spec.vocab_size) for s in seqs], np.int32)
        outs = []
        for _ in range(3):
            nxt, fx = eng.compute(seqs, tokens=tok, want_final=True)
            outs.append((nxt.copy(), fx.copy()))
            tok = nxt
        eng.close()
        kv.close()
        w.close()
        return outs

    a, b = run(True), run(False)
    for (t1, x1), (t2, x2) in zip(a, b):
        assert np.array_equal(t1, t2)
        assert np.array_equal(x1.view(np.uint32), x2.view(np.uint32))


@pytest.mark.parametrize("mode", ["bf16", "tf32"])
def test_fused_head_argmax_matches_logits_argmax(sd, oracle, mode):
    """argmax_token folded into the head GEMM's epilogue (per-tile keys,
    atomicMax per row) picks exactly the token the separate logits + argmax
    path picks, including ties across tiles (first maximum wins,
    dense.cpp:80-88): two identical head rows far apart in the vocabulary."""
    W = oracle.Weights(oracle.make_spec(2, 64, 4, 256, 1024), 3)
    tensors = [W.raw("embedding")]
    for l in range(W.spec.num_layers):
        for n in ("w_q", "w_k", "w_v", "w_o", "w_mlp_in", "w_mlp_out"):
            tensors.append(W.raw(n, l))
    head = np.array(W.raw("head"), np.float32, copy=True).reshape(64, 1024)  # (k, j): w(j, k) col-major
    head[:, 700] *= 40.0
    head[:, 900] = head[:, 700]
    tensors.append(head.reshape(-1))
    spec = sd.make_model_spec(2, 64, 4, 256, 1024)
    dw = sd.DeviceWeights(spec, tensors, mode, 0)
    x = np.random.default_rng(1).uniform(-1, 1, (40, 64)).astype(np.float32)
    seqs = list(range(1, 41))
    kv1 = sd.KvShard(spec, 0, 4, 1 << 12, "single")
    t1, _, lg = sd.Engine(dw, kv1).compute(seqs, features=x, want_logits=True)
    kv2 = sd.KvShard(spec, 0, 4, 1 << 12, "single")
    t2, _, _ = sd.Engine(dw, kv2).compute(seqs, features=x)
    assert np.array_equal(t1, np.argmax(lg, axis=1))
    assert np.array_equal(t2, t1)
    assert (t1 == 700).any() and not (t1 == 900).any()


@pytest.mark.parametrize("mode", ["bf16", "tf32"])
def test_fused_append_is_bitwise_equal(monkeypatch, mode):
    """append_lane folded into the QKV GEMM's epilogue (fp16 pages, lockstep
    layers) stores exactly the bytes the append kernel stores: KV lanes,
    tokens and final activations are bitwise equal over several steps,
    across page boundaries (P = 16 positions; 20 steps from context 9)."""
    import paper_2403_11421_b200 as sd
    spec = sd.make_model_spec(3, 512, 8, 1024, 2048, 2)
    seqs = list(range(1, 301))
    tok0 = np.array([sd.prompt_token(0, s, spec.vocab_size) for s in seqs], np.int32)

    def run(fused):
        if fused:
            monkeypatch.delenv("SD_NO_FUSED_APPEND", raising=False)
        else:
            monkeypatch.setenv("SD_NO_FUSED_APPEND", "1")
        w = sd.DeviceWeights(spec, None, mode, 0, seed=2)
        kv = sd.KvShard(spec, 0, 2, 300 * 64, "half", 0, max_sequences=300, max_seq_len=64)
        kv.prefill_synthetic(seqs, 9, salt=1)
        eng = sd.Engine(w, kv)
        tok, outs = tok0.copy(), []
        for _ in range(20):
            tok, fx = eng.compute(seqs, tokens=tok, want_final=True)
            outs.append((tok.copy(), fx.copy()))
        lanes = [kv.export_lane(q, l, which) for q in (1, 150, 300) for l in range(3) for which in (0, 1)]
        return outs, lanes

    a, la = run(True)
    b, lb = run(False)
    for (t1, x1), (t2, x2) in zip(a, b):
        assert np.array_equal(t1, t2)
        assert np.array_equal(x1.view(np.uint32), x2.view(np.uint32))
    for (x, _), (y, _) in zip(la, lb):  # fp16 pages: bytes, no scales
        assert x.size and np.array_equal(x, y)
