"""tcgen05 GEMM parity (S-Part, dense.cpp:16-70) in the tensor-core modes.

Reference: float64 products of the operands as the tensor core sees them
(bf16-rounded activations and weights for kind::f16; tf32-truncated for
kind::tf32), so the only difference left is the fp32 accumulation order:
tolerance 2e-5 relative to the row's |x|.|w| scale. Against the exact fp32
reference the end-to-end bound is the operand rounding itself (bf16 2^-9,
tf32 2^-11 relative per product), checked on whole decode runs below."""
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


def fp16(x):
    return np.ascontiguousarray(x, np.float32).astype(np.float16).astype(np.float32)


def bf16(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def tf32(x):
    # tensor cores read the top 19 bits of the fp32 operand (truncation);
    # allow either truncation or round-to-nearest in the tolerance below
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return (u & np.uint32(0xFFFFE000)).view(np.float32)


def _ref(x, wT, mode):
    r = {"bf16": bf16, "fp16": fp16, "tf32": tf32}[mode]
    xe, we = r(x).astype(np.float64), r(wT).astype(np.float64)
    return xe @ we, np.abs(xe) @ np.abs(we)


SHAPES = [(2, 64, 4, 256, 128), (1, 512, 8, 1024, 1000), (1, 256, 2, 512, 300)]


@pytest.mark.parametrize("mode", ["bf16", "fp16", "tf32"])
@pytest.mark.parametrize("shape", SHAPES, ids=["toy", "d512", "d256"])
@pytest.mark.parametrize("B", [1, 3, 130, 257])
def test_linear_matches_rounded_reference(sd, oracle, mode, shape, B):
    W = oracle.Weights(oracle.make_spec(*shape), 3)
    dw = upload_oracle_weights(W, mode)
    D, F = shape[1], shape[3]
    rng = np.random.default_rng(B)
    for which, name, n_in in ((4, "w_o", D), (5, "w_mlp_in", D), (6, "w_mlp_out", F), (7, "head", D)):
        x = rng.uniform(-1, 1, (B, n_in)).astype(np.float32)
        y = sd.apply_linear(dw, 0, which, x)
        wT = W.tensor(name).T  # (in, out)
        ref, scale = _ref(x, wT, mode)
        tol = 1e-3 if mode == "tf32" else 2e-5  # tf32: rounding mode of operands unspecified
        assert np.all(np.abs(y - ref) <= tol * scale + 1e-6), (which, float(np.abs(y - ref).max()))


@pytest.mark.parametrize("mode", ["bf16", "fp16", "tf32"])
def test_fused_epilogues(sd, oracle, mode):
    W = oracle.Weights(oracle.make_spec(1, 512, 8, 1024, 64), 5)
    dw = upload_oracle_weights(W, mode)
    rng = np.random.default_rng(7)
    o = rng.uniform(-1, 1, (77, 512)).astype(np.float32)
    res = rng.uniform(-1, 1, (77, 512)).astype(np.float32)
    got = sd.finish_block(dw, 0, o, res)
    exact = oracle.finish_block(W, 0, o, res)
    rel = 2.0**-7 if mode == "bf16" else 2.0**-9  # fp16 / tf32: 11-bit significands
    assert np.abs(got - exact).max() <= rel * max(1.0, float(np.abs(exact).max()))


@pytest.mark.parametrize("mode", ["bf16", "fp16", "tf32"])
def test_golden_transcript_tensor_core_modes(sd, oracle, mode):
    """The reference transcript survives tensor-core operand rounding
    (SURVEY §0 finding 2: minimum top-1/top-2 logit margin 4.3e-3)."""
    W = oracle.Weights(oracle.make_spec(2, 64, 4, 256, 128), 0)
    dw = upload_oracle_weights(W, mode)
    kv = sd.KvShard(dw.spec, 0, 4, 1 << 16)
    eng = sd.Engine(dw, kv)
    recs, _, _ = sd.run_generation(eng, 3, 20, 20, 20, seed=0)
    with open(os.path.join(GOLDEN, "golden_transcript_2x64_3seq_20.csv")) as f:
        assert sd.transcript_csv(recs) == f.read()


@pytest.mark.parametrize("kind", ["bf16", "fp16", "tf32"])
@pytest.mark.parametrize("M,N,K", [(512, 1024, 512), (300, 640, 256), (1000, 2080, 384), (384, 96, 128)])
def test_pair_tile_variants_are_bitwise_equal(sd, kind, M, N, K):
    """Every pair-tile variant accumulates each output over the same K
    sequence of MMAs: the 128 / 192 / 256 instantiations picked by tile width
    (tile widths 112 / 176 / 208 and the cost model's choice), and single-CTA
    tiles. Outputs are bitwise equal for every epilogue (plain, residual +
    16-bit copy, SiLU), ragged M included, and match the rounded reference."""
    import torch
    dev = torch.device("cuda")
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "tf32": torch.float32}[kind]
    cdt = torch.float16 if kind == "fp16" else torch.bfloat16
    A = (torch.rand(M, K, generator=g) * 2 - 1).to(dt).to(dev)
    B = ((torch.rand(N, K, generator=g) * 2 - 1) / K**0.5).to(dt).to(dev)
    res = (torch.rand(M, N, generator=g) * 2 - 1).to(dev)
    variants = [{}] + [{"gemm_bn": bn} for bn in (112, 176, 208)]
    outs = []
    for tv in variants:
        with sd.tuned(**tv):
            C0 = torch.empty(M, N, device=dev)
            C1 = torch.empty(M, N, device=dev)
            Cb1 = torch.empty(M, N, device=dev, dtype=cdt)
            C2 = torch.empty(M, N, device=dev)
            sd.gemm_dev(kind, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C0.data_ptr(), N)
            sd.gemm_dev(kind, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C1.data_ptr(), N, Cb1.data_ptr(), N,
                        epi=1, res=res.data_ptr(), ldr=N)
            sd.gemm_dev(kind, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C2.data_ptr(), N, epi=2)
            torch.cuda.synchronize()
            outs.append([t.cpu() for t in (C0, C1, Cb1, C2)])
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert torch.equal(a.view(torch.int16) if a.element_size() == 2 else a.view(torch.int32),
                               b.view(torch.int16) if b.element_size() == 2 else b.view(torch.int32))
    # the 16-bit copy is the RNE conversion of the fp32 result
    assert torch.equal(outs[0][2].view(torch.int16), outs[0][1].to(cdt).view(torch.int16))
    ref = A.float().cpu().double() @ B.float().cpu().double().T
    scale = A.float().cpu().double().abs() @ B.float().cpu().double().abs().T
    tol = 1e-3 if kind == "tf32" else 2e-5
    assert bool(((outs[0][0].double() - ref).abs() <= tol * scale + 1e-6).all())


@pytest.mark.parametrize("kind", ["bf16", "fp16", "tf32"])
def test_single_cta_tiles_match_pair_tiles(sd, kind):
    """gemm_pair=0 (single-CTA 128-row tiles) against the CTA-pair tiles: the
    same MMAs per output, bitwise equal."""
    import torch
    M, N, K = 640, 1536, 512
    g = torch.Generator(device="cpu").manual_seed(11)
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "tf32": torch.float32}[kind]
    A = (torch.rand(M, K, generator=g) * 2 - 1).to(dt).cuda()
    B = ((torch.rand(N, K, generator=g) * 2 - 1) / K**0.5).to(dt).cuda()
    outs = []
    for pair in (1, 0):
        with sd.tuned(gemm_pair=pair):
            C = torch.empty(M, N, device="cuda")
            sd.gemm_dev(kind, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
            torch.cuda.synchronize()
            outs.append(C.cpu())
    assert torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))
