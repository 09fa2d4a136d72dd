"""Distributed ≡ monolithic on >= 2 GPUs (proj/tests/test_workers.cpp:280-332,
acceptance.cpp:259-301): the DistEngine's NCCL Q/K/V / O exchange over
sequence-sharded KV with one S-rank (the paper's topology) or data-parallel
S-ranks; identical tokens, activations <= 1e-5 against the oracle."""
import os
import pickle
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, args, nprocs, **kw):
    """mp.spawn whose rendezvous port (args[1]) is drawn again when another
    process took it between _free_port() and the bind (EADDRINUSE)."""
    import torch.multiprocessing as mp
    for attempt in range(3):
        try:
            return mp.spawn(fn, args=args, nprocs=nprocs, **kw)
        except Exception as e:  # ProcessRaisedException carrying the rank's DistNetworkError
            if "EADDRINUSE" not in str(e) or attempt == 2:
                raise
            args = (args[0], _free_port()) + tuple(args[2:])


TOY = (2, 64, 4, 256, 128)


def _worker(rank, world, port, s_ranks, cfg, out_path, exchange="nccl", shard_mode="sequence", drain=False,
            pipeline=False, spec_args=TOY, fmt="single"):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle"), os.path.join(root, "tests")]
    import torch
    import torch.distributed as dist
    import oracle as o
    import paper_2403_11421_b200 as sd
    from conftest import upload_oracle_weights
    # "p2p-one-device": every rank on cuda:0, no NCCL communicator; the
    # exchange and the next-token gather run as CUDA-IPC peer stores
    dev = 0 if exchange == "p2p-one-device" else rank
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    obj = [sd.nccl_unique_id() if rank == 0 and exchange != "p2p-one-device" else None]
    dist.broadcast_object_list(obj, src=0)
    W = o.Weights(o.make_spec(*spec_args), 0)
    is_s = s_ranks == world or rank == 0
    dw = upload_oracle_weights(W, "exact", device=dev) if is_s else None
    spec = sd.make_model_spec(*spec_args)
    heads = spec.num_kv_heads
    if shard_mode == "sequence":
        h0, hc = 0, heads
    else:
        h0, hc = sd.ShardMap(shard_mode, heads, world).head_range(rank)
    kv = sd.KvShard(spec, h0, hc, 1 << 16, fmt, dev)
    eng = sd.DistEngine(dw, kv, rank, world, obj[0], s_ranks, shard_mode=shard_mode)
    if exchange.startswith("p2p"):
        eng.enable_p2p(64)
    if pipeline:
        eng.pipeline(True)
    recs, acts, _ = sd.run_generation(eng, *cfg, seed=0, record_activations=True)
    rows = [(r, acts[i].tolist()) for i, r in enumerate(recs)]
    # after a run to completion every sequence has retired on every rank
    # that stores it (DROP_SEQ to all links outside by-sequence sharding,
    # workers.cpp:482-501)
    left = (kv.token_count(), kv.warning_count()) if drain else None
    allr, alll = [None] * world, [None] * world
    dist.all_gather_object(allr, rows)
    dist.all_gather_object(alll, left)
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump(([x for part in allr for x in part], alll), f)
    eng.close()
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("s_ranks", [1, 2])
@pytest.mark.parametrize("cfg", [(8, 32, 32, 32), (8, 16, 4, 48)], ids=["batch", "stabilized"])
@pytest.mark.parametrize("exchange,shard_mode,pipeline", [("nccl", "sequence", False), ("p2p", "sequence", False),
                                                          ("p2p", "head", False), ("p2p", "sequence", True)])
def test_two_gpu_distributed_equals_monolithic(oracle, tmp_path, s_ranks, cfg, exchange, shard_mode, pipeline):
    """`exchange`: NCCL grouped send/recv, or direct NVLink stores into the
    peers' receive buffers with epoch flags (dist_p2p.cu). `shard_mode`
    "head": each rank attends every sequence for its half of the heads
    (ShardMap by-head, transport.cpp:345-380) and the o slices are gathered
    back into the S-rank's rows."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "rows.pkl")
    _spawn(_worker, args=(2, _free_port(), s_ranks, cfg, out, exchange, shard_mode, False, pipeline), nprocs=2,
             join=True)
    _check_rows(oracle, out, cfg)


def _check_rows(oracle, out, cfg, spec_args=TOY, fmt="single", bar=1e-5):
    rows, left = pickle.load(open(out, "rb"))
    W = oracle.Weights(oracle.make_spec(*spec_args), 0)
    orecs, oacts = oracle.run_monolithic(W, *cfg, seed=0, fmt=fmt, record=True)
    ref = {(s, q): (t, oacts[i]) for i, (s, q, t) in enumerate(orecs)}
    assert len(rows) == len(ref)
    worst = 0.0
    for (s, q, t), x in rows:
        rt, rx = ref[(s, q)]
        assert t == rt
        worst = max(worst, float(np.abs(np.asarray(x, np.float32) - rx).max()))
    assert worst <= bar
    return left


def _fused_worker(rank, world, port, out_path, s_ranks):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root]
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2403_11421_b200 as sd
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    spec = sd.make_model_spec(2, 1024, 8, 1024, 512, 2)
    seqs = list(range(1, 97))
    B = len(seqs)
    results = {}
    homes = ("affinity", "modulo") if s_ranks == world else ("affinity",)
    for home_policy in homes:
        for fused in (True, False):
            sd.tune("dist_fuse", int(fused))
            obj = [sd.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            is_s = s_ranks == world or rank == 0
            w = sd.DeviceWeights(spec, None, "bf16", rank, seed=5) if is_s else None
            plan = sd.dist_plan(world, rank, s_ranks, seqs, home=home_policy)
            mine = [seqs[i] for i in plan["shard_rows"]]  # prefill is sequence-keyed
            kv = sd.KvShard(spec, 0, 2, 96 * 64, "half", rank, max_sequences=96, max_seq_len=64)
            kv.prefill_synthetic(mine, 20, salt=0)
            eng = sd.DistEngine(w, kv, rank, world, obj[0], s_ranks, home=home_policy)
            eng.enable_p2p(len(seqs))
            tok = np.array([sd.prompt_token(0, s, spec.vocab_size) for s in seqs], np.int32)
            outs = []
            for _ in range(3):
                nxt, fx = eng.compute(seqs, tok, want_final=True)
                home = np.asarray(plan["home_rows"], np.int64)
                allt = [None] * world
                dist.all_gather_object(allt, (home.tolist(), nxt[home].tolist(), fx[home].tolist()))
                full_t = np.zeros(B, np.int32)
                full_x = np.zeros((B, spec.model_dim), np.float32)
                for h, t, x in allt:
                    full_t[np.asarray(h, np.int64)] = np.asarray(t, np.int32)
                    full_x[np.asarray(h, np.int64)] = np.asarray(x, np.float32).reshape(-1, spec.model_dim)
                outs.append((full_t, full_x))
                tok = full_t.copy()
            results[(home_policy, fused)] = outs
            eng.close()
            kv.close()
            if w is not None:
                w.close()
            dist.barrier()
    # fused vs scatter: bitwise under each placement
    ok = all(np.array_equal(a[0], b[0]) and np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
             for h in homes for a, b in zip(results[(h, True)], results[(h, False)]))
    # across placements a shard attends the same rows in another order (the
    # split-K plan follows the order) and a last-bit change of an attention
    # output can flip a bf16 operand rounding in the next GEMM: same tokens,
    # activations within the bf16 S-Part's relative precision (2^-8 per
    # rounding, a few roundings deep)
    worst = 0.0
    for h in homes[1:]:
        for a, b in zip(results[(homes[0], True)], results[(h, True)]):
            ok = ok and np.array_equal(a[0], b[0])
            worst = max(worst, float(np.abs(a[1] - b[1]).max() / max(np.abs(a[1]).max(), 1e-30)))
    ok = ok and worst <= 2e-2
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        with open(out_path, "w") as f:
            f.write("ok" if all(flags) else f"mismatch (relative placement delta {worst:g})")
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("s_ranks", [1, 2])
def test_two_gpu_fused_exchange_is_bitwise_equal(tmp_path, s_ranks):
    """The exchange fused into the producers (the QKV GEMM epilogue stores each
    home row into its shard's receive buffer over NVLink; the attention stores
    o rows into the home rank's buffer; the last CTA of each publishes the
    epoch) moves exactly the bytes of the separate scatter kernel: tokens and
    final activations of the whole batch are bitwise equal over three steps,
    under either S-Part placement (balanced shard-affine homes, seq % world).
    Between the placements tokens match and activations agree within the
    bf16 S-Part's relative precision."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "fused.txt")
    _spawn(_fused_worker, args=(2, _free_port(), out, s_ranks), nprocs=2, join=True)
    assert open(out).read() == "ok"


@pytest.mark.skipif(_ngpus() < 1, reason="needs a GPU")
@pytest.mark.parametrize("pipeline", [False, True], ids=["one-batch", "two-minibatches"])
@pytest.mark.parametrize("s_ranks", [1, 2])
@pytest.mark.parametrize("shard_mode", ["sequence", "head", "hybrid"])
def test_two_ranks_one_device_distributed_equals_monolithic(oracle, tmp_path, s_ranks, shard_mode, pipeline):
    """DistributedComputation with two ranks on ONE device (two processes,
    no NCCL: the per-layer Q/K/V and O exchange and the next-token gather are
    CUDA-IPC peer stores with epoch flags), run to completion: tokens equal
    the monolithic oracle's, activations <= 1e-5 (test_workers.cpp:280-321),
    and every rank's shard is empty afterwards with no drop warnings, in all
    three ShardMap modes (retire routing, workers.cpp:482-501). With the
    reference's two interleaved mini-batches (seq % 2, workers.cpp:405-452)
    the transcript is the same."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "rows.pkl")
    cfg = (8, 16, 4, 0)
    _spawn(_worker, args=(2, _free_port(), s_ranks, cfg, out, "p2p-one-device", shard_mode, True, pipeline),
             nprocs=2, join=True)
    left = _check_rows(oracle, out, cfg)
    assert left == [(0, 0), (0, 0)]


@pytest.mark.skipif(_ngpus() < 1, reason="needs a GPU")
@pytest.mark.parametrize("s_ranks", [1, 4])
def test_four_ranks_one_device_hybrid_shardmap(oracle, tmp_path, s_ranks):
    """ShardMap hybrid with two sequence groups (4 workers over 2 kv heads:
    HG = gcd(4, 2) = 2 head groups x SG = 2 sequence groups,
    transport.cpp:354-376): four ranks on one device, run to completion,
    tokens equal the monolithic oracle, activations <= 1e-5, every shard
    empty afterwards."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "rows.pkl")
    cfg = (8, 12, 4, 0)
    spec_args = (2, 64, 2, 256, 128)
    _spawn(_worker, args=(4, _free_port(), s_ranks, cfg, out, "p2p-one-device", "hybrid", True, False, spec_args),
             nprocs=4, join=True)
    left = _check_rows(oracle, out, cfg, spec_args)
    assert left == [(0, 0)] * 4


@pytest.mark.parametrize("shard_mode,s_ranks", [("sequence", 1), ("sequence", 8), ("hybrid", 8)])
def test_eight_ranks_one_device(oracle, tmp_path, shard_mode, s_ranks):
    """The full 8-rank geometry of one 8xB200 box (flag slots, peer maps and
    the token gather at their maximum width) on the driver's one device:
    by-sequence with one or eight S-ranks, and hybrid (8 workers over 4 kv
    heads: 4 head groups x 2 sequence groups); tokens equal the monolithic
    oracle, every shard empty after retirement."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "rows.pkl")
    cfg = (16, 12, 4, 0)
    spec_args = (2, 64, 4, 256, 128)
    _spawn(_worker, args=(8, _free_port(), s_ranks, cfg, out, "p2p-one-device", shard_mode, True, False, spec_args),
             nprocs=8, join=True)
    left = _check_rows(oracle, out, cfg, spec_args)
    assert left == [(0, 0)] * 8


@pytest.mark.parametrize("fmt", ["half", "int8", "int4"])
@pytest.mark.parametrize("shard_mode", ["sequence", "hybrid"])
def test_two_ranks_one_device_stored_kv_formats(oracle, tmp_path, fmt, shard_mode):
    """The distributed step over fp16 / int8 / int4 KV shards (two ranks, one
    device): the same transcript as the oracle's run_monolithic over a
    KvShard in that format, activations <= 1e-4."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "rows.pkl")
    cfg = (8, 16, 4, 0)
    _spawn(_worker, args=(2, _free_port(), 2, cfg, out, "p2p-one-device", shard_mode, True, False, TOY, fmt),
             nprocs=2, join=True)
    left = _check_rows(oracle, out, cfg, TOY, fmt, 1e-4)
    assert left == [(0, 0), (0, 0)]
