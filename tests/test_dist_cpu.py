"""Multi-GPU host logic on CPU: the distributed step's row plan (sd_dist_plan)
and a world-size-2 gloo run of DistributedComputation's exchange protocol
(workers.cpp:399-501) with oracle S- and R-workers, checked against the
monolithic oracle (test_workers.cpp:280-332 intent)."""
import os
import socket

import numpy as np
import pytest


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


def _affinity_homes(world, seqs, oracle):
    """Restatement of the balanced shard-affine home assignment
    (dist.cpp assign_homes): quotas floor/ceil(B / world), rows fill their
    KV rank's quota in batch order, the overflow fills the rest in rank order."""
    B = len(seqs)
    quota = [B // world + (1 if r < B % world else 0) for r in range(world)]
    cnt, home, over = [0] * world, [0] * B, []
    for i, q in enumerate(seqs):
        r = oracle.shardmap_worker_for("by-sequence", 8, world, q, 0)
        if cnt[r] < quota[r]:
            home[i], cnt[r] = r, cnt[r] + 1
        else:
            over.append(i)
    r = 0
    for i in over:
        while cnt[r] >= quota[r]:
            r += 1
        home[i], cnt[r] = r, cnt[r] + 1
    return home


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("s_mode", ["single", "all"])
@pytest.mark.parametrize("home", ["affinity", "modulo"])
def test_plan_partitions_rows_and_follows_shardmap(oracle, world, s_mode, home):
    import paper_2403_11421_b200 as sd
    s_ranks = 1 if s_mode == "single" else world
    rng = np.random.default_rng(world)
    seqs = [int(x) for x in rng.choice(10**6, size=97, replace=False) + 1]
    plans = [sd.dist_plan(world, r, s_ranks, seqs, home=home) for r in range(world)]
    homes = sorted(i for p in plans for i in p["home_rows"])
    shards = sorted(i for p in plans for i in p["shard_rows"])
    assert homes == list(range(len(seqs))) and shards == list(range(len(seqs)))
    if s_ranks == 1:
        want = [0] * len(seqs)
    elif home == "modulo":
        want = [q % s_ranks for q in seqs]
    else:
        want = _affinity_homes(world, seqs, oracle)
    for r, p in enumerate(plans):
        for i in p["shard_rows"]:  # ShardMap by-sequence, bit-exact (transport.cpp:352-353)
            assert oracle.shardmap_worker_for("by-sequence", 8, world, seqs[i], 0) == r
        for i in p["home_rows"]:
            assert want[i] == r
    if s_ranks == world and home == "affinity":
        # balanced S-Part, and only the unavoidable rows cross between ranks
        B = len(seqs)
        assert all(len(p["home_rows"]) in (B // world, -(-B // world)) for p in plans)
        shard_n = [len(p["shard_rows"]) for p in plans]
        quota = [B // world + (1 if r < B % world else 0) for r in range(world)]
        cross = sum(c for r, p in enumerate(plans) for d, c in enumerate(p["send_counts"]) if d != r)
        assert cross == sum(max(0, n - q) for n, q in zip(shard_n, quota))
    for r in range(world):
        for d in range(world):
            assert plans[r]["send_counts"][d] == plans[d]["recv_counts"][r]
    # rank d receives rank r's rows in r's send order
    for r in range(world):
        off_s = np.cumsum([0] + plans[r]["send_counts"])
        for d in range(world):
            off_r = np.cumsum([0] + plans[d]["recv_counts"])
            sent = plans[r]["home_rows"][off_s[d]:off_s[d + 1]]
            got = plans[d]["shard_rows"][off_r[r]:off_r[r + 1]]
            assert sent == got


@pytest.mark.parametrize("mode,world,heads", [("head", 2, 8), ("head", 4, 8), ("head", 8, 8), ("head", 3, 8),
                                              ("hybrid", 4, 2), ("hybrid", 8, 4), ("hybrid", 6, 4),
                                              ("hybrid", 2, 3)])
@pytest.mark.parametrize("s_mode", ["single", "all"])
def test_plan_head_and_hybrid_sharding(oracle, mode, world, heads, s_mode):
    """By-head / hybrid ShardMap on the data path: worker w holds the kv heads
    of its head group for the sequences of its sequence group; every (row,
    head group) is attended exactly once, by the worker the reference's
    ShardMap names (transport.cpp:345-380), and each worker receives an
    S-rank's rows in that S-rank's send order."""
    import paper_2403_11421_b200 as sd
    s_ranks = 1 if s_mode == "single" else world
    rng = np.random.default_rng(world * 10 + heads)
    seqs = [int(x) for x in rng.choice(10**6, size=61, replace=False) + 1]
    plans = [sd.dist_plan(world, r, s_ranks, seqs, mode, heads) for r in range(world)]
    name = "by-head" if mode == "head" else "hybrid"
    sm = sd.ShardMap(name, heads, world)
    ranges = [sm.head_range(w) for w in range(world)]
    assert sorted(i for p in plans for i in p["home_rows"]) == list(range(len(seqs)))
    # per head group, the shard rows partition the batch
    groups = {}
    for w, (h0, hc) in enumerate(ranges):
        groups.setdefault((h0, hc), []).append(w)
    for (h0, hc), ws in groups.items():
        rows = sorted(i for w in ws for i in plans[w]["shard_rows"])
        assert rows == list(range(len(seqs)))
        for w in ws:
            for i in plans[w]["shard_rows"]:
                assert oracle.shardmap_worker_for(name, heads, world, seqs[i], h0) == w
    for r in range(world):
        for d in range(world):
            assert plans[r]["send_counts"][d] == plans[d]["recv_counts"][r]
            off_r = np.cumsum([0] + plans[d]["recv_counts"])
            got = plans[d]["shard_rows"][off_r[r]:off_r[r + 1]]
            sent = [i for i in plans[r]["home_rows"]
                    if oracle.shardmap_worker_for(name, heads, world, seqs[i], ranges[d][0]) == d]
            assert got == sent


def test_plan_head_mode_rejects_more_workers_than_heads():
    import paper_2403_11421_b200 as sd
    with pytest.raises(sd.ConfigError):
        sd.dist_plan(4, 0, 4, [1, 2, 3], "head", 2)


def _gloo_worker(rank, world, port, s_ranks, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import torch
    import torch.distributed as dist
    import oracle as o
    import paper_2403_11421_b200 as sd
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    spec = o.make_spec(2, 64, 4, 256, 128)
    W = o.Weights(spec, 0)
    emb = W.tensor("embedding")
    kv = o.KvShard(spec, 0, 4, 1 << 12)  # this rank's R-shard
    seqs = list(range(1, 9))
    tokens = {q: o.prompt_token(0, q, 128) for q in seqs}
    D, qkvw = 64, 3 * 64
    out = []
    for step in range(6):
        plan = sd.dist_plan(world, rank, s_ranks, seqs)
        home, shard = plan["home_rows"], plan["shard_rows"]
        x = np.stack([emb[:, tokens[seqs[i]]] for i in home]).astype(np.float32) if home else np.zeros((0, D), np.float32)
        for layer in range(2):
            # S-Part on home rows (project_qkv), scatter to shards (send_layer)
            if home:
                q, k, v = o.project_qkv(W, layer, [seqs[i] for i in home], x)
                qkv = np.concatenate([q, k, v], axis=1)
            else:
                qkv = np.zeros((0, qkvw), np.float32)
            recv = torch.zeros(len(shard) * qkvw)
            dist.all_to_all_single(recv, torch.from_numpy(qkv.reshape(-1).copy()),
                                   [c * qkvw for c in plan["recv_counts"]],
                                   [c * qkvw for c in plan["send_counts"]])
            r = recv.numpy().reshape(len(shard), qkvw)
            # R-Part on the shard (AttentionWorkerSession QKV handler)
            ids = [seqs[i] for i in shard]
            if ids:
                pos = [kv.stored_length(s, layer) for s in ids]
                kv.append_request(layer, ids, pos, r[:, D:2 * D], r[:, 2 * D:])
                oo = kv.attend(layer, ids, r[:, :D])
            else:
                oo = np.zeros((0, D), np.float32)
            # gather O back to the S-ranks (receive_layer)
            back = torch.zeros(len(home) * D)
            dist.all_to_all_single(back, torch.from_numpy(oo.reshape(-1).copy()),
                                   [c * D for c in plan["send_counts"]],
                                   [c * D for c in plan["recv_counts"]])
            if home:
                x = o.finish_block(W, layer, back.numpy().reshape(len(home), D), x)
        nxt = {}
        if home:
            lg = o.output_logits(W, x)
            for j, i in enumerate(home):
                nxt[seqs[i]] = o.argmax_token(lg[j])
                out.append((step, seqs[i], nxt[seqs[i]], x[j].tolist()))
        # tokens are needed only by the home rank; share them for the next step
        allm = [None] * world
        dist.all_gather_object(allm, nxt)
        for m in allm:
            tokens.update(m)
    allo = [None] * world
    dist.all_gather_object(allo, out)
    if rank == 0:
        import pickle
        with open(out_path, "wb") as f:
            pickle.dump([r for part in allo for r in part], f)
    dist.destroy_process_group()


@pytest.mark.parametrize("s_ranks", [1, 2])
def test_gloo_two_ranks_equal_monolithic(oracle, tmp_path, s_ranks):
    import pickle
    import torch.multiprocessing as mp
    out = str(tmp_path / "rows.pkl")
    _spawn(_gloo_worker, args=(2, _free_port(), s_ranks, out), nprocs=2, join=True)
    rows = pickle.load(open(out, "rb"))
    # monolithic oracle over the same batch and steps
    spec = oracle.make_spec(2, 64, 4, 256, 128)
    W = oracle.Weights(spec, 0)
    emb = W.tensor("embedding")
    kv = oracle.KvShard(spec, 0, 4, 1 << 12)
    seqs = list(range(1, 9))
    toks = [oracle.prompt_token(0, q, 128) for q in seqs]
    ref = {}
    for step in range(6):
        x = np.stack([emb[:, t] for t in toks]).astype(np.float32)
        nt, fx, _ = oracle.decode_step_monolithic(W, kv, seqs, x)
        for i, q in enumerate(seqs):
            ref[(step, q)] = (int(nt[i]), fx[i])
        toks = [int(t) for t in nt]
    assert len(rows) == len(ref)
    for step, q, tok, x in rows:
        rt, rx = ref[(step, q)]
        assert tok == rt
        assert np.array_equal(np.asarray(x, np.float32), rx)  # row-independent math: bitwise
