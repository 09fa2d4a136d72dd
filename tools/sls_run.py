"""The reference's own `run` measurement on B200s: drive_schedule
(workers.cpp:547-684) with the SLS cold start (scheduler.cpp) over the GPU
StepComputation (N = 1) or the DistributedComputation (N > 1, one process
per GPU, KV sharded by the reference's ShardMap, NVLink peer exchange),
tokens emitted / wall seconds as summarize_run computes it
(workers.cpp:713-733). Sequences start from one prompt token and decode to
target_len, so KV lengths are ragged (SURVEY §8d synthetic inputs (ii)):
after the cold start, S/F micro-batches of B*F/S rows sit at every length
step of F, mean ~ (S+F)/2.

After an untimed short drive (one-time setup), two drives of the same
config at different step counts give the steady window by difference: (tokens2 - tokens1) / (wall2 - wall1). With N > 1 the
batch is B per GPU (weak scaling, as bench.py), every rank an S-rank (the
data-parallel topology) unless --s-ranks 1; tokens are summed over ranks,
wall is the max over ranks.

  python tools/sls_run.py [--gpus N] [--batch 512] [--target 2048] [--interval 256] [--model 8b]
"""
import argparse
import json
import os
import socket
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {"8b": (32, 4096, 32, 14336, 128256, 8), "7b": (32, 4096, 32, 11008, 32000, 32)}

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=1)
ap.add_argument("--model", default="8b", choices=sorted(SHAPES))
ap.add_argument("--batch", type=int, default=512, help="rows per GPU")
ap.add_argument("--target", type=int, default=2048)
ap.add_argument("--interval", type=int, default=256)
ap.add_argument("--kv", default="half")
ap.add_argument("--dense", default="fp16")
ap.add_argument("--s-ranks", type=int, default=0, help="N > 1: S-workers (1 = the paper's single S-rank; 0 = every rank)")
ap.add_argument("--extra", type=int, default=512, help="steady steps measured past the cold start")
a = ap.parse_args()

if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))

import torch  # noqa: E402
import paper_2403_11421_b200 as sd  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("gloo")

L, D, H, F, V, Hkv = SHAPES[a.model]
spec = sd.make_model_spec(L, D, H, F, V, Hkv)
B = a.batch * world
s_ranks = world if a.s_ranks == 0 else a.s_ranks
is_s = world == 1 or s_ranks == world or rank == 0
w = sd.DeviceWeights(spec, None, a.dense, local, seed=0, generator="reference") if is_s else None


def drive(steps):
    if world == 1:
        cap = B * (a.target + 1)
    else:  # SLS keeps <= B (S+F)/2 live tokens; a shard holds ~1/world of them (mix64 hash, margin)
        cap = int(B / world * 1.2 + 64) * ((a.target + a.interval) // 2 + 64)
    kv = sd.KvShard(spec, 0, Hkv, cap, a.kv, local, max_sequences=2 * B + 64, max_seq_len=a.target + 16)
    if world == 1:
        eng = sd.Engine(w, kv)
    else:
        eng = sd.DistEngine(w, kv, rank, world, None, s_ranks)
        eng.enable_p2p(B)
    recs, _, wall = sd.run_generation(eng, B, a.target, a.interval, steps, seed=0)
    eng.close()
    kv.close()
    n = len(recs)
    per_step = {}
    for st, _, _ in recs:
        per_step[st] = per_step.get(st, 0) + 1
    if dist is not None:
        t = torch.tensor([float(n), wall], dtype=torch.float64)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        n = int(sum(p[0].item() for p in parts))
        wall = max(p[1].item() for p in parts)
    return n, wall, per_step


s1 = a.target + a.interval
s2 = s1 + a.extra
drive(2 * a.interval)  # untimed: first-touch allocations and one-time setup stay out of drive 1
n1, w1, _ = drive(s1)
n2, w2, ps2 = drive(s2)
steady_rows = [ps2[s] for s in range(s1 + 1, s2 + 1) if s in ps2] if world == 1 else []
if rank == 0:
    print(json.dumps({
        "what": "drive_schedule over the GPU " + ("StepComputation" if world == 1 else
                                                   f"DistributedComputation ({world} GPUs, {s_ranks} S-rank(s))")
                + " (reference `run` metric: tokens / wall seconds)",
        "model": a.model, "gpus": world, "batch": B, "target_len": a.target, "interval": a.interval, "kv": a.kv,
        "dense": a.dense, "cold_start": "fixed-interval",
        "run_to_steps": [s1, s2], "tokens": [n1, n2], "wall_s": [w1, w2],
        "tokens_per_s_including_cold_start": [n1 / w1, n2 / w2],
        "steady_window": {"steps": [s1 + 1, s2], "tokens": n2 - n1, "wall_s": w2 - w1,
                          "tokens_per_s": (n2 - n1) / (w2 - w1),
                          "rows_per_step_min_max": [min(steady_rows), max(steady_rows)] if steady_rows else None,
                          "mean_kv_length": (a.target + a.interval) / 2},
    }), flush=True)
if dist is not None:
    dist.barrier()
    dist.destroy_process_group()
