"""The reference's own `run` measurement on one B200: drive_schedule
(workers.cpp:547-684) with the SLS cold start (scheduler.cpp) over the GPU
StepComputation, tokens emitted / wall seconds as summarize_run computes it
(workers.cpp:713-733). Sequences start from one prompt token and decode to
target_len, so KV lengths are ragged (SURVEY §8d synthetic inputs (ii)):
after the cold start, S/F micro-batches of B*F/S rows sit at every length
step of F, mean ~ (S+F)/2.

Two drives of the same config at different step counts give the steady
window by difference: (tokens2 - tokens1) / (wall2 - wall1).

  python tools/sls_run.py [--batch 512] [--target 2048] [--interval 256] [--model 8b] [--kv half]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd

SHAPES = {"8b": (32, 4096, 32, 14336, 128256, 8), "7b": (32, 4096, 32, 11008, 32000, 32)}

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="8b", choices=sorted(SHAPES))
ap.add_argument("--batch", type=int, default=512)
ap.add_argument("--target", type=int, default=2048)
ap.add_argument("--interval", type=int, default=256)
ap.add_argument("--kv", default="half")
ap.add_argument("--dense", default="fp16")
ap.add_argument("--extra", type=int, default=512, help="steady steps measured past the cold start")
a = ap.parse_args()

L, D, H, F, V, Hkv = SHAPES[a.model]
spec = sd.make_model_spec(L, D, H, F, V, Hkv)
w = sd.DeviceWeights(spec, None, a.dense, 0, seed=0, generator="reference")


def drive(steps):
    kv = sd.KvShard(spec, 0, Hkv, a.batch * (a.target + 1), a.kv, 0, max_sequences=2 * a.batch + 64,
                    max_seq_len=a.target + 16)
    eng = sd.Engine(w, kv)
    recs, _, wall = sd.run_generation(eng, a.batch, a.target, a.interval, steps, seed=0)
    per_step = {}
    for st, _, _ in recs:
        per_step[st] = per_step.get(st, 0) + 1
    eng.close()
    kv.close()
    return len(recs), wall, per_step


s1 = a.target + a.interval
s2 = s1 + a.extra
n1, w1, ps1 = drive(s1)
n2, w2, ps2 = drive(s2)
steady_rows = [ps2[s] for s in range(s1 + 1, s2 + 1) if s in ps2]
out = {
    "what": "drive_schedule over the GPU StepComputation (reference `run` metric: tokens / wall seconds)",
    "model": a.model, "batch": a.batch, "target_len": a.target, "interval": a.interval, "kv": a.kv,
    "dense": a.dense, "cold_start": "fixed-interval",
    "run_to_steps": [s1, s2], "tokens": [n1, n2], "wall_s": [w1, w2],
    "tokens_per_s_including_cold_start": [n1 / w1, n2 / w2],
    "steady_window": {"steps": [s1 + 1, s2], "tokens": n2 - n1, "wall_s": w2 - w1,
                      "tokens_per_s": (n2 - n1) / (w2 - w1),
                      "rows_per_step_min_max": [min(steady_rows), max(steady_rows)] if steady_rows else None,
                      "mean_kv_length": (a.target + a.interval) / 2},
}
print(json.dumps(out))
