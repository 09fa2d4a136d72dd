"""R-Part microbenchmark: attention kernel GB/s on synthetic prefilled KV
(one layer). Usage: python tools/bench_rpart.py [--D 4096 --H 32 --Hkv 32 --B 1024 --L 1024 --fmt half]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd

ap = argparse.ArgumentParser()
ap.add_argument("--D", type=int, default=4096)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--Hkv", type=int, default=0)
ap.add_argument("--B", type=int, default=1024)
ap.add_argument("--L", type=int, default=1024)
ap.add_argument("--layers", type=int, default=1)
ap.add_argument("--fmt", default="half")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tune", action="append", default=[], help="name=value (sd_tune switch)")
a = ap.parse_args()
for t in a.tune:
    k, v = t.split("=")
    sd.tune(k, int(v))
import torch
spec = sd.make_model_spec(a.layers, a.D, a.H, 64, 64, a.Hkv)
hkv = spec.num_kv_heads
kv = sd.KvShard(spec, 0, hkv, a.B * (a.L + 1), a.fmt, max_sequences=a.B, max_seq_len=a.L + 16)
seqs = list(range(1, a.B + 1))
kv.prefill_synthetic(seqs, a.L)
q = torch.randn(a.B, a.D, device="cuda")
o = torch.empty_like(q)
torch.cuda.synchronize()
for _ in range(3):
    kv.attend_dev(0, seqs, q.data_ptr(), o.data_ptr())
torch.cuda.synchronize()
kv.timing(True)
for l in range(a.reps):
    kv.attend_dev(l % a.layers, seqs, q.data_ptr(), o.data_ptr())
ms, n, byt = kv.timing_read()
torch.cuda.synchronize()
gbs = byt / (ms / 1e3) / 1e9
print(json.dumps({"tune": a.tune, "D": a.D, "H": a.H, "Hkv": hkv, "B": a.B, "L": a.L, "fmt": a.fmt,
                  "ms_per_launch": ms / n, "GBps": gbs, "frac_of_6524": gbs / 6524}))
