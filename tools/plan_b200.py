"""Measure a B200 perf profile (the reference planner's inputs) and plan.

T(B): one block's S-Part at each batch (sd_bench_dense_block, bf16 tcgen05).
R: attend seconds per token-position per layer (sd_bench_attention_per_token,
fp16 KV, all kv heads). C: KV tokens of the full model that fit the free HBM
after weights. Writes the profile in the reference's JSON format and the
planner's operating points (Eq. 7-11) for the requested lengths.

  python tools/plan_b200.py [7b|13b|8b] [out.json] [fp16|bf16|tf32]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd
from paper_2403_11421_b200 import planner as pl

SHAPES = {  # (layers, D, heads, F, V, kv_heads) - BASELINE geometries
    "7b": (32, 4096, 32, 11008, 32000, 32),
    "13b": (40, 5120, 40, 13824, 32000, 40),
    "8b": (32, 4096, 32, 14336, 128256, 8),
}
name = sys.argv[1] if len(sys.argv) > 1 else "7b"
mode = sys.argv[3] if len(sys.argv) > 3 else "fp16"
out = sys.argv[2] if len(sys.argv) > 2 else f"profiles/r02_perf_profile_b200_{name}_{mode}.json"
L, D, H, F, V, Hkv = SHAPES[name]
one = sd.make_model_spec(1, D, H, F, V, Hkv)
w = sd.DeviceWeights(one, None, mode, 0, seed=7)
table = pl.bench_dense_block(w, [1, 8, 64, 256, 512, 1024, 2048, 4096], reps=5)
w.close()
r = pl.bench_attention_per_token(one, "half", batch=256, seq_len=1024, reps=5)
full = sd.make_model_spec(L, D, H, F, V, Hkv)
weights_bytes = 2.0 * (L * (D * (H + 2 * Hkv) * (D // H) + D * D + 2 * D * F) + 2 * D * V)
cap = pl.kv_capacity_tokens(full, "half", reserve_bytes=weights_bytes + 8e9)
prof = pl.PerfProfile(table, r, cap, f"B200/sm_100a/{name}/{mode}-S/fp16-KV")
plans = {}
for S in (1024, 2048, 4096):
    for budget in (None,):
        p = pl.plan(prof, pl.PlanRequest(num_layers=L, target_len=S))
        plans[f"S={S}"] = p.__dict__
doc = {"profile": prof.to_json(), "plans_knee": plans,
       "note": "R-workers per S-worker (worker_count) from B*S*R/(2*T(B)) with B200-measured T(B), R"}
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc))
