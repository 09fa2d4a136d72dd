"""BASELINE config 5 context sweep: Llama-3-8B GQA shape, batch 512, context
512..8192, one B200, fp16 KV, bf16 S-Part.

Full-depth KV at long contexts exceeds one GPU (32 layers x 512 seqs x 8192
positions x 4 KB = 550 GB), so each context is timed on the real engine at
two reduced depths L1 < L2 that fit, and the step time is fitted as
t(L) = a*L + b (a = per-layer cost, b = embedding + head + argmax) and
extrapolated to L = 32 ("report tokens/s for N_eff and
extrapolate"). Contexts whose full 32 layers fit are also measured directly.
Prints one JSON line per context; device-timed with CUDA events."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd

D, H, HKV, F, V, B, NL = 4096, 32, 8, 14336, 128256, 512, 32
STEPS, WARM = 5, 3
KV_BUDGET = 150e9  # bytes of KV per run (180 GB HBM minus weights and activations)


def step_ms(layers: int, ctx: int) -> float:
    spec = sd.make_model_spec(layers, D, H, F, V, HKV)
    total = STEPS + WARM + 4
    w = sd.DeviceWeights(spec, None, "bf16", 0, seed=0)
    kv = sd.KvShard(spec, 0, HKV, B * (ctx + total), "half", 0, max_sequences=B, max_seq_len=ctx + total + 16)
    eng = sd.Engine(w, kv)
    seqs = list(range(1, B + 1))
    kv.prefill_synthetic(seqs, ctx, salt=0)
    tok = np.array([sd.prompt_token(0, s, V) for s in seqs], dtype=np.int32)
    _, tok = eng.bench(seqs, tok, WARM)
    torch.cuda.synchronize()
    ms, _ = eng.bench(seqs, tok, STEPS)
    eng.close()
    kv.close()
    w.close()
    torch.cuda.synchronize()
    return ms / STEPS


def main():
    ctxs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [512, 1024, 2048, 4096, 8192]
    for ctx in ctxs:
        per_layer_kv = B * ctx * 2 * HKV * 128 * 2
        fit_max = int(KV_BUDGET // per_layer_kv)
        row = {"context": ctx, "batch": B, "kv_bytes_full_depth": per_layer_kv * NL}
        if fit_max >= NL:
            t = step_ms(NL, ctx)
            row.update({"method": "measured at 32 layers", "ms_per_step": t, "tokens_per_s": B / t * 1e3})
        else:
            l2 = min(fit_max, 16)
            l1 = max(1, l2 // 2)
            t1, t2 = step_ms(l1, ctx), step_ms(l2, ctx)
            a = (t2 - t1) / (l2 - l1)
            b = t1 - a * l1
            t = a * NL + b
            row.update({"method": f"fit t(L)=a*L+b at L={l1},{l2}, extrapolated to 32",
                        "ms_per_layer": a, "ms_fixed": b, "ms_per_step": t, "tokens_per_s": B / t * 1e3,
                        "measured": {str(l1): t1, str(l2): t2}})
        # attention floor: all KV bytes of the step at the measured copy peak
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json"))).get("hbm_gbs", 6524.0)
        row["kv_read_floor_ms"] = per_layer_kv * NL / (peak * 1e9) * 1e3
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
