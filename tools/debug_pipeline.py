import os, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [root, os.path.join(root, "oracle"), os.path.join(root, "tests")]
import oracle as o
import paper_2403_11421_b200 as sd
from conftest import upload_oracle_weights
W = o.Weights(o.make_spec(2, 64, 4, 256, 128), 0)
res = {}
for pipe in (False, True):
    dw = upload_oracle_weights(W, "exact")
    kv = sd.KvShard(dw.spec, 0, 4, 1 << 16)
    eng = sd.Engine(dw, kv)
    if pipe:
        eng.pipeline(True, 100)
    recs, acts, _ = sd.run_generation(eng, 8, 16, 4, 48, seed=0, record_activations=True)
    res[pipe] = (recs, acts)
orecs, oacts = o.run_monolithic(W, 8, 16, 4, 48, seed=0, record=True)
for pipe in (False, True):
    recs, acts = res[pipe]
    bad = [i for i, (a, b) in enumerate(zip(recs, orecs)) if a != b]
    print("pipe", pipe, "n", len(recs), len(orecs), "first bad", bad[:5], [recs[i] for i in bad[:3]], [orecs[i] for i in bad[:3]])
    d = np.abs(acts - oacts).max(axis=1)
    first = int(np.argmax(d > 1e-5)) if (d > 1e-5).any() else -1
    print("  first act row > 1e-5:", first, recs[first] if first >= 0 else None, float(d.max()))
# bf16: pipelined vs non-pipelined vs oracle
for rep in range(3):
    out = {}
    for pipe in (False, True):
        dw = upload_oracle_weights(W, "bf16")
        kv = sd.KvShard(dw.spec, 0, 4, 1 << 16)
        eng = sd.Engine(dw, kv)
        if pipe:
            eng.pipeline(True, 100)
        out[pipe] = sd.run_generation(eng, 8, 16, 4, 48, seed=0, record_activations=True)
    a, b = out[False], out[True]
    print("bf16 rep", rep, "nonpipe==oracle", a[0] == orecs, "pipe==nonpipe", a[0] == b[0],
          "act diff", float(np.abs(a[1] - b[1]).max()),
          "first diff", next((i for i, (x, y) in enumerate(zip(a[0], b[0])) if x != y), None))
