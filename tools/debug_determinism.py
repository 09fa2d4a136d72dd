import os, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [root, os.path.join(root, "oracle"), os.path.join(root, "tests")]
import oracle as o
import paper_2403_11421_b200 as sd
from conftest import upload_oracle_weights
W = o.Weights(o.make_spec(2, 64, 4, 256, 128), 0)
dw = upload_oracle_weights(W, "bf16")
rng = np.random.default_rng(0)
for B in (4, 8, 130):
    x = rng.uniform(-1, 1, (B, 64)).astype(np.float32)
    outs = [sd.project_qkv(dw, 0, x)[0] for _ in range(20)]
    print("qkv B", B, "max dev across 20 runs", max(float(np.abs(a - outs[0]).max()) for a in outs))
    h = rng.uniform(-1, 1, (B, 256)).astype(np.float32)
    outs = [sd.apply_linear(dw, 0, 6, h) for _ in range(20)]
    print("w_out B", B, "max dev", max(float(np.abs(a - outs[0]).max()) for a in outs))
    outs = [sd.apply_linear(dw, 0, 7, x) for _ in range(20)]
    print("head B", B, "max dev", max(float(np.abs(a - outs[0]).max()) for a in outs))
# engine: identical runs
for mode in ("exact", "bf16"):
    res = []
    for rep in range(4):
        d = upload_oracle_weights(W, mode)
        kv = sd.KvShard(d.spec, 0, 4, 1 << 16)
        eng = sd.Engine(d, kv)
        recs, acts, _ = sd.run_generation(eng, 8, 16, 4, 48, seed=0, record_activations=True)
        res.append((recs, acts))
    print(mode, "engine runs identical:", [r[0] == res[0][0] for r in res], [float(np.abs(r[1] - res[0][1]).max()) for r in res])
