import os, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [root, os.path.join(root, "oracle"), os.path.join(root, "tests")]
import oracle as o
import paper_2403_11421_b200 as sd
from conftest import upload_oracle_weights
W = o.Weights(o.make_spec(2, 64, 4, 256, 128), 0)
mode = sys.argv[1] if len(sys.argv) > 1 else "bf16"
runs = []
for rep in range(6):
    d = upload_oracle_weights(W, mode)
    kv = sd.KvShard(d.spec, 0, 4, 1 << 16)
    eng = sd.Engine(d, kv)
    seqs = list(range(1, 9))
    toks = [o.prompt_token(0, q, 128) for q in seqs]
    hist = []
    for step in range(12):
        nt, fx = eng.compute(seqs, tokens=toks, want_final=True)
        hist.append((list(nt), fx.copy()))
        toks = [int(t) for t in nt]
    runs.append(hist)
for rep in range(1, 6):
    for step in range(12):
        a, b = runs[0][step], runs[rep][step]
        if a[0] != b[0] or not np.array_equal(a[1], b[1]):
            rows = np.where(np.abs(a[1] - b[1]).max(axis=1) > 0)[0]
            print("rep", rep, "first diff step", step, "rows", rows.tolist(), "tok", a[0], b[0], "maxdiff", float(np.abs(a[1]-b[1]).max()))
            break
    else:
        print("rep", rep, "identical")
