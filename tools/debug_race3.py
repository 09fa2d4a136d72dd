import os, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [root, os.path.join(root, "oracle"), os.path.join(root, "tests")]
import oracle as o
import paper_2403_11421_b200 as sd
from conftest import upload_oracle_weights
W = o.Weights(o.make_spec(2, 64, 4, 256, 128), 0)
emb = W.tensor("embedding")
def mk():
    d = upload_oracle_weights(W, "bf16")
    kv = sd.KvShard(d.spec, 0, 4, 1 << 16)
    return d, kv, sd.Engine(d, kv)
for trial in range(4):
    A, B = mk(), mk()
    live, toks, nxt = [], {}, 1
    found = False
    for step in range(30):
        if step % 3 == 0:
            for _ in range(2):
                live.append(nxt); toks[nxt] = o.prompt_token(0, nxt, 128); nxt += 1
        if len(live) > 6:
            gone = live[:2]; live = live[2:]
            A[2].retire(gone); B[2].retire(gone)
        seqs = list(live); t = [toks[q] for q in seqs]
        na, fa = A[2].compute(seqs, tokens=t, want_final=True)
        nb, fb = B[2].compute(seqs, tokens=t, want_final=True)
        if not np.array_equal(fa, fb):
            rows = np.where(np.abs(fa - fb).max(axis=1) > 0)[0]
            print("trial", trial, "step", step, "B", len(seqs), "rows", rows.tolist(), "seqs", [seqs[r] for r in rows],
                  "pos", [A[1].stored_length(seqs[r], 0) for r in rows], "maxdiff", float(np.abs(fa - fb).max()))
            found = True
            break
        for i, q in enumerate(seqs): toks[q] = int(na[i])
    if not found: print("trial", trial, "identical")
