import os, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [root, os.path.join(root, "oracle"), os.path.join(root, "tests")]
import oracle as o
import paper_2403_11421_b200 as sd
from conftest import upload_oracle_weights
W = o.Weights(o.make_spec(2, 64, 4, 256, 128), 0)
mode = sys.argv[1]
variant = sys.argv[2]

def run():
    d = upload_oracle_weights(W, mode)
    kv = sd.KvShard(d.spec, 0, 4, 1 << 16)
    eng = sd.Engine(d, kv)
    okv = o.KvShard(W.spec, 0, 4, 1 << 16)
    emb = W.tensor("embedding")
    toks = {}
    out = []
    live = []
    nxt = 1
    for step in range(24):
        if variant == "grow" and step % 3 == 0 and len(live) < 8:
            for _ in range(2):
                live.append(nxt); toks[nxt] = o.prompt_token(0, nxt, 128); nxt += 1
        if variant == "retire":
            if step % 3 == 0:
                for _ in range(2):
                    live.append(nxt); toks[nxt] = o.prompt_token(0, nxt, 128); nxt += 1
            if len(live) > 6:
                gone = live[:2]; live = live[2:]
                eng.retire(gone)
                for q in gone: okv.drop_sequence(q)
        seqs = list(live)
        t = [toks[q] for q in seqs]
        nt, fx = eng.compute(seqs, tokens=t, want_final=True)
        x = np.stack([emb[:, tk] for tk in t]).astype(np.float32)
        ont, ofx, _ = o.decode_step_monolithic(W, okv, seqs, x)
        out.append((step, list(nt), list(ont), float(np.abs(fx - ofx).max())))
        for i, q in enumerate(seqs): toks[q] = int(ont[i])  # follow the oracle's tokens
    return out

for rep in range(4):
    out = run()
    bad = [(s, a, b, e) for s, a, b, e in out if e > 1e-3 or (mode == "exact" and a != b)]
    print(mode, variant, "rep", rep, "worst", max(e for *_, e in out), "first bad", bad[:1])
