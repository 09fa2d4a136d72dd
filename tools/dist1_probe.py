"""One-rank DistEngine over the peer-exchange path (world 1: every route
points at this rank), for profiling the routed producers under ncu, which
cannot follow a multi-rank job:

  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm \
      --csv python tools/dist1_probe.py
  PROBE_NO_FUSE=1 ... (the same kernels without the routed epilogue)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2403_11421_b200 as sd  # noqa: E402


def main():
    B = int(os.environ.get("PROBE_B", "512"))
    if os.environ.get("PROBE_NO_FUSE"):
        sd.tune("dist_fuse", 0)
    ctx = int(os.environ.get("PROBE_CTX", "64"))
    spec = sd.make_model_spec(32, 4096, 32, 14336, 128256, 8)
    w = sd.DeviceWeights(spec, None, "bf16", 0, seed=0)
    seqs = list(range(1, B + 1))
    kv = sd.KvShard(spec, 0, 8, B * (ctx + 16), "half", 0, max_sequences=B, max_seq_len=ctx + 16)
    kv.prefill_synthetic(seqs, ctx, salt=0)
    eng = sd.DistEngine(w, kv, 0, 1, None, 1)
    eng.p2p_connect([eng.p2p_handles(B)])
    tok = np.array([sd.prompt_token(0, s, spec.vocab_size) for s in seqs], np.int32)
    ms = eng.bench(seqs, tok, 3)
    print(f"world-1 dist step: {ms / 3:.3f} ms")
    eng.close()
    kv.close()
    w.close()


if __name__ == "__main__":
    main()
