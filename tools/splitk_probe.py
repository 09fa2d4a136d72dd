"""Is the S-Part GEMM bound by per-SM operand ingress? Times the N=4096
decode GEMMs (W_o, MLP-out) at M=512 as launched today, and the main loop a
split-K=2 version would run (each CTA pair: bn=256 over half of K, emulated
as one GEMM with N doubled and K halved). Weights rotate through buffers
larger than L2, as in the model, so every launch streams them from HBM."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd  # noqa: E402

M = 512
dev = torch.device("cuda")


def timed(N, K, env):
    for k in ("SD_GEMM_PAIR", "SD_GEMM_BN"):
        os.environ.pop(k, None)
    os.environ.update(env)
    nbuf = max(2, int(192e6 // (N * K * 2)) + 1)
    A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
    Bs = [((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(torch.bfloat16) for _ in range(nbuf)]
    C = torch.empty(M, N, device=dev)
    for i in range(3):
        sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, Bs[i % nbuf].data_ptr(), K, C.data_ptr(), N)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    reps = 40
    for i in range(reps):
        sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, Bs[i % nbuf].data_ptr(), K, C.data_ptr(), N)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 2)


for name, N, K in (("w_o", 4096, 4096), ("mlp_out", 4096, 14336), ("qkv", 6144, 4096), ("mlp_in", 14336, 4096)):
    out = {"shape": name, "auto_us": timed(N, K, {})}
    for bn in (256, 224, 192):
        out[f"split2_bn{bn}_mainloop_us"] = timed(2 * N, K // 2, {"SD_GEMM_PAIR": "1", "SD_GEMM_BN": str(bn)})
    out["bn256_unsplit_us"] = timed(N, K, {"SD_GEMM_PAIR": "1", "SD_GEMM_BN": "256"})
    print(json.dumps(out), flush=True)
