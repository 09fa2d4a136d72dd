"""Tile-width sweep of the pair GEMM at M = 512 (weights streamed from HBM):
checks pick_pair_bn's choice per decode shape against forced widths."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd  # noqa: E402

M = 512
dev = torch.device("cuda")


def timed(N, K, bn):
    sd.tune("gemm_bn", bn)  # 0: the wave cost model
    nbuf = max(2, int(192e6 // (N * K * 2)) + 1)
    A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
    Bs = [((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(torch.bfloat16) for _ in range(nbuf)]
    C = torch.empty(M, N, device=dev)
    for i in range(3):
        sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, Bs[i % nbuf].data_ptr(), K, C.data_ptr(), N)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(30):
        sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, Bs[i % nbuf].data_ptr(), K, C.data_ptr(), N)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / 30 * 1e3, 2)


SHAPES = {"qkv": (6144, 4096, (0, 144, 160, 176, 192, 208)), "w_o": (4096, 4096, (0, 96, 112, 128, 144)),
          "mlp_in": (14336, 4096, (0, 176, 192, 208, 224, 240, 256)), "mlp_out": (4096, 14336, (0, 96, 112, 128, 144))}
for name, (N, K, bns) in SHAPES.items():
    print(json.dumps({"shape": name, **{f"bn{b}" if b else "auto": timed(N, K, b) for b in bns}}), flush=True)
