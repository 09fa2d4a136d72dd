"""MMA-rate probe: times GEMM configs with SD_GEMM_DIAG=0 (normal) and 1
(operands stay resident in smem after the first ring fill, so the time is the
tensor pipe + epilogue alone). Results are not checked in diag mode."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd

M = 512
SHAPES = {"qkv": (6144, 4096), "w_o": (4096, 4096), "mlp_in": (14336, 4096), "mlp_out": (4096, 14336), "head": (128256, 4096)}
CONFIGS = {"single": {"SD_GEMM_PAIR": "0"}, "pair": {}}
dev = torch.device("cuda")
for name, (N, K) in SHAPES.items():
    A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
    B = ((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev)
    out = {}
    for cname, env in CONFIGS.items():
        for diag in ("0", "1", "2"):
            for k in ("SD_GEMM_PAIR", "SD_GEMM_BN", "SD_GEMM_CS"):
                os.environ.pop(k, None)
            os.environ.update(env)
            os.environ["SD_GEMM_DIAG"] = diag
            for _ in range(3):
                sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            out[f"{cname}_d{diag}"] = (round(us, 1), round(2 * M * N * K / us / 1e6))
    os.environ.pop("SD_GEMM_DIAG", None)
    print(json.dumps({"shape": name, **out}), flush=True)
