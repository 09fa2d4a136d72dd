"""tcgen05 GEMM microbenchmark at the decode S-Part shapes (CUDA events,
inputs resident). Checks each result against torch (bf16 operands, fp32
accumulate) before timing. argv: [M] [kind bf16|fp16|tf32] [forced pair-tile width]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd

M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
KIND = sys.argv[2] if len(sys.argv) > 2 else "bf16"
BN = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sd.tune("gemm_bn", BN)
DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "tf32": torch.float32}[KIND]
SHAPES = {"qkv": (6144, 4096), "w_o": (4096, 4096), "mlp_in": (14336, 4096), "mlp_out": (4096, 14336),
          "head": (128256, 4096), "7b_qkv": (12288, 4096), "7b_mlp_in": (11008, 4096), "7b_mlp_out": (4096, 11008)}
dev = torch.device("cuda")
out = {}
for name, (N, K) in SHAPES.items():
    A = (torch.rand(M, K, device=dev) * 2 - 1).to(DT)
    B = ((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(DT)
    C = torch.empty(M, N, device=dev)
    sd.gemm_dev(KIND, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    for _ in range(3):
        sd.gemm_dev(KIND, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        sd.gemm_dev(KIND, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    # cuBLAS (torch.matmul, bf16 out) on the same operands, for reference only
    for _ in range(3):
        torch.matmul(A, B.T)
    e0.record()
    for _ in range(reps):
        torch.matmul(A, B.T)
    e1.record()
    torch.cuda.synchronize()
    us_cublas = e0.elapsed_time(e1) / reps * 1e3
    out[name] = {"us": round(us, 1), "tflops": round(2 * M * N * K / us / 1e6, 1), "rel_err": err,
                 "cublas_us": round(us_cublas, 1)}
print(json.dumps({"M": M, "kind": KIND, "bn": BN or "auto", "shapes": out}))
