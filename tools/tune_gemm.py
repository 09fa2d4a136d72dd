"""Sweep the tcgen05 GEMM variants (gemm_kernel tiles and the swapped-operand
kernel's NC / swizzle / cluster) at the decode S-Part shapes. Every config is
checked against torch (bf16 operands, fp32 accumulate) before it is timed
with CUDA events; prints one JSON line per shape with the ranking."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd

M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
SHAPES = {"qkv": (6144, 4096), "w_o": (4096, 4096), "mlp_in": (14336, 4096), "mlp_out": (4096, 14336),
          "head": (128256, 4096)}
CONFIGS = [("single_auto", {"SD_GEMM_PAIR": "0"}), ("pair_auto", {})]
for bn in (256, 224, 208, 192, 176, 160, 128, 112):
    CONFIGS.append((f"pair_bn{bn}", {"SD_GEMM_PAIR": "1", "SD_GEMM_BN": str(bn)}))
KEYS = ("SD_GEMM_PAIR", "SD_GEMM_BN", "SD_GEMM_CS", "SD_GEMM_SWAB", "SD_GEMM_NC", "SD_GEMM_SWB")
dev = torch.device("cuda")
for name, (N, K) in SHAPES.items():
    if only and name not in only:
        continue
    A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
    B = ((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev)
    ref = A.float() @ B.float().T
    res = {}
    for cname, env in CONFIGS:
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        C.fill_(float("nan"))
        try:
            sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            res[cname] = {"error": str(e)[:120]}
            continue
        err = ((C - ref).abs().max() / ref.abs().max()).item()
        if not err < 1e-2:
            res[cname] = {"bad": err}
            continue
        for _ in range(3):
            sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        torch.cuda._sleep(20_000_000)  # GPU busy while the host enqueues: times the kernels, not the launches
        e0.record()
        for _ in range(reps):
            sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        res[cname] = {"us": round(us, 1), "tflops": round(2 * M * N * K / us / 1e6, 1)}
    for k in KEYS:
        os.environ.pop(k, None)
    timed = sorted((v["us"], k) for k, v in res.items() if "us" in v)
    print(json.dumps({"M": M, "shape": name, "N": N, "K": K, "best": timed[:3], "all": res}), flush=True)
