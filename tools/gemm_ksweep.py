"""Mainloop rate vs fixed cost of the tcgen05 GEMM: time one shape at several
K (same M, N, tiles) with the host enqueue hidden behind a GPU sleep; the
slope over K is the mainloop, the intercept the per-tile fixed cost
(launch, prologue, pipeline fill, epilogue)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd

M = 512
dev = torch.device("cuda")
DIAG = os.environ.get("KSWEEP_DIAG", "0").split(",")
for N in (6144, 4096):
    for epi, diag in [("none", d) for d in DIAG]:
        os.environ["SD_GEMM_DIAG"] = diag
        row = {}
        for K in (512, 1024, 2048, 4096, 8192, 16384):
            A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
            B = ((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(torch.bfloat16)
            C = torch.empty(M, N, device=dev)
            Cb = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
            args = (C.data_ptr(), N, Cb.data_ptr(), N) if epi == "bf16_out" else (C.data_ptr(), N)
            for _ in range(3):
                sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, *args)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(20_000_000)
            e0.record()
            for _ in range(20):
                sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, *args)
            e1.record()
            torch.cuda.synchronize()
            row[K] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
        print(json.dumps({"M": M, "N": N, "epi": epi, "diag": diag, "us_by_K": row}), flush=True)
