"""Fixed per-call cost of the tcgen05 GEMM at K = 512 (4 k-stages): normal,
store-free epilogue (SD_GEMM_DIAG=4), and an empty-ish launch for scale."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd
M, dev = 512, torch.device("cuda")
for N, K in ((6144, 512), (6144, 128), (4096, 128)):
    A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
    B = ((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev)
    out = {}
    for diag in ("0", "4"):
        os.environ["SD_GEMM_DIAG"] = diag
        for _ in range(3):
            sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        e0.record()
        for _ in range(50):
            sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N)
        e1.record()
        torch.cuda.synchronize()
        out["diag" + diag] = round(e0.elapsed_time(e1) / 50 * 1e3, 2)
    x = torch.empty(1, device=dev)
    torch.cuda._sleep(20_000_000)
    e0.record()
    for _ in range(50):
        x.add_(1)
    e1.record()
    torch.cuda.synchronize()
    out["tiny_torch_kernel"] = round(e0.elapsed_time(e1) / 50 * 1e3, 2)
    print(json.dumps({"N": N, "K": K, **out}), flush=True)
