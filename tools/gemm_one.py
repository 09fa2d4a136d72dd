"""One GEMM shape, ours then cuBLAS (torch.matmul), for ncu captures."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd
M, N, K = (int(x) for x in sys.argv[1:4])
dev = torch.device("cuda")
A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
B = ((torch.rand(N, K, device=dev) * 2 - 1) / K**0.5).to(torch.bfloat16)
C = torch.empty(M, N, device=dev)
Cb = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    sd.gemm_dev("bf16", M, N, K, A.data_ptr(), K, B.data_ptr(), K, None, 0, Cb.data_ptr(), N)
    torch.matmul(A, B.T)
torch.cuda.synchronize()
print("ok")
