"""S-Part across GPUs (paper §5.3): tensor parallelism vs
the data-parallel S-ranks this repo uses, measured on B200s.

Per layer and per GPU at a global batch of B = 512 x N rows (C5 shape, fp16
operands, tcgen05 GEMMs of this repo):
  DP: every GPU runs the four layer GEMMs on its B / N = 512 rows, full width;
      no S-Part collective.
  TP (Megatron split): every GPU runs the GEMMs on all B rows with the QKV and
      MLP-in outputs column-split (N / TP) and the W_o and MLP-out inputs
      row-split (K / TP), plus two all-reduces of the B x D fp32 activations
      per layer (after W_o and after MLP-out).
Launch under torchrun with N ranks (N = 2 or 4); rank 0 prints one JSON line.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11421_b200 as sd  # noqa: E402

D, HKV, HD, F = 4096, 8, 128, 14336
QKV = D + 2 * HKV * HD


def gemm_ms(M, N, K, reps=20):
    """Mean ms of one fp16 tcgen05 GEMM C[M][N] = A[M][K] B[N][K]^T, weights
    rotated through buffers larger than L2 (streamed from HBM as in the step)."""
    nbuf = max(2, int(256e6 // (N * K * 2)) + 1)
    A = (torch.rand(M, K, device="cuda") * 2 - 1).half()
    Bs = [((torch.rand(N, K, device="cuda") * 2 - 1) / K**0.5).half() for _ in range(nbuf)]
    C = torch.empty(M, N, device="cuda")
    for i in range(3):
        sd.gemm_dev("fp16", M, N, K, A.data_ptr(), K, Bs[i % nbuf].data_ptr(), K, C.data_ptr(), N)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(reps):
        sd.gemm_dev("fp16", M, N, K, A.data_ptr(), K, Bs[i % nbuf].data_ptr(), K, C.data_ptr(), N)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    B = 512 * world
    dp = {"qkv": gemm_ms(512, QKV, D), "w_o": gemm_ms(512, D, D), "mlp_in": gemm_ms(512, F, D),
          "mlp_out": gemm_ms(512, D, F)}
    tp = {"qkv": gemm_ms(B, QKV // world, D), "w_o": gemm_ms(B, D, D // world), "mlp_in": gemm_ms(B, F // world, D),
          "mlp_out": gemm_ms(B, D, F // world)}
    x = torch.rand(B, D, device="cuda")
    for _ in range(5):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dist.all_reduce(x)
    e1.record()
    torch.cuda.synchronize()
    ar = e0.elapsed_time(e1) / 20
    t = torch.tensor([sum(dp.values()), sum(tp.values()) + 2 * ar], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"world": world, "global_batch": B, "shape": "C5 (D 4096, F 14336, 8 kv heads), fp16",
                          "dp_ms_per_layer": t[0].item(), "tp_ms_per_layer": t[1].item(),
                          "dp_gemm_ms": dp, "tp_gemm_ms": tp, "allreduce_fp32_BxD_ms": ar,
                          "tp_over_dp": t[1].item() / t[0].item()}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
