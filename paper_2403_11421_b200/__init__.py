"""B200-native FastDecode decode hot path (arXiv 2403.11421).

R-Part: paged HBM KV store + split-K flash-decode attention (sm_100a CUDA).
S-Part: QKV / O / MLP / head GEMMs on tcgen05 tensor cores (or the exact
fp32 CUDA-core path). Host: the reference's KvShard / StepComputation /
drive_schedule / ShardMap interfaces over the C-ABI in include/sd_abi.h.
"""
from .api import (AdmissionError, AttentionItem, AttentionRequest, CapacityError, ConfigError,
                  CudaError, InfeasiblePlanError, DeviceWeights, DistEngine, Engine, dist_plan, nccl_unique_id, KvShard, LogicError, ProtocolError, ShardMap,
                  SplitDecodeError, UnknownSequenceError, apply_linear, cold_start_schedule,
                  finish_block, gemm_dev, launch_count, make_model_spec, micro_batch_size, mix64, output_logits_argmax,
                  project_qkv, prompt_token, run_generation, transcript_csv, tune, tuned, RWorker,
                  serve_rworker)
from ._lib import LIB_PATH, ModelSpec, lib

__all__ = [n for n in dir() if not n.startswith("_")]
from . import planner  # noqa: E402
