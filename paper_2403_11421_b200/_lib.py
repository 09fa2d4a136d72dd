"""Loads libsd_b200.so (the C-ABI of include/sd_abi.h) and declares its
signatures. There is no fallback: if the CUDA library is missing or cannot
be loaded the import fails loudly."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsd_b200.so")


class LibraryMissing(ImportError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2403_11421_b200/csrc). There is no CPU fallback.")
    return C.CDLL(LIB_PATH)


lib = _load()


class ModelSpec(C.Structure):
    """ModelSpec (core.hpp:43-50) + num_kv_heads (GQA extension)."""
    _fields_ = [(n, C.c_int32) for n in ("num_layers", "model_dim", "num_heads", "head_dim",
                                          "mlp_dim", "vocab_size", "num_kv_heads")]

    def __repr__(self):
        return ("ModelSpec(" + ", ".join(f"{n}={getattr(self, n)}" for n, _ in self._fields_) + ")")


class KvOptions(C.Structure):
    _fields_ = [("max_sequences", C.c_int32), ("max_seq_len", C.c_int32),
                ("page_positions", C.c_int32), ("pool_pages", C.c_int32)]


class DriveConfig(C.Structure):
    _fields_ = [("batch", C.c_int32), ("target_len", C.c_int32), ("interval", C.c_int32),
                ("cold_start", C.c_int32), ("steps", C.c_int64), ("load_limit", C.c_int64),
                ("seed", C.c_uint64), ("record_activations", C.c_int32)]


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
FP = C.POINTER(C.c_float)
U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
DP = C.POINTER(C.c_double)
SPEC_P = C.POINTER(ModelSpec)

class PerfProfileC(C.Structure):
    _fields_ = [("batch", C.POINTER(C.c_int32)), ("seconds", C.POINTER(C.c_double)), ("n", C.c_int32),
                ("r_per_token", C.c_double), ("capacity_c", C.c_int64)]


class PlanRequestC(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("target_len", C.c_int32), ("has_latency_budget", C.c_int32),
                ("latency_budget", C.c_double),
                ("candidates", C.POINTER(C.c_int32)), ("n_candidates", C.c_int32),
                ("knee_threshold", C.c_double), ("balance_tolerance", C.c_double)]


class HardwarePlanC(C.Structure):
    _fields_ = [("batch_size", C.c_int32), ("worker_count", C.c_int32), ("worker_estimate", C.c_double),
                ("predicted_seq_seconds", C.c_double), ("efficiency", C.c_double),
                ("balance_residual", C.c_double), ("balanced", C.c_int32), ("binding_constraint", C.c_int32),
                ("tightest_batch", C.c_int32)]


SIGNATURES = {
    "sd_last_error": (C.c_char_p, []),
    "sd_abi_version": (C.c_int, []),
    "sd_make_model_spec": (C.c_int, [C.c_int] * 6 + [SPEC_P]),
    "sd_mix64": (C.c_uint64, [C.c_uint64]),
    "sd_prompt_token": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int]),
    "sd_kv_create": (C.c_int, [SPEC_P, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int,
                               C.POINTER(KvOptions), PP]),
    "sd_kv_destroy": (C.c_int, [P]),
    "sd_kv_append": (C.c_int, [P, C.c_uint64, C.c_int, C.c_uint32, FP, FP]),
    "sd_kv_append_request": (C.c_int, [P, C.c_int, C.c_int32, U64P, U32P, FP, FP]),
    "sd_kv_attend": (C.c_int, [P, C.c_int, C.c_int32, U64P, FP, FP]),
    "sd_kv_append_attend": (C.c_int, [P, C.c_int, C.c_int32, U64P, U32P, FP, FP, FP, FP]),
    "sd_kv_append_request_dev": (C.c_int, [P, C.c_int, C.c_int32, U64P, U32P, P, P, P]),
    "sd_kv_attend_dev": (C.c_int, [P, C.c_int, C.c_int32, U64P, P, P, P]),
    "sd_kv_append_attend_dev": (C.c_int, [P, C.c_int, C.c_int32, U64P, U32P, P, P, P, P, P]),
    "sd_kv_drop": (C.c_int, [P, C.c_int32, U64P]),
    "sd_kv_stored_length": (C.c_int, [P, C.c_uint64, C.c_int, I32P]),
    "sd_kv_has_sequence": (C.c_int, [P, C.c_uint64, I32P]),
    "sd_kv_token_count": (C.c_int, [P, I64P]),
    "sd_kv_warning_count": (C.c_int, [P, I32P]),
    "sd_kv_bytes_per_token": (C.c_int, [P, I64P]),
    "sd_kv_width": (C.c_int, [P, I32P, I32P]),
    "sd_kv_export_lane": (C.c_int64, [P, C.c_uint64, C.c_int, C.c_int, P, C.c_size_t, FP,
                                      C.c_size_t]),
    "sd_kv_prefill_synthetic": (C.c_int, [P, C.c_int32, U64P, C.c_int32, C.c_uint64]),
    "sd_kv_timing": (C.c_int, [P, C.c_int]),
    "sd_kv_timing_read": (C.c_int, [P, DP, I64P, DP, C.c_int]),
    "sd_weights_upload": (C.c_int, [SPEC_P, C.POINTER(FP), C.c_int, C.c_int, PP]),
    "sd_weights_destroy": (C.c_int, [P]),
    "sd_s_project_qkv": (C.c_int, [P, C.c_int, C.c_int32, FP, FP, FP, FP]),
    "sd_s_finish_block": (C.c_int, [P, C.c_int, C.c_int32, FP, FP, FP]),
    "sd_s_logits_argmax": (C.c_int, [P, C.c_int32, FP, FP, I32P]),
    "sd_s_apply_linear": (C.c_int, [P, C.c_int, C.c_int, C.c_int32, FP, FP]),
    "sd_gemm_dev": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int64, P, C.c_int64, P,
                              C.c_int64, P, C.c_int64, C.c_int, P, C.c_int64, P]),
    "sd_engine_create": (C.c_int, [P, P, PP]),
    "sd_engine_destroy": (C.c_int, [P]),
    "sd_engine_step": (C.c_int, [P, C.c_int32, U64P, I32P, I32P, FP]),
    "sd_engine_step_features": (C.c_int, [P, C.c_int32, U64P, FP, I32P, FP, FP]),
    "sd_engine_retire": (C.c_int, [P, C.c_int32, U64P]),
    "sd_engine_bench": (C.c_int, [P, C.c_int32, U64P, I32P, C.c_int32, I32P, DP]),
    "sd_engine_timing": (C.c_int, [P, C.c_int]),
    "sd_engine_timing_read": (C.c_int, [P, DP, DP, I64P, C.c_int]),
    "sd_launch_count": (C.c_int64, []),
    "sd_engine_pipeline": (C.c_int, [P, C.c_int, C.c_int]),
    "sd_weights_synthetic": (C.c_int, [SPEC_P, C.c_int, C.c_uint64, C.c_int, PP]),
    "sd_weights_seed_random": (C.c_int, [SPEC_P, C.c_uint64, C.c_int, C.c_int, PP]),
    "sd_tune": (C.c_int, [C.c_char_p, C.c_int]),
    "sd_dist_pipeline": (C.c_int, [C.c_void_p, C.c_int]),
    "sd_rworker_create": (C.c_int, [C.c_int64, C.c_int, C.c_int, PP]),
    "sd_rworker_destroy": (C.c_int, [C.c_void_p]),
    "sd_rworker_feed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "sd_rworker_shutdown_requested": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "sd_rworker_serve": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double]),
    "sd_weights_export_embedding": (C.c_int, [C.c_void_p, FP, C.c_size_t]),
    "sd_drive": (C.c_int, [P, C.POINTER(DriveConfig), PP]),
    "sd_drive_count": (C.c_int64, [P]),
    "sd_drive_record": (C.c_int, [P, C.c_int64, I64P, U64P, I32P]),
    "sd_drive_activations": (FP, [P]),
    "sd_drive_wall_seconds": (C.c_double, [P]),
    "sd_drive_destroy": (C.c_int, [P]),
    "sd_nccl_unique_id": (C.c_int, [P, C.c_size_t]),
    "sd_dist_create": (C.c_int, [P, P, C.c_int, C.c_int, P, C.c_int, C.c_int, PP]),
    "sd_dist_destroy": (C.c_int, [P]),
    "sd_dist_step": (C.c_int, [P, C.c_int32, U64P, I32P, I32P, FP]),
    "sd_dist_retire": (C.c_int, [P, C.c_int32, U64P]),
    "sd_dist_bench": (C.c_int, [P, C.c_int32, U64P, I32P, C.c_int32, DP]),
    "sd_dist_drive": (C.c_int, [P, C.POINTER(DriveConfig), PP]),
    "sd_dist_timing": (C.c_int, [P, C.c_int]),
    "sd_dist_timing_read": (C.c_int, [P, DP, DP, C.c_int]),
    "sd_dist_p2p_setup": (C.c_int, [P, C.c_int32, P]),
    "sd_bench_dense_block": (C.c_int, [P, I32P, C.c_int32, C.c_int32, DP]),
    "sd_bench_attention_per_token": (C.c_int, [SPEC_P, C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int, DP]),
    "sd_kv_capacity_tokens": (C.c_int, [SPEC_P, C.c_int, C.c_int, C.c_double, I64P]),
    "sd_plan": (C.c_int, [C.POINTER(PerfProfileC), C.POINTER(PlanRequestC), C.POINTER(HardwarePlanC)]),
    "sd_plan_batch_size": (C.c_int, [C.POINTER(PerfProfileC), C.POINTER(PlanRequestC), I32P, I32P]),
    "sd_plan_block_seconds": (C.c_int, [C.POINTER(PerfProfileC), C.c_int32, DP]),
    "sd_plan_worker_count": (C.c_int, [C.POINTER(PerfProfileC), C.c_int32, C.c_int32, I32P, DP]),
    "sd_plan_check_memory": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, I32P, I32P]),
    "sd_plan_check_balance": (C.c_int, [C.POINTER(PerfProfileC), C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                        DP, DP, I32P]),
    "sd_dist_p2p_connect": (C.c_int, [P, P]),
    "sd_dist_plan": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int32, U64P, I32P, I32P, I32P, I32P,
                               I32P, I32P]),
    "sd_shardmap_worker_for": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, I32P]),
    "sd_shardmap_head_range": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, I32P, I32P]),
    "sd_micro_batch_size": (C.c_int, [C.c_int, C.c_int, C.c_int, I32P]),
    "sd_cold_start_schedule": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, I64P,
                                         C.c_int64, I64P]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)  # AttributeError = the .so lacks an ABI symbol: fail loudly
    _f.restype = _res
    _f.argtypes = _args
