"""Capacity planning over B200-measured inputs: the reference planner
(planner.hpp:25-109, planner.cpp:48-222; Eq. 7-11 of the paper) behind the
C ABI, and the GPU measurements that feed it (sd_bench_dense_block for T(B),
sd_bench_attention_per_token for R, sd_kv_capacity_tokens for C).

Profiles read and write the reference's perf-profile JSON
(`{"t_table": [{"batch_size", "seconds_per_block"}], "r_per_token",
"capacity_c", "machine_tag"}`), so `splitdecode plan --profile` can consume a
profile measured here and vice versa."""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

from ._lib import HardwarePlanC, PerfProfileC, PlanRequestC, lib
from .api import InfeasiblePlanError, ModelSpec, _check

BINDINGS = {0: "latency", 1: "efficiency-knee", 2: "memory"}
KV_FORMATS = {"single": 0, "half": 1, "int8": 2}


@dataclass
class PerfProfile:
    t_table: list  # [(batch, seconds per block)], ascending batch
    r_per_token: float
    capacity_c: int
    machine_tag: str = ""

    def to_json(self) -> dict:
        return {"t_table": [{"batch_size": b, "seconds_per_block": t} for b, t in self.t_table],
                "r_per_token": self.r_per_token, "capacity_c": self.capacity_c, "machine_tag": self.machine_tag}

    @staticmethod
    def from_json(j: dict) -> "PerfProfile":
        return PerfProfile([(int(r["batch_size"]), float(r["seconds_per_block"])) for r in j["t_table"]],
                           float(j["r_per_token"]), int(j["capacity_c"]), j.get("machine_tag", ""))

    def _c(self):
        n = len(self.t_table)
        b = (C.c_int32 * max(n, 1))(*[x[0] for x in self.t_table])
        s = (C.c_double * max(n, 1))(*[x[1] for x in self.t_table])
        p = PerfProfileC(C.cast(b, C.POINTER(C.c_int32)), C.cast(s, C.POINTER(C.c_double)), n,
                         float(self.r_per_token), int(self.capacity_c))
        return p, (b, s)


@dataclass
class PlanRequest:
    num_layers: int
    target_len: int
    latency_budget: float | None = None
    candidate_batches: list = field(default_factory=list)
    knee_threshold: float = 0.10
    balance_tolerance: float = 0.15

    def _c(self):
        n = len(self.candidate_batches)
        c = (C.c_int32 * max(n, 1))(*self.candidate_batches)
        has = self.latency_budget is not None
        return PlanRequestC(self.num_layers, self.target_len, int(has), float(self.latency_budget) if has else 0.0,
                            C.cast(c, C.POINTER(C.c_int32)), n, self.knee_threshold, self.balance_tolerance), c


@dataclass
class HardwarePlan:
    batch_size: int
    worker_count: int
    worker_estimate: float
    predicted_seq_seconds: float
    efficiency: float
    balance_residual: float
    balanced: bool
    binding_constraint: str


def _raise_infeasible(rc: int, tightest: int):
    try:
        _check(rc)
    except InfeasiblePlanError as e:
        e.tightest_batch = tightest
        raise


def block_seconds(profile: PerfProfile, batch: int) -> float:
    p, keep = profile._c()
    out = C.c_double()
    _check(lib.sd_plan_block_seconds(C.byref(p), batch, C.byref(out)))
    return out.value


def batch_efficiency(profile: PerfProfile, batch: int) -> float:
    return batch / block_seconds(profile, batch)


def plan_batch_size(profile: PerfProfile, request: PlanRequest) -> int:
    p, keep = profile._c()
    q, keep2 = request._c()
    b, t = C.c_int32(), C.c_int32()
    _raise_infeasible(lib.sd_plan_batch_size(C.byref(p), C.byref(q), C.byref(b), C.byref(t)), t.value)
    return b.value


def plan_worker_count(profile: PerfProfile, batch: int, target_len: int):
    p, keep = profile._c()
    w, e = C.c_int32(), C.c_double()
    _check(lib.sd_plan_worker_count(C.byref(p), batch, target_len, C.byref(w), C.byref(e)))
    return w.value, e.value


def check_memory(batch: int, target_len: int, capacity: int, workers: int):
    f, m = C.c_int32(), C.c_int32()
    _check(lib.sd_plan_check_memory(batch, target_len, capacity, workers, C.byref(f), C.byref(m)))
    return bool(f.value), m.value


def check_balance(profile: PerfProfile, batch: int, target_len: int, workers: int, tolerance: float = 0.15):
    p, keep = profile._c()
    st, res, ok = C.c_double(), C.c_double(), C.c_int32()
    _check(lib.sd_plan_check_balance(C.byref(p), batch, target_len, workers, tolerance, C.byref(st),
                                     C.byref(res), C.byref(ok)))
    return st.value, res.value, bool(ok.value)


def plan(profile: PerfProfile, request: PlanRequest) -> HardwarePlan:
    p, keep = profile._c()
    q, keep2 = request._c()
    h = HardwarePlanC()
    _raise_infeasible(lib.sd_plan(C.byref(p), C.byref(q), C.byref(h)), h.tightest_batch)
    return HardwarePlan(h.batch_size, h.worker_count, h.worker_estimate, h.predicted_seq_seconds, h.efficiency,
                        h.balance_residual, bool(h.balanced), BINDINGS[h.binding_constraint])


# ------------------------------------------------------ GPU measurements
def bench_dense_block(weights, batches, reps: int = 5) -> list:
    """T(B) on the GPU for each batch (ascending): [(batch, seconds per block)]."""
    b = (C.c_int32 * len(batches))(*batches)
    out = (C.c_double * len(batches))()
    _check(lib.sd_bench_dense_block(weights.h, b, len(batches), reps, out))
    return list(zip(batches, list(out)))


def bench_attention_per_token(spec: ModelSpec, kv_format: str = "half", batch: int = 256, seq_len: int = 1024,
                              reps: int = 5, device: int = 0) -> float:
    """R on the GPU: seconds of attend per token-position per layer."""
    out = C.c_double()
    _check(lib.sd_bench_attention_per_token(C.byref(spec), KV_FORMATS[kv_format], batch, seq_len, reps, device,
                                            C.byref(out)))
    return out.value


def kv_capacity_tokens(spec: ModelSpec, kv_format: str = "half", device: int = 0,
                       reserve_bytes: float = 0.0) -> int:
    out = C.c_int64()
    _check(lib.sd_kv_capacity_tokens(C.byref(spec), KV_FORMATS[kv_format], device, reserve_bytes, C.byref(out)))
    return out.value
