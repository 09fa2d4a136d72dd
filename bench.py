"""Decode benchmark for the B200 FastDecode hot path (BASELINE.json metric:
decode tokens/sec at 1/2/4/8 B200; R-Part HBM GB/s as % of peak).

One "step" = one full decode step (all layers: QKV GEMM, KV append,
split-K attention over the KV cache, W_o + MLP GEMMs, head + argmax) over the
resident batch, exactly StepComputation::compute (workers.hpp:151-158).

Default workload (N=1): BASELINE config 5, Llama-3-8B GQA shape at batch 512,
context 2048 — the largest BASELINE config whose full 32-layer KV cache fits
one B200 (config 2, Llama-2-7B at B=1024 / ctx 1024, needs 550 GB of fp16 KV;
its R-Part is measured per layer and reported as `r_part_c2`). Synthetic
counter-hash weights and KV prefill; inputs (137 GB of KV) exceed the 126 MB
L2 by 1000x, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (layers, model_dim, heads, kv_heads, mlp_dim, vocab, batch/GPU, context, kv fmt, dense)
    "c5-llama3-8b-gqa-b512-ctx2048": (32, 4096, 32, 8, 14336, 128256, 512, 2048, "half", "bf16"),
    "c5-llama3-8b-gqa-b512-ctx1024": (32, 4096, 32, 8, 14336, 128256, 512, 1024, "half", "bf16"),
    "c1-tiny-b16-ctx128": (2, 256, 2, 2, 1024, 256, 16, 128, "single", "exact"),
}
DEFAULT = "c5-llama3-8b-gqa-b512-ctx2048"
TIMING_EVERY = 8  # bench.py samples per-kernel CUDA events on every 8th layer
METRIC = "decode tokens/sec at 1/2/4/8 B200; R-Part HBM GB/s as % of peak"


def peaks():
    p = {"hbm_gbs": 6524.0, "bf16_tflops": 1657.6, "bf16_tflops_sustained": 1413.6, "src": "measured"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: float(m[k]) for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
    except (OSError, ValueError, KeyError):
        p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}
    return p


class Clocks:
    """SM clock / throttle-reason sampling during the timed region
    (B200_PROFILING.md clocks line), in-process through NVML on a background
    thread. SD_BENCH_CLOCKS=smi uses an nvidia-smi subprocess instead;
    SD_BENCH_CLOCKS=off disables sampling (reported as such)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, dev, interval=0.25):
        import threading
        self.mode = os.environ.get("SD_BENCH_CLOCKS", "nvml")
        self.samples, self.reasons, self.mx = [], set(), None
        self._stop = threading.Event()
        self.t = None
        self.p = None
        if self.mode == "off":
            return
        if self.mode == "smi":
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms", "250"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except OSError:
                self.p = None
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[dev]) if vis else dev
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001
            self.mode = "unavailable"
            return

        def loop():
            while not self._stop.is_set():
                try:
                    self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for n, bit in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(n)
                except Exception:  # noqa: BLE001
                    pass
                self._stop.wait(interval)

        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()

    def stop(self):
        if self.mode == "smi" and self.p:
            self.p.terminate()
            out, _ = self.p.communicate(timeout=10)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in out.strip().splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) < 6:
                    continue
                try:
                    self.samples.append(float(f[0]))
                    self.mx = float(f[1])
                except ValueError:
                    continue
                for n, v in zip(names, f[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(n)
        if self.t:
            self._stop.set()
            self.t.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "samples": 0,
                    "reasons": [f"clock sampling {self.mode}"]}
        loaded = [x for x in self.samples if x > 0.5 * (self.mx or 1)] or self.samples
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.mx, "samples": len(self.samples),
                "source": self.mode, "reasons": sorted(self.reasons)}


# ------------------------------------------------------------ CPU baseline
def cpu_estimate(wl, threads, reps=1):
    """Reference CPU path (the oracle port of KvShard::attend and
    apply_linear/finish_block, built -O2 -ffp-contract=off) timed on this
    host on a bounded sample, turned into decode tokens/s with the
    reference's own performance model: step = N*(T(B) + R(B)) + head
    (serial S then R, as in decode_step_monolithic; dense.cpp:90-129)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    L, D, H, Hkv, F, V, B, ctx, fmt, _ = wl
    spec = oracle.make_spec(1, D, H, F, 8, Hkv)
    n_s = max(2 * threads, 8)
    b_s = 16
    t0 = time.perf_counter()
    t_att = oracle.bench_attend(spec, n_s, ctx, fmt, threads, reps)
    t_dense = oracle.bench_dense(spec, b_s, threads, reps)
    wall = time.perf_counter() - t0
    kvw = Hkv * (D // H)
    flop_tok_layer = 2 * D * (D + 2 * kvw) + 2 * D * D + 4 * D * F
    dense_flops = b_s * flop_tok_layer / t_dense
    r_layer = t_att * B / n_s
    s_layer = t_dense * B / b_s
    head = 2.0 * D * V * B / dense_flops
    step = L * (s_layer + r_layer) + head
    kv_bytes = n_s * ctx * 2 * kvw * {"single": 4, "half": 2, "int8": 1}[fmt]
    return {"value": B / step, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": (f"oracle KvShard::attend over {n_s} seqs x ctx {ctx} ({fmt} KV, 1 layer) + "
                       f"project_qkv/finish_block at B={b_s} (1 layer), {threads} host threads; "
                       f"scaled by the reference model B/(N*(T(B)+R)+head) to B={B}, N={L}"),
            "r_part_gbs": kv_bytes / t_att / 1e9, "dense_gflops": dense_flops / 1e9,
            "sample_wall_s": wall}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------- ours, N GPUs
def run_dist(args, wl, rank, world, dev, dist):
    """DistributedComputation over NCCL (workers.cpp:264-501): every rank an
    R-shard of the sequences ShardMap by-sequence gives it, every rank an
    S-worker for its home rows (seq % N); per layer Q/K/V rows go to the
    owning shard and O rows come back over NVLink. Weak scaling: B rows and
    ~B KV sequences per GPU."""
    import numpy as np
    import torch
    import paper_2403_11421_b200 as sd

    L, D, H, Hkv, F, V, B, ctx, fmt, dense = wl
    pk = peaks()
    spec = sd.make_model_spec(L, D, H, F, V, Hkv)
    steps_total = args.warmup + args.steps + args.e2e_steps + 8
    s_ranks = world if args.s_ranks == 0 else args.s_ranks
    seqs = list(range(1, B * world + 1))
    mode = args.shard_mode
    if mode != "sequence" and args.exchange != "p2p":
        raise SystemExit("--shard-mode head/hybrid needs --exchange p2p")
    plan = sd.dist_plan(world, rank, s_ranks, seqs, mode, Hkv, home=args.home)
    h0, hc = (0, Hkv) if mode == "sequence" else sd.ShardMap(mode, Hkv, world).head_range(rank)
    mine = [seqs[i] for i in plan["shard_rows"]]
    nmax = torch.tensor([len(mine)], device=f"cuda:{dev}")
    dist.all_reduce(nmax, op=dist.ReduceOp.MAX)
    cap_seqs = int(nmax.item())
    is_s = s_ranks == world or rank == 0
    weights = sd.DeviceWeights(spec, None, dense, dev, seed=0) if is_s else None
    kv = sd.KvShard(spec, h0, hc, cap_seqs * (ctx + steps_total), fmt, dev,
                    max_sequences=cap_seqs, max_seq_len=ctx + steps_total + 16)
    kv.prefill_synthetic(mine, ctx, salt=rank)
    obj = [sd.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    eng = sd.DistEngine(weights, kv, rank, world, obj[0], s_ranks, shard_mode=mode, home=args.home)
    if args.exchange == "p2p":  # direct NVLink stores into the peers' receive buffers
        eng.enable_p2p(len(seqs))
    tokens = np.array([sd.prompt_token(0, s, V) for s in seqs], dtype=np.int32)

    # the clock sampler starts before warm-up: nvidia-smi's NVML start-up can
    # stall the driver for ~100 ms, which must not land in the timed region
    clk = Clocks(dev)
    eng.bench(seqs, tokens, args.warmup)
    torch.cuda.synchronize(dev)
    kv.timing(TIMING_EVERY)
    eng.timing(True)
    kv.timing_read(reset=True)
    eng.timing_read(reset=True)
    dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = sd.launch_count()
    ms = eng.bench(seqs, tokens, args.steps)
    l1 = sd.launch_count()
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    a_ms, a_n, a_bytes = kv.timing_read()
    x_ms, x_bytes = eng.timing_read()
    kv.timing(False)
    eng.timing(False)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = B * world * args.steps / (ms / 1e3)

    pin_in = torch.empty(len(seqs), dtype=torch.int32).pin_memory().numpy()
    pin_in[:] = tokens
    eng.compute(seqs, pin_in)  # untimed: NCCL connects the token all-reduce lazily
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        nxt, _ = eng.compute(seqs, pin_in)
        pin_in[:] = nxt  # the whole batch's next tokens on every rank
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    eng.close()
    kv.close()
    if weights is not None:
        weights.close()
    achieved = a_bytes / (a_ms / 1e3) / 1e9 if a_ms > 0 else 0.0
    return {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-hash weights and KV prefill; no checkpoint)",
        "config": {"workload": args.workload, "model": "Llama-3-8B GQA shape (reference 2-matrix SiLU MLP)",
                   "layers": L, "model_dim": D, "heads": H, "kv_heads": Hkv, "mlp_dim": F, "vocab": V,
                   "batch_per_gpu": B, "global_batch": B * world, "context": ctx, "kv_format": fmt,
                   "s_part": f"{dense} tcgen05, fp32 accumulate", "r_part": "fp32 math over fp16 KV",
                   "parallelism": (f"kv sharded by mix64(seq)%{world} (ShardMap by-sequence); " if mode == "sequence"
                                   else f"kv sharded {mode} over {Hkv} kv heads (ShardMap {mode}); ")
                                  + f"{s_ranks} S-rank(s)"
                                  + (f" with {args.home} homes" if s_ranks == world and mode == "sequence" else "")
                                  + "; per-layer Q/K/V->shard, O->S over "
                                  + ("NVLink peer stores (CUDA IPC)" if args.exchange == "p2p" else "NCCL send/recv"),
                   "l2": "inputs larger than L2 (KV cache 1000x the 126 MB L2)"},
        "roofline": {"bound": "hbm", "kernel": "attention (rank 0)", "achieved": achieved,
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                     "traffic": None, "launches": a_n, "ms_per_launch": a_ms / max(a_n, 1),
                     "launches_timed_of": args.steps * L,
                     "share_of_step": (a_ms / max(a_n, 1)) * args.steps * L / ms if ms else None},
        "exchange": {"ms_per_step": x_ms / args.steps, "bytes_per_step_rank0": x_bytes / args.steps,
                     "gbs": x_bytes / (x_ms / 1e3) / 1e9 if x_ms else None, "shard_rows_rank0": len(mine),
                     "home_rows_rank0": len(plan["home_rows"]),
                     "remote_rows_rank0": int(sum(c for d, c in enumerate(plan["send_counts"]) if d != rank)),
                     "max_shard_rows": cap_seqs},
        "e2e": {"value": B * world * args.e2e_steps / e2e_s, "unit": "tokens/s",
                "h2d_bytes_per_step": int(len(plan["home_rows"]) * 4),
                "d2h_bytes_per_step": int(len(seqs) * 4),  # every rank reads the batch's next tokens
                "steps": args.e2e_steps, "api": "sd_dist_step (include/sd_abi.h)"},
        "gpu_launches": int(l1 - l0),
        "clocks": clocks,
    }


# ------------------------------------------------------------------ ours
def run_ours(args, wl, rank, world, dev, dist):
    if world > 1:
        return run_dist(args, wl, rank, world, dev, dist)
    import numpy as np
    import torch
    import paper_2403_11421_b200 as sd

    L, D, H, Hkv, F, V, B, ctx, fmt, dense = wl
    pk = peaks()
    spec = sd.make_model_spec(L, D, H, F, V, Hkv)
    steps_total = args.warmup + args.steps + args.e2e_steps + 8
    weights = sd.DeviceWeights(spec, None, dense, dev, seed=rank)
    kv = sd.KvShard(spec, 0, spec.num_kv_heads, B * (ctx + steps_total), fmt, dev,
                    max_sequences=B, max_seq_len=ctx + steps_total + 16)
    eng = sd.Engine(weights, kv)
    if args.r_sms > 0:  # two-mini-batch S/R pipeline (workers.cpp:405-452)
        eng.pipeline(True, args.r_sms)
    # sequence ids of this rank's shard: ids whose mix64 hash lands here
    # (ShardMap by-sequence, transport.cpp:352-353), B per GPU
    seqs, q = [], 1
    while len(seqs) < B:
        if world == 1 or sd.mix64(q) % world == rank:
            seqs.append(q)
        q += 1
    kv.prefill_synthetic(seqs, ctx, salt=rank)
    tokens = np.array([sd.prompt_token(0, s, V) for s in seqs], dtype=np.int32)

    # warm-up (untimed); the clock sampler starts first (see run_dist)
    clk = Clocks(dev)
    _, tok = eng.bench(seqs, tokens, args.warmup)
    torch.cuda.synchronize(dev)

    # ---- device-timed region: K steps, CUDA events on the engine stream
    # (SD_BENCH_NO_KTIMING=1: no per-kernel events, for A/B experiments only;
    # the roofline fields are then empty)
    # per-kernel CUDA events on every 8th layer only (layers are identical;
    # an event pair around every launch costs ~1 ms of a ~28 ms step)
    every = 0 if os.environ.get("SD_BENCH_NO_KTIMING") else TIMING_EVERY
    kv.timing(every)
    eng.timing(every)
    kv.timing_read(reset=True)
    eng.timing_read(reset=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = sd.launch_count()
    ms, tok = eng.bench(seqs, tok, args.steps)
    l1 = sd.launch_count()
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    a_ms, a_n, a_bytes = kv.timing_read()
    g_ms, g_flops, g_n = eng.timing_read()
    kv.timing(False)
    eng.timing(False)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tokens_total = B * world * args.steps
    value = tokens_total / (ms / 1e3)

    # ---- end to end through the public C-ABI with host buffers: every step
    # copies the step's token ids H2D from pinned memory and reads the next
    # tokens back D2H (sd_engine_step is synchronous)
    pin_in = torch.empty(B, dtype=torch.int32).pin_memory().numpy()
    pin_in[:] = tok
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        nxt, _ = eng.compute(seqs, tokens=pin_in)
        pin_in[:] = nxt
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": B * world * args.e2e_steps / e2e_s, "unit": "tokens/s",
           "h2d_bytes_per_step": int(B * 4), "d2h_bytes_per_step": int(B * 4),
           "steps": args.e2e_steps, "api": "sd_engine_step (include/sd_abi.h)"}

    eng.close()
    kv.close()
    weights.close()

    extra = {}
    if rank == 0 and world == 1 and not args.no_c2:
        extra["r_part_c2"] = rpart_c2(sd, torch, dev, pk)
    achieved = a_bytes / (a_ms / 1e3) / 1e9 if a_ms > 0 else 0.0
    hd = D // H
    step_flops = 2.0 * B * (L * (D * (H + 2 * Hkv) * hd + D * D + 2 * D * F) + D * V)  # this rank's GEMMs
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_attention_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                traffic = json.load(f).get(args.workload)
        except (OSError, ValueError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-hash weights and KV prefill; no checkpoint)",
        "config": {"workload": args.workload, "model": "Llama-3-8B GQA shape (reference 2-matrix SiLU MLP)",
                   "layers": L, "model_dim": D, "heads": H, "kv_heads": Hkv, "mlp_dim": F, "vocab": V,
                   "batch_per_gpu": B, "global_batch": B * world, "context": ctx, "kv_format": fmt,
                   "s_part": f"{dense} tcgen05, fp32 accumulate", "r_part": "fp32 math over fp16 KV",
                   "parallelism": f"kv-sharded x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (KV cache 1000x the 126 MB L2)"},
        "roofline": {"bound": "hbm", "kernel": "attn_mma_kernel (split-K decode attention, mma.sync over fp16 KV)",
                     "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                     "launches": a_n, "ms_per_launch": a_ms / max(a_n, 1),
                     "launches_timed_of": args.steps * L * (2 if args.r_sms > 0 else 1),
                     "share_of_step": (a_ms / max(a_n, 1)) * args.steps * L * (2 if args.r_sms > 0 else 1) / ms
                     if ms else None,
                     "peak_src": pk["src"] + " (MEASURED_PEAKS.json hbm_gbs)"},
        "s_part": {"bound": "tensor", "achieved": g_flops / (g_ms / 1e3) / 1e12 if g_ms else 0.0,
                   "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                   "frac": (g_flops / (g_ms / 1e3) / 1e12) / pk["bf16_tflops_sustained"] if g_ms else 0.0,
                   "share_of_step": (g_ms * step_flops * args.steps / g_flops) / ms if ms and g_flops else None,
                   "launches": g_n, "timing": f"CUDA events on the GEMMs of every {TIMING_EVERY}th layer + head"},
        "e2e": e2e,
        "gpu_launches": int(l1 - l0),
        "clocks": clocks,
    }
    line.update(extra)
    return line


def rpart_c2(sd, torch, dev, pk):
    """BASELINE config 2 R-Part: Llama-2-7B heads (32 x 128, MHA), B=1024,
    ctx 1024, fp16 KV, one layer resident (full depth needs 550 GB)."""
    spec = sd.make_model_spec(1, 4096, 32, 11008, 32000)
    B, ctx = 1024, 1024
    kv = sd.KvShard(spec, 0, 32, B * (ctx + 1), "half", dev, max_sequences=B, max_seq_len=ctx + 16)
    seqs = list(range(1, B + 1))
    kv.prefill_synthetic(seqs, ctx)
    q = torch.randn(B, 4096, device=f"cuda:{dev}")
    o = torch.empty_like(q)
    for _ in range(3):
        kv.attend_dev(0, seqs, q.data_ptr(), o.data_ptr())
    torch.cuda.synchronize(dev)
    kv.timing(True)
    kv.timing_read(reset=True)
    for _ in range(10):
        kv.attend_dev(0, seqs, q.data_ptr(), o.data_ptr())
    ms, n, byt = kv.timing_read()
    kv.close()
    gbs = byt / (ms / 1e3) / 1e9
    return {"workload": "c2 Llama-2-7B MHA heads, B=1024, ctx 1024, fp16 KV, 1 layer",
            "ms_per_layer": ms / n, "achieved_gbs": gbs, "frac": gbs / pk["hbm_gbs"],
            "projected_32_layer_r_ms": 32 * ms / n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT, choices=sorted(WORKLOADS))
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--r-sms", type=int, default=0,
                    help="two-mini-batch S/R pipeline: SMs for the R-Part (0 = off)")
    ap.add_argument("--s-ranks", type=int, default=0,
                    help="N>1: S-workers (1 = the paper's single S-rank; 0 = every rank)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N>1: per-layer activation exchange transport")
    ap.add_argument("--home", default="affinity", choices=["affinity", "modulo"],
                    help="N>1, data-parallel S-ranks, by-sequence: S-Part placement (affinity: balanced "
                         "homes on the KV's own rank where possible; modulo: seq %% world)")
    ap.add_argument("--shard-mode", default="sequence", choices=["sequence", "head", "hybrid"],
                    help="N>1: ShardMap mode of the KV shards (head/hybrid need --exchange p2p)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        # the reference CPU path (oracle port), rank 0 only, all host threads
        if rank != 0:
            return
        threads = host_threads()
        vals, last = [], None
        for _ in range(args.warmup if args.warmup < 2 else 1):
            cpu_estimate(wl, threads)
        for _ in range(args.steps):
            last = cpu_estimate(wl, threads)
            vals.append(last["value"])
        v = statistics.median(vals)
        L, D, H, Hkv, F, V, B, ctx, fmt, dense = wl
        out = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * B / v,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic", "impl": "reference",
               "config": {"workload": args.workload, "batch_per_gpu": B, "context": ctx,
                          "kv_format": fmt, "layers": L},
               "cpu_baseline": {k: last[k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": "tokens/s"},
               "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    import torch
    dist = None
    if world > 1:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist = tdist
    torch.cuda.set_device(local)
    line = run_ours(args, wl, rank, world, local, dist)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_estimate(wl, host_threads())
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
