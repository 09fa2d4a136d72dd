"""Host-side mirror of the reference `splitdecode` hot-path interfaces over
the C-ABI (include/sd_abi.h). Names, argument meaning and error types follow
the reference:

  KvShard            attention.hpp:68-140   (R-Part worker interface)
  project_qkv ...    dense.hpp:20-50        (S-Part step interface)
  Engine             workers.hpp:151-158    (StepComputation on the GPU)
  run_generation     workers.cpp:547-701    (drive_schedule over the engine)
  ShardMap           transport.hpp:150-170
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from ._lib import (DriveConfig, FP, I32P, I64P, KvOptions, ModelSpec, U32P, U64P, lib)

# ------------------------------------------------------------------ errors
class SplitDecodeError(RuntimeError):
    code = 6


class ConfigError(SplitDecodeError):       # core.hpp:25-28
    code = 8


class ProtocolError(SplitDecodeError):     # core.hpp:30-33
    code = 3


class UnknownSequenceError(ProtocolError):  # attention.hpp:19-22
    code = 5


class CapacityError(SplitDecodeError):     # core.hpp:35-38
    code = 4


class LogicError(SplitDecodeError):        # std::logic_error
    code = 7


class AdmissionError(SplitDecodeError):    # scheduler.hpp:20-23
    code = 11


class CudaError(SplitDecodeError):
    code = 9


class InfeasiblePlanError(SplitDecodeError):  # planner.hpp:18-23
    code = 12
    tightest_batch = 0


_BY_CODE = {c.code: c for c in (ConfigError, ProtocolError, UnknownSequenceError, CapacityError,
                                LogicError, AdmissionError, CudaError, InfeasiblePlanError)}


def _check(rc: int):
    if rc != 0:
        msg = lib.sd_last_error().decode()
        raise _BY_CODE.get(rc, SplitDecodeError)(msg)


FORMATS = {"single": 0, "half": 1, "int8": 2, "int4": 3}
DENSE_MODES = {"exact": 0, "bf16": 1, "tf32": 2, "fp16": 3}
SHARD_MODES = {"by-sequence": 0, "by-head": 1, "hybrid": 2, "sequence": 0, "head": 1}
# home (S-Part) placement with data-parallel S-ranks (SD_HOME_MODULO, include/sd_abi.h)
HOME_POLICIES = {"affinity": 0, "modulo": 0x100}


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(FP)


def _u64(seqs):
    a = np.ascontiguousarray(seqs, dtype=np.uint64)
    return a, a.ctypes.data_as(U64P)


# -------------------------------------------------------------------- core
def make_model_spec(num_layers: int, model_dim: int, num_heads: int, mlp_dim: int,
                    vocab_size: int, num_kv_heads: int = 0) -> ModelSpec:
    """make_model_spec (core.cpp:11-30)."""
    s = ModelSpec()
    _check(lib.sd_make_model_spec(num_layers, model_dim, num_heads, mlp_dim, vocab_size,
                                  num_kv_heads, C.byref(s)))
    return s


def launch_count() -> int:
    """Kernel launches issued by libsd_b200 in this process."""
    return int(lib.sd_launch_count())


_TUNED = {"gemm_bn": 0, "gemm_pair": 1, "fused_append": 1, "fused_argmax": 1, "dist_fuse": 1,
          "attn_mma": 1, "pdl": 1, "dist_phases": 0, "attn_i8_quad": 1,
          "attn_l2_prefetch": 0, "attn_max_stages": 0, "attn_imma": 1,
          "attn_rps8": 1, "attn_ivalue": 1}


def tune(name: str, value: int):
    """Process-wide tuning switch (sd_tune); defaults are the measured-best paths."""
    _check(lib.sd_tune(name.encode(), int(value)))


class tuned:
    """Context manager: set tuning switches, restore the defaults on exit."""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        for k, v in self.kw.items():
            tune(k, v)
        return self

    def __exit__(self, *exc):
        for k in self.kw:
            tune(k, _TUNED[k])
        return False


def mix64(x: int) -> int:
    return int(lib.sd_mix64(x & (2**64 - 1)))


def prompt_token(seed: int, seq: int, vocab_size: int) -> int:
    return int(lib.sd_prompt_token(seed, seq, vocab_size))


# ------------------------------------------------------------------ R-Part
@dataclass
class AttentionItem:
    """AttentionItem (attention.hpp:44-48)."""
    seq: int
    position: int
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray


@dataclass
class AttentionRequest:
    """AttentionRequest (attention.hpp:50-53)."""
    layer: int = 0
    items: list = field(default_factory=list)


class KvShard:
    """KvShard (attention.hpp:68-140) on a B200: paged HBM KV store plus the
    split-K decode-attention kernel. head_start / head_count index kv heads."""

    def __init__(self, spec: ModelSpec, head_start: int, head_count: int, capacity_tokens: int,
                 fmt: str = "single", device: int = 0, max_sequences: int = 0,
                 max_seq_len: int = 0, page_positions: int = 0, pool_pages: int = 0):
        self.spec = spec
        self.h = C.c_void_p()
        opts = KvOptions(max_sequences, max_seq_len, page_positions, pool_pages)
        _check(lib.sd_kv_create(C.byref(spec), head_start, head_count, capacity_tokens,
                                FORMATS[fmt], device, C.byref(opts), C.byref(self.h)))
        w, qw = C.c_int32(), C.c_int32()
        _check(lib.sd_kv_width(self.h, C.byref(w), C.byref(qw)))
        self._width, self.q_width = w.value, qw.value
        self._fmt = fmt
        self._head_start, self._head_count = head_start, head_count
        self._capacity = capacity_tokens

    def close(self):
        if getattr(self, "h", None):
            lib.sd_kv_destroy(self.h)
            self.h = None

    __del__ = close

    # queries (attention.hpp:73-111)
    def head_start(self): return self._head_start
    def head_count(self): return self._head_count
    def width(self): return self._width
    def format(self): return self._fmt
    def capacity(self): return self._capacity

    def token_count(self) -> int:
        out = C.c_int64()
        _check(lib.sd_kv_token_count(self.h, C.byref(out)))
        return out.value

    def has_sequence(self, seq: int) -> bool:
        out = C.c_int32()
        _check(lib.sd_kv_has_sequence(self.h, seq, C.byref(out)))
        return bool(out.value)

    def stored_length(self, seq: int, layer: int) -> int:
        out = C.c_int32()
        _check(lib.sd_kv_stored_length(self.h, seq, layer, C.byref(out)))
        return out.value

    def warning_count(self) -> int:
        out = C.c_int32()
        _check(lib.sd_kv_warning_count(self.h, C.byref(out)))
        return out.value

    def bytes_per_token(self) -> int:
        out = C.c_int64()
        _check(lib.sd_kv_bytes_per_token(self.h, C.byref(out)))
        return out.value

    # operations
    def append(self, seq: int, layer: int, position: int, k, v):
        """KvShard::append (attention.hpp:91-92)."""
        k, v = _f32(k), _f32(v)
        if k.size != self._width or v.size != self._width:
            raise ProtocolError("append: K/V width does not match the shard's head range")
        _check(lib.sd_kv_append(self.h, seq, layer, position, _fp(k), _fp(v)))

    def append_request(self, request_or_layer, seqs=None, positions=None, k=None, v=None):
        """KvShard::append_request (attention.hpp:96). Accepts an
        AttentionRequest or (layer, seqs, positions, k[n,w], v[n,w])."""
        layer, seqs, positions, k, v = self._unpack(request_or_layer, seqs, positions, k, v)
        s, sp = _u64(seqs)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        k, v = _f32(k).reshape(len(s), -1), _f32(v).reshape(len(s), -1)
        if len(s) and (k.shape[1] != self._width or v.shape[1] != self._width):
            raise ProtocolError("append: K/V width does not match the shard's head range")
        _check(lib.sd_kv_append_request(self.h, layer, len(s), sp, pos.ctypes.data_as(U32P),
                                        _fp(k), _fp(v)))

    def attend(self, request_or_layer, seqs=None, q=None) -> np.ndarray:
        """KvShard::attend (attention.hpp:102); returns O rows in item order."""
        if isinstance(request_or_layer, AttentionRequest):
            r = request_or_layer
            layer, seqs = r.layer, [it.seq for it in r.items]
            q = np.stack([_f32(it.q) for it in r.items]) if r.items else np.zeros((0, self.q_width))
        else:
            layer = request_or_layer
        s, sp = _u64(seqs)
        q = _f32(q).reshape(len(s), -1)
        if len(s) and q.shape[1] != self.q_width:
            raise ProtocolError("attend: Q width does not match the shard's head range")
        o = np.zeros((len(s), self.q_width), dtype=np.float32)
        _check(lib.sd_kv_attend(self.h, layer, len(s), sp, _fp(q), _fp(o)))
        return o

    def append_attend(self, layer, seqs, positions, q, k, v) -> np.ndarray:
        """append_request + attend, the R-worker QKV handler (workers.cpp:110-111)."""
        s, sp = _u64(seqs)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        q, k, v = (_f32(a).reshape(len(s), -1) for a in (q, k, v))
        o = np.zeros((len(s), self.q_width), dtype=np.float32)
        _check(lib.sd_kv_append_attend(self.h, layer, len(s), sp, pos.ctypes.data_as(U32P),
                                       _fp(q), _fp(k), _fp(v), _fp(o)))
        return o

    def append_attend_dev(self, layer, seqs, positions, q_ptr, k_ptr, v_ptr, o_ptr, stream=0):
        """Device-pointer variant (e.g. torch CUDA tensors' data_ptr())."""
        s, sp = _u64(seqs)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        _check(lib.sd_kv_append_attend_dev(self.h, layer, len(s), sp, pos.ctypes.data_as(U32P),
                                           q_ptr, k_ptr, v_ptr, o_ptr, stream))

    def attend_dev(self, layer, seqs, q_ptr, o_ptr, stream=0):
        s, sp = _u64(seqs)
        _check(lib.sd_kv_attend_dev(self.h, layer, len(s), sp, q_ptr, o_ptr, stream))

    def drop_sequence(self, seq: int):
        """KvShard::drop_sequence (attention.hpp:106)."""
        s, sp = _u64([seq])
        _check(lib.sd_kv_drop(self.h, 1, sp))

    def export_lane(self, seq: int, layer: int, which: int):
        """Stored bytes of lane K (0) / V (1) in the reference [pos][head][d]
        order, plus int8 / int4 scales [pos][head]."""
        n = lib.sd_kv_export_lane(self.h, seq, layer, which, None, 0, None, 0)
        if n < 0:
            _check(int(-n))
        buf = np.zeros(n, dtype=np.uint8)
        L = self.stored_length(seq, layer)
        sc = np.zeros(L * self._head_count, np.float32) if self._fmt in ("int8", "int4") else None
        r = lib.sd_kv_export_lane(self.h, seq, layer, which, buf.ctypes.data_as(C.c_void_p), n,
                                  _fp(sc) if sc is not None else None,
                                  sc.size if sc is not None else 0)
        if r < 0:
            _check(int(-r))
        return buf, sc

    def prefill_synthetic(self, seqs, length: int, salt: int = 0):
        s, sp = _u64(seqs)
        _check(lib.sd_kv_prefill_synthetic(self.h, len(s), sp, length, salt))

    def timing(self, enable):
        """CUDA-event timing of the attention launches: False/0 off, True/1
        every launch, k > 1 the launches of every k-th layer."""
        _check(lib.sd_kv_timing(self.h, int(enable)))

    def timing_read(self, reset=True):
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        _check(lib.sd_kv_timing_read(self.h, C.byref(ms), C.byref(n), C.byref(b), int(reset)))
        return ms.value, n.value, b.value

    @staticmethod
    def _unpack(r, seqs, positions, k, v):
        if isinstance(r, AttentionRequest):
            items = r.items
            return (r.layer, [it.seq for it in items], [it.position for it in items],
                    np.stack([_f32(it.k) for it in items]) if items else np.zeros((0, 1), np.float32),
                    np.stack([_f32(it.v) for it in items]) if items else np.zeros((0, 1), np.float32))
        return r, seqs, positions, k, v


# ------------------------------------------------------------------ S-Part
class DeviceWeights:
    """WeightSet (core.hpp:85-90) uploaded to a device. `tensors` follow the
    reference storage: [embedding (D x V), per layer w_q, w_k, w_v, w_o,
    w_mlp_in, w_mlp_out, head (V x D)], each a flat column-major buffer.
    tensors=None generates the weights: generator "reference" is
    seed_random_weights(spec, seed) (core.cpp:97-127), bit-identical to the
    reference's WeightSet (host mt19937 stream, uploaded); "counter" is a
    device-side counter hash of the same distribution (fast, not the
    reference's values)."""

    def __init__(self, spec: ModelSpec, tensors: Sequence[np.ndarray] | None, mode: str = "exact",
                 device: int = 0, seed: int = 0, generator: str = "counter"):
        self.spec = spec
        self.mode = mode
        self.h = C.c_void_p()
        if tensors is None and generator == "reference":
            _check(lib.sd_weights_seed_random(C.byref(spec), seed, DENSE_MODES[mode], device,
                                              C.byref(self.h)))
        elif tensors is None:
            if generator != "counter":
                raise ConfigError(f"unknown weight generator {generator!r}")
            _check(lib.sd_weights_synthetic(C.byref(spec), DENSE_MODES[mode], seed, device,
                                            C.byref(self.h)))
        else:
            self._keep = [_f32(t).reshape(-1) for t in tensors]
            arr = (FP * len(self._keep))(*[_fp(t) for t in self._keep])
            _check(lib.sd_weights_upload(C.byref(spec), arr, DENSE_MODES[mode], device,
                                         C.byref(self.h)))
            self._keep = None

    def embedding_host(self, out=None) -> np.ndarray:
        """The embedding as stored, as a (vocab, model_dim) array whose row t is
        embedding column t (the TokenBatch.features of token t)."""
        shape = (self.spec.vocab_size, self.spec.model_dim)
        if out is None:
            out = np.empty(shape, np.float32)
        assert out.dtype == np.float32 and out.flags["C_CONTIGUOUS"] and out.size >= shape[0] * shape[1]
        _check(lib.sd_weights_export_embedding(self.h, _fp(out), out.size))
        return out.reshape(shape)

    def close(self):
        if getattr(self, "h", None):
            lib.sd_weights_destroy(self.h)
            self.h = None

    __del__ = close


def project_qkv(w: DeviceWeights, layer: int, x):
    """project_qkv (dense.hpp:26-27) -> (q, k, v)."""
    x = _f32(x)
    B = x.shape[0]
    s = w.spec
    kvw = s.num_kv_heads * s.head_dim
    q = np.zeros((B, s.model_dim), np.float32)
    k = np.zeros((B, kvw), np.float32)
    v = np.zeros((B, kvw), np.float32)
    _check(lib.sd_s_project_qkv(w.h, layer, B, _fp(x), _fp(q), _fp(k), _fp(v)))
    return q, k, v


def finish_block(w: DeviceWeights, layer: int, o, residual):
    """finish_block (dense.hpp:31-32)."""
    o, r = _f32(o), _f32(residual)
    out = np.zeros_like(r)
    _check(lib.sd_s_finish_block(w.h, layer, o.shape[0], _fp(o), _fp(r), _fp(out)))
    return out


def output_logits_argmax(w: DeviceWeights, x):
    """output_logits + argmax_token (dense.hpp:35-38) -> (logits, tokens)."""
    x = _f32(x)
    B = x.shape[0]
    lg = np.zeros((B, w.spec.vocab_size), np.float32)
    tk = np.zeros(B, np.int32)
    _check(lib.sd_s_logits_argmax(w.h, B, _fp(x), _fp(lg), tk.ctypes.data_as(I32P)))
    return lg, tk


def apply_linear(w: DeviceWeights, layer: int, which: int, x):
    """apply_linear (dense.hpp:20) over uploaded tensor `which`."""
    x = _f32(x)
    outs = {1: w.spec.model_dim, 2: w.spec.num_kv_heads * w.spec.head_dim,
            3: w.spec.num_kv_heads * w.spec.head_dim, 4: w.spec.model_dim, 5: w.spec.mlp_dim,
            6: w.spec.model_dim, 7: w.spec.vocab_size}
    y = np.zeros((x.shape[0], outs[which]), np.float32)
    _check(lib.sd_s_apply_linear(w.h, layer, which, x.shape[0], _fp(x), _fp(y)))
    return y


def gemm_dev(kind: str, M: int, N: int, K: int, A, lda, B, ldb, C=None, ldc=0, Cb=None, ldcb=0,
             epi: int = 0, res=None, ldr=0, stream=0):
    """tcgen05 GEMM on device pointers (ints, e.g. torch .data_ptr()):
    C = A . B^T (+ epilogue). kind: "bf16" | "fp16" | "tf32"."""
    _check(lib.sd_gemm_dev(DENSE_MODES[kind], M, N, K, A, lda, B, ldb, C, ldc, Cb, ldcb, epi, res,
                           ldr, stream))


# ----------------------------------------------------------------- runtime
class Engine:
    """The GPU StepComputation (workers.hpp:151-158)."""

    def __init__(self, weights: DeviceWeights, kv: KvShard):
        self.weights, self.kv = weights, kv
        self.h = C.c_void_p()
        _check(lib.sd_engine_create(weights.h, kv.h, C.byref(self.h)))

    def close(self):
        if getattr(self, "h", None):
            lib.sd_engine_destroy(self.h)
            self.h = None

    __del__ = close

    def compute(self, seqs, tokens=None, features=None, want_final=False, want_logits=False,
                out_next=None, out_final=None):
        """StepComputation::compute -> DecodeStepResult(next_tokens, final_activations).
        out_next / out_final: caller-owned result buffers (e.g. pinned)."""
        s, sp = _u64(seqs)
        B = len(s)
        nxt = out_next if out_next is not None else np.zeros(B, np.int32)
        if out_final is not None:
            fx = out_final
        else:
            fx = np.zeros((B, self.weights.spec.model_dim), np.float32) if want_final else None
        if features is not None:
            x = _f32(features)
            lg = np.zeros((B, self.weights.spec.vocab_size), np.float32) if want_logits else None
            _check(lib.sd_engine_step_features(self.h, B, sp, _fp(x), nxt.ctypes.data_as(I32P),
                                               _fp(fx) if fx is not None else None,
                                               _fp(lg) if lg is not None else None))
            return nxt, fx, lg
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        _check(lib.sd_engine_step(self.h, B, sp, t.ctypes.data_as(I32P), nxt.ctypes.data_as(I32P),
                                  _fp(fx) if fx is not None else None))
        return nxt, fx

    def retire(self, seqs):
        s, sp = _u64(seqs)
        _check(lib.sd_engine_retire(self.h, len(s), sp))

    def pipeline(self, enable: bool, r_sms: int = 96):
        """Two-mini-batch S/R pipeline (workers.cpp:405-452): attention of one
        mini-batch on r_sms SMs beside the GEMMs of the other."""
        _check(lib.sd_engine_pipeline(self.h, int(enable), r_sms))

    def timing(self, enable):
        """CUDA-event timing of the S-Part GEMMs: False/0 off, True/1 every
        GEMM, k > 1 the GEMMs of every k-th layer (and the head)."""
        _check(lib.sd_engine_timing(self.h, int(enable)))

    def timing_read(self, reset=True):
        ms, fl, n = C.c_double(), C.c_double(), C.c_int64()
        _check(lib.sd_engine_timing_read(self.h, C.byref(ms), C.byref(fl), C.byref(n), int(reset)))
        return ms.value, fl.value, n.value

    def bench(self, seqs, tokens, steps: int):
        """Device-timed loop of `steps` decode steps; returns (ms, next_tokens)."""
        s, sp = _u64(seqs)
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        nxt = np.zeros(len(s), np.int32)
        ms = C.c_double()
        _check(lib.sd_engine_bench(self.h, len(s), sp, t.ctypes.data_as(I32P), steps,
                                   nxt.ctypes.data_as(I32P), C.byref(ms)))
        return ms.value, nxt


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes), to be broadcast to every rank."""
    buf = (C.c_uint8 * 128)()
    _check(lib.sd_nccl_unique_id(buf, 128))
    return bytes(buf)


def dist_plan(world: int, rank: int, s_ranks: int, seqs, shard_mode: str = "sequence", heads: int = 1,
              home: str = "affinity"):
    """Host row plan of one distributed step (sd_dist_plan); `heads` are the
    kv heads the ShardMap splits under by-head / hybrid sharding. `home`:
    "affinity" (balanced, shard-affine homes under by-sequence sharding with
    s_ranks == world) or "modulo" (home = seq % s_ranks)."""
    s, sp = _u64(seqs)
    B = len(s)
    flags = SHARD_MODES[shard_mode] | HOME_POLICIES[home]
    home = np.zeros(max(B, 1), np.int32)
    shard = np.zeros(max(B, 1), np.int32)
    nh, ns = C.c_int32(), C.c_int32()
    sc, rc = np.zeros(world, np.int32), np.zeros(world, np.int32)
    _check(lib.sd_dist_plan(world, rank, s_ranks, flags, heads, B, sp,
                            home.ctypes.data_as(I32P), C.byref(nh),
                            shard.ctypes.data_as(I32P), C.byref(ns), sc.ctypes.data_as(I32P),
                            rc.ctypes.data_as(I32P)))
    return {"home_rows": home[:nh.value].tolist(), "shard_rows": shard[:ns.value].tolist(),
            "send_counts": sc.tolist(), "recv_counts": rc.tolist()}


class DistEngine:
    """DistributedComputation (workers.cpp:264-501) over NCCL: this rank's
    R-shard (`kv`, sequences with mix64(seq) % world == rank) and, on
    S-ranks, the weights. s_ranks = 1: rank 0 is the only S-worker (the
    paper's topology); s_ranks = world: data-parallel S-workers."""

    def __init__(self, weights, kv: KvShard, rank: int, world: int, nccl_id: bytes | None,
                 s_ranks: int = 1, shard_mode: str = "sequence", home: str = "affinity"):
        """shard_mode: "sequence" (ShardMap by-sequence, the default), "head" or
        "hybrid" (over kv heads; `kv` holds this rank's head range, see
        ShardMap.head_range; needs enable_p2p before the first step).
        home: S-Part placement with s_ranks == world (see dist_plan)."""
        self.weights, self.kv, self.rank, self.world = weights, kv, rank, world
        self.spec = kv.spec
        self.h = C.c_void_p()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        _check(lib.sd_dist_create(weights.h if weights is not None else None, kv.h, rank, world,
                                  idbuf, s_ranks, SHARD_MODES[shard_mode] | HOME_POLICIES[home],
                                  C.byref(self.h)))

    def close(self):
        if getattr(self, "h", None):
            lib.sd_dist_destroy(self.h)
            self.h = None

    __del__ = close

    def compute(self, seqs, tokens, want_final=False):
        """One step over the full batch: next tokens of every row (homes can move
        between steps); final activations for this rank's home rows."""
        s, sp = _u64(seqs)
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        nxt = np.full(len(s), -1, np.int32)
        fx = np.zeros((len(s), self.spec.model_dim), np.float32) if want_final else None
        _check(lib.sd_dist_step(self.h, len(s), sp, t.ctypes.data_as(I32P), nxt.ctypes.data_as(I32P),
                                _fp(fx) if fx is not None else None))
        return nxt, fx

    def pipeline(self, enable: bool):
        """The reference's two interleaved mini-batches (seq % 2,
        workers.cpp:405-452); needs enable_p2p first when world > 1."""
        _check(lib.sd_dist_pipeline(self.h, int(enable)))

    def retire(self, seqs):
        s, sp = _u64(seqs)
        _check(lib.sd_dist_retire(self.h, len(s), sp))

    def bench(self, seqs, tokens, steps: int) -> float:
        s, sp = _u64(seqs)
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        ms = C.c_double()
        _check(lib.sd_dist_bench(self.h, len(s), sp, t.ctypes.data_as(I32P), steps, C.byref(ms)))
        return ms.value

    def timing(self, enable: bool):
        _check(lib.sd_dist_timing(self.h, int(enable)))

    def timing_read(self, reset=True):
        ms, b = C.c_double(), C.c_double()
        _check(lib.sd_dist_timing_read(self.h, C.byref(ms), C.byref(b), int(reset)))
        return ms.value, b.value

    IPC_BYTES = 384

    def p2p_handles(self, max_rows: int) -> bytes:
        """Allocate this rank's peer-exchange receive buffers (up to `max_rows`
        rows) and return their CUDA IPC handles."""
        buf = (C.c_uint8 * self.IPC_BYTES)()
        _check(lib.sd_dist_p2p_setup(self.h, int(max_rows), buf))
        return bytes(buf)

    def p2p_connect(self, all_handles):
        """Map every rank's buffers (handles in rank order) and switch the
        per-layer exchange from NCCL send/recv to direct NVLink stores."""
        blob = b"".join(all_handles)
        if len(blob) != self.IPC_BYTES * self.world:
            raise ConfigError("p2p_connect: need one handle block per rank")
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(lib.sd_dist_p2p_connect(self.h, buf))

    def enable_p2p(self, max_rows: int, group=None):
        """Collective over torch.distributed: exchange handles and connect."""
        import torch.distributed as dist
        mine = self.p2p_handles(max_rows)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self.p2p_connect(allh)


def run_generation(engine, batch: int, target_len: int, interval: int, steps: int,
                   seed: int = 0, cold_start: str = "fixed-interval", load_limit: int = 0,
                   record_activations: bool = False):
    """drive_schedule (workers.cpp:547-684) over the GPU engine (Engine or
    DistEngine) -> (transcript [(step, seq, token)], activations, wall_seconds).
    A DistEngine returns the rows its rank produced (its home rows)."""
    cfg = DriveConfig(batch, target_len, interval,
                      {"fixed-interval": 0, "ramped-limit": 1}[cold_start], steps, load_limit,
                      seed, int(record_activations))
    h = C.c_void_p()
    fn = lib.sd_dist_drive if isinstance(engine, DistEngine) else lib.sd_drive
    _check(fn(engine.h, C.byref(cfg), C.byref(h)))
    try:
        n = lib.sd_drive_count(h)
        st, sq, tk = C.c_int64(), C.c_uint64(), C.c_int32()
        recs = []
        for i in range(n):
            _check(lib.sd_drive_record(h, i, C.byref(st), C.byref(sq), C.byref(tk)))
            recs.append((st.value, sq.value, tk.value))
        acts = None
        if record_activations and n:
            p = lib.sd_drive_activations(h)
            D = engine.spec.model_dim if isinstance(engine, DistEngine) else engine.weights.spec.model_dim
            acts = np.ctypeslib.as_array(p, shape=(n * D,)).reshape(n, -1).copy()
        return recs, acts, lib.sd_drive_wall_seconds(h)
    finally:
        lib.sd_drive_destroy(h)


class RWorker:
    """A B200 attention worker speaking the reference's SDWP wire protocol
    (AttentionWorkerSession, workers.cpp:40-160): feed() takes stream bytes
    and returns the reply frames' bytes."""

    def __init__(self, capacity_tokens: int, fmt: str = "single", device: int = 0):
        self.h = C.c_void_p()
        _check(lib.sd_rworker_create(capacity_tokens, FORMATS[fmt], device, C.byref(self.h)))

    def close(self):
        if getattr(self, "h", None):
            lib.sd_rworker_destroy(self.h)
            self.h = None

    __del__ = close

    def feed(self, data: bytes) -> bytes:
        buf = C.create_string_buffer(bytes(data), len(data)) if data else None
        p, n = C.c_void_p(), C.c_size_t()
        _check(lib.sd_rworker_feed(self.h, buf, len(data), C.byref(p), C.byref(n)))
        return C.string_at(p, n.value) if n.value else b""

    def shutdown_requested(self) -> bool:
        v = C.c_int32()
        _check(lib.sd_rworker_shutdown_requested(self.h, C.byref(v)))
        return bool(v.value)


def serve_rworker(listen_addr: str, capacity_tokens: int, fmt: str = "single", device: int = 0,
                  port_file: str | None = None, once: bool = True, recv_timeout: float = 0.0):
    """serve_attention_worker (workers.cpp:162-214) on this process (blocking)."""
    _check(lib.sd_rworker_serve(listen_addr.encode(), port_file.encode() if port_file else None,
                                capacity_tokens, FORMATS[fmt], device, int(once), float(recv_timeout)))


def transcript_csv(recs) -> str:
    """transcript_csv (workers.cpp:746-755)."""
    return "step,seq_id,token_id\n" + "".join(f"{s},{q},{t}\n" for s, q, t in recs)


# ---------------------------------------------------------------- ShardMap
class ShardMap:
    """ShardMap (transport.hpp:150-170)."""

    def __init__(self, mode: str, num_heads: int, workers: int):
        self.mode, self.num_heads, self.workers = SHARD_MODES[mode], num_heads, workers
        self.head_range(0)  # validates

    def worker_for(self, seq: int, head: int) -> int:
        out = C.c_int32()
        _check(lib.sd_shardmap_worker_for(self.mode, self.num_heads, self.workers, seq, head,
                                          C.byref(out)))
        return out.value

    def head_range(self, worker: int):
        a, b = C.c_int32(), C.c_int32()
        _check(lib.sd_shardmap_head_range(self.mode, self.num_heads, self.workers, worker,
                                          C.byref(a), C.byref(b)))
        return a.value, b.value


def micro_batch_size(batch: int, interval: int, target_len: int) -> int:
    out = C.c_int32()
    _check(lib.sd_micro_batch_size(batch, interval, target_len, C.byref(out)))
    return out.value


def cold_start_schedule(batch, target_len, interval, mode="fixed-interval", horizon=0):
    m = {"fixed-interval": 0, "ramped-limit": 1}[mode]
    n = C.c_int64()
    cap = horizon + 2
    buf = np.zeros(3 * cap, np.int64)
    _check(lib.sd_cold_start_schedule(batch, target_len, interval, m, horizon,
                                      buf.ctypes.data_as(I64P), cap, C.byref(n)))
    return [tuple(int(x) for x in buf[3 * i:3 * i + 3]) for i in range(n.value)]
