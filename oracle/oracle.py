"""ctypes wrapper over the CPU ORACLE (oracle/sd_oracle.cpp).

TEST INFRASTRUCTURE ONLY. Imported by tests/, by __graft_entry__.smoke() as
the checker, and by bench.py's cpu_baseline / --impl reference legs. The
product package (paper_2403_11421_b200) never imports this module.

Every function restates a reference function; see the file:line citations in
sd_oracle.cpp. Activations are row-major numpy float32 arrays [rows, width];
weights keep the reference's column-major (out x in) storage.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libsd_oracle.so")

FORMATS = {"single": 0, "half": 1, "int8": 2, "int4": 3}
ERR_NAMES = {3: "ProtocolError", 4: "CapacityError", 5: "UnknownSequenceError",
             6: "InternalError", 7: "LogicError", 8: "ConfigError", 11: "AdmissionError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))


def build() -> str:
    """Compile the oracle (make); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    if not os.path.exists(_LIB_PATH):
        build()
    return C.CDLL(_LIB_PATH)


_lib = _load()


class Spec(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("num_layers", "model_dim", "num_heads", "head_dim",
                                        "mlp_dim", "vocab_size", "num_kv_heads")]


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
FP = C.POINTER(C.c_float)
U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)
IP = C.POINTER(C.c_int)
LP = C.POINTER(C.c_long)

_sig("orc_last_error", C.c_char_p)
_sig("orc_make_spec", C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Spec))
_sig("orc_mix64", C.c_uint64, C.c_uint64)
_sig("orc_prompt_token", C.c_int, C.c_uint64, C.c_uint64, C.c_int)
_sig("orc_f2h", C.c_uint16, C.c_float)
_sig("orc_h2f", C.c_float, C.c_uint16)
_sig("orc_quantize_int8", C.c_float, FP, C.c_int, C.POINTER(C.c_int8))
_sig("orc_quantize_int4", C.c_float, FP, C.c_int, C.POINTER(C.c_uint8))
_sig("orc_eigen_dot", C.c_float, FP, FP, C.c_int)
_sig("orc_synth_value", C.c_float, C.c_uint64)
_sig("orc_weights_create", C.c_int, C.POINTER(Spec), C.c_uint64, PP)
_sig("orc_weights_destroy", None, P)
_sig("orc_weights_checksum", C.c_uint64, P)
_sig("orc_weights_tensor", FP, P, C.c_int, C.c_int, IP, IP)
_sig("orc_kv_create", C.c_int, C.POINTER(Spec), C.c_int, C.c_int, C.c_long, C.c_int, PP)
_sig("orc_kv_destroy", None, P)
_sig("orc_kv_append", C.c_int, P, C.c_uint64, C.c_int, C.c_uint32, FP, FP)
_sig("orc_kv_append_request", C.c_int, P, C.c_int, C.c_int, U64P, U32P, FP, FP)
_sig("orc_kv_attend", C.c_int, P, C.c_int, C.c_int, U64P, FP, FP)
_sig("orc_kv_prefill_synthetic", C.c_int, P, C.c_int, U64P, C.c_int, C.c_uint64)
_sig("orc_kv_prefill_index", C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int)
_sig("orc_kv_drop", None, P, C.c_uint64)
_sig("orc_kv_stored_length", C.c_int, P, C.c_uint64, C.c_int)
_sig("orc_kv_token_count", C.c_long, P)
_sig("orc_kv_warning_count", C.c_int, P)
_sig("orc_kv_has_sequence", C.c_int, P, C.c_uint64)
_sig("orc_kv_bytes_per_token", C.c_size_t, P)
_sig("orc_kv_export_lane", C.c_long, P, C.c_uint64, C.c_int, C.c_int, P, C.c_size_t, FP, C.c_size_t)
_sig("orc_apply_linear", C.c_int, C.c_int, C.c_int, C.c_int, FP, FP, FP, C.c_int)
_sig("orc_project_qkv", C.c_int, P, C.c_int, C.c_int, U64P, FP, FP, FP, FP, C.c_int)
_sig("orc_finish_block", C.c_int, P, C.c_int, C.c_int, FP, FP, FP, C.c_int)
_sig("orc_output_logits", C.c_int, P, C.c_int, FP, FP, C.c_int)
_sig("orc_argmax", C.c_int, FP, C.c_int)
_sig("orc_decode_step", C.c_int, P, P, C.c_int, U64P, FP, IP, FP, FP, C.c_int)
_sig("orc_shardmap_worker_for", C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, IP)
_sig("orc_shardmap_head_range", C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, IP, IP)
_sig("orc_micro_batch_size", C.c_int, C.c_int, C.c_int, C.c_int, IP)
_sig("orc_cold_start_schedule", C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_long, LP, C.c_long, LP)
_sig("orc_run_schedule", C.c_int, LP, C.c_long, C.c_long, C.c_long, LP)
_sig("orc_tracker_create", C.c_int, C.c_long, PP)
_sig("orc_tracker_destroy", None, P)
_sig("orc_tracker_earliest_start", C.c_int, P, C.c_int, C.c_int, LP)
_sig("orc_tracker_add", C.c_int, P, C.c_long, C.c_int, C.c_int, IP)
_sig("orc_tracker_step", C.c_long, P, IP, IP, C.c_int, IP)
_sig("orc_tracker_recomputed_load", C.c_long, P, C.c_long)
_sig("orc_tracker_current", C.c_long, P)
_sig("orc_tracker_num_batches", C.c_int, P)
_sig("orc_tracker_batch", None, P, C.c_int, LP, LP)
_sig("orc_tracker_limit", C.c_long, P)
_sig("orc_drive_monolithic", C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_long, C.c_int, C.c_long,
     C.c_uint64, C.c_int, C.c_long, C.c_int, C.c_int, PP)
_sig("orc_drive_count", C.c_long, P)
_sig("orc_drive_record", None, P, C.c_long, LP, U64P, IP)
_sig("orc_drive_activations", FP, P)
_sig("orc_drive_destroy", None, P)
_sig("orc_bench_attend", C.c_int, C.POINTER(Spec), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
     C.POINTER(C.c_double))
_sig("orc_bench_dense", C.c_int, C.POINTER(Spec), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double))


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, _lib.orc_last_error().decode())


def _f(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(FP)


def _u64(a):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return a, a.ctypes.data_as(U64P)


def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ------------------------------------------------------------------ core ---
def make_spec(num_layers, model_dim, num_heads, mlp_dim, vocab_size, num_kv_heads=0) -> Spec:
    s = Spec()
    _check(_lib.orc_make_spec(num_layers, model_dim, num_heads, mlp_dim, vocab_size,
                              num_kv_heads, C.byref(s)))
    return s


def mix64(x: int) -> int:
    return int(_lib.orc_mix64(x & (2**64 - 1)))


def prompt_token(seed: int, seq: int, vocab: int) -> int:
    return int(_lib.orc_prompt_token(seed, seq, vocab))


def float_to_half_bits(x: float) -> int:
    return int(_lib.orc_f2h(x))


def half_bits_to_float(h: int) -> float:
    return float(_lib.orc_h2f(h))


def quantize_int8(x) -> tuple[np.ndarray, float]:
    x = f32(x)
    q = np.zeros(x.size, dtype=np.int8)
    s = _lib.orc_quantize_int8(_f(x), x.size, q.ctypes.data_as(C.POINTER(C.c_int8)))
    return q, float(np.float32(s))


def quantize_int4(x) -> tuple[np.ndarray, float]:
    """The 4-bit extension codec (sd_oracle.cpp quantize_int4): packed bytes, scale."""
    x = f32(x)
    q = np.zeros((x.size + 1) // 2, dtype=np.uint8)
    s = _lib.orc_quantize_int4(_f(x), x.size, q.ctypes.data_as(C.POINTER(C.c_uint8)))
    return q, float(np.float32(s))


def unpack_int4(packed, n) -> np.ndarray:
    """Packed nibbles (element 2i low) -> signed integers."""
    b = np.asarray(packed, dtype=np.uint8)
    nib = np.stack([b & 0xF, b >> 4], axis=-1).reshape(*b.shape[:-1], -1)[..., :n].astype(np.int8)
    return np.where(nib >= 8, nib - 16, nib).astype(np.int8)


def eigen_dot(a, b) -> float:
    a, b = f32(a), f32(b)
    return float(_lib.orc_eigen_dot(_f(a), _f(b), a.size))


def synth_value(idx: int) -> float:
    return float(_lib.orc_synth_value(idx))


def prefill_index(seq, layer, pos, kv, h, d, kv_heads, hd) -> int:
    """Element index of the sequence-keyed synthetic prefill."""
    return int(_lib.orc_kv_prefill_index(seq, layer, pos, kv, h, d, kv_heads, hd))


class Weights:
    """seed_random_weights (core.cpp:97-127)."""

    NAMES = {"embedding": 0, "w_q": 1, "w_k": 2, "w_v": 3, "w_o": 4, "w_mlp_in": 5,
             "w_mlp_out": 6, "head": 7}

    def __init__(self, spec: Spec, seed: int):
        self.spec = spec
        self.h = C.c_void_p()
        _check(_lib.orc_weights_create(C.byref(spec), seed, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            _lib.orc_weights_destroy(self.h)
            self.h = None

    def checksum(self) -> int:
        return int(_lib.orc_weights_checksum(self.h))

    def tensor(self, name: str, layer: int = 0) -> np.ndarray:
        """Column-major (out x in) reference storage, returned as the Eigen
        matrix view (rows=out, cols=in); shares memory with the oracle."""
        r, c = C.c_int(), C.c_int()
        p = _lib.orc_weights_tensor(self.h, layer, self.NAMES[name], C.byref(r), C.byref(c))
        flat = np.ctypeslib.as_array(p, shape=(r.value * c.value,))
        return flat.reshape(c.value, r.value).T  # (rows, cols) view of column-major data

    def raw(self, name: str, layer: int = 0) -> np.ndarray:
        """Flat column-major buffer exactly as the reference stores it."""
        r, c = C.c_int(), C.c_int()
        p = _lib.orc_weights_tensor(self.h, layer, self.NAMES[name], C.byref(r), C.byref(c))
        return np.ctypeslib.as_array(p, shape=(r.value * c.value,))


class KvShard:
    """KvShard (attention.hpp:68-140)."""

    def __init__(self, spec: Spec, head_start: int, head_count: int, capacity_tokens: int,
                 fmt: str = "single"):
        self.spec = spec
        self.head_count = head_count
        self.width = head_count * spec.head_dim
        self.q_width = self.width * (spec.num_heads // spec.num_kv_heads)
        self.h = C.c_void_p()
        _check(_lib.orc_kv_create(C.byref(spec), head_start, head_count, capacity_tokens,
                                  FORMATS[fmt], C.byref(self.h)))
        self.fmt = fmt

    def __del__(self):
        if getattr(self, "h", None):
            _lib.orc_kv_destroy(self.h)
            self.h = None

    def append(self, seq, layer, position, k, v):
        k, v = f32(k), f32(v)
        _check(_lib.orc_kv_append(self.h, seq, layer, position, _f(k), _f(v)))

    def append_request(self, layer, seqs, positions, k, v):
        seqs_a, sp = _u64(seqs)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        k, v = f32(k), f32(v)
        _check(_lib.orc_kv_append_request(self.h, layer, len(seqs_a), sp,
                                          pos.ctypes.data_as(U32P), _f(k), _f(v)))

    def prefill_synthetic(self, seqs, length: int, salt: int = 0):
        """Synthetic context (sequence-keyed) appended position by
        position in every layer: the bench / GPU prefill restated."""
        seqs_a, sp = _u64(seqs)
        _check(_lib.orc_kv_prefill_synthetic(self.h, len(seqs_a), sp, length, salt))

    def attend(self, layer, seqs, q) -> np.ndarray:
        seqs_a, sp = _u64(seqs)
        q = f32(q)
        o = np.zeros((len(seqs_a), self.q_width), dtype=np.float32)
        _check(_lib.orc_kv_attend(self.h, layer, len(seqs_a), sp, _f(q), _f(o)))
        return o

    def drop_sequence(self, seq):
        _lib.orc_kv_drop(self.h, seq)

    def stored_length(self, seq, layer) -> int:
        return int(_lib.orc_kv_stored_length(self.h, seq, layer))

    def token_count(self) -> int:
        return int(_lib.orc_kv_token_count(self.h))

    def warning_count(self) -> int:
        return int(_lib.orc_kv_warning_count(self.h))

    def has_sequence(self, seq) -> bool:
        return bool(_lib.orc_kv_has_sequence(self.h, seq))

    def bytes_per_token(self) -> int:
        return int(_lib.orc_kv_bytes_per_token(self.h))

    def export_lane(self, seq, layer, which):
        """(storage bytes, int8 scales or None) for lane K (0) or V (1)."""
        n = _lib.orc_kv_export_lane(self.h, seq, layer, which, None, 0, None, 0)
        if n < 0:
            _check(int(-n))
        buf = np.zeros(n, dtype=np.uint8)
        L = self.stored_length(seq, layer)
        scales = np.zeros(L * self.head_count, dtype=np.float32) if self.fmt in ("int8", "int4") else None
        _lib.orc_kv_export_lane(self.h, seq, layer, which, buf.ctypes.data_as(C.c_void_p), n,
                                _f(scales) if scales is not None else None,
                                scales.size if scales is not None else 0)
        return buf, scales


# ----------------------------------------------------------------- dense ---
def apply_linear(x, w_colmajor_flat, out_dim, threads=1) -> np.ndarray:
    x = f32(x)
    B, n_in = x.shape
    w = f32(w_colmajor_flat)
    y = np.zeros((B, out_dim), dtype=np.float32)
    _check(_lib.orc_apply_linear(B, n_in, out_dim, _f(x), _f(w), _f(y), threads))
    return y


def project_qkv(W: Weights, layer, seqs, x, threads=1):
    s = W.spec
    x = f32(x)
    B = x.shape[0]
    kvw = s.num_kv_heads * s.head_dim
    q = np.zeros((B, s.model_dim), np.float32)
    k = np.zeros((B, kvw), np.float32)
    v = np.zeros((B, kvw), np.float32)
    _, sp = _u64(seqs)
    seqs_a, sp = _u64(seqs)
    _check(_lib.orc_project_qkv(W.h, layer, B, sp, _f(x), _f(q), _f(k), _f(v), threads))
    return q, k, v


def finish_block(W: Weights, layer, o, residual, threads=1):
    o, r = f32(o), f32(residual)
    out = np.zeros_like(r)
    _check(_lib.orc_finish_block(W.h, layer, o.shape[0], _f(o), _f(r), _f(out), threads))
    return out


def output_logits(W: Weights, x, threads=1):
    x = f32(x)
    lg = np.zeros((x.shape[0], W.spec.vocab_size), np.float32)
    _check(_lib.orc_output_logits(W.h, x.shape[0], _f(x), _f(lg), threads))
    return lg


def argmax_token(logits) -> int:
    lg = f32(logits)
    return int(_lib.orc_argmax(_f(lg), lg.size))


def decode_step_monolithic(W: Weights, kv: KvShard, seqs, x, threads=1):
    """decode_step_monolithic (dense.cpp:90-129) -> (tokens, final_x, logits)."""
    x = f32(x)
    B = x.shape[0]
    seqs_a, sp = _u64(seqs)
    toks = np.zeros(B, np.int32)
    fx = np.zeros_like(x)
    lg = np.zeros((B, W.spec.vocab_size), np.float32)
    _check(_lib.orc_decode_step(W.h, kv.h, B, sp, _f(x), toks.ctypes.data_as(IP), _f(fx), _f(lg),
                                threads))
    return toks, fx, lg


# -------------------------------------------------------------- ShardMap ---
SHARD_MODES = {"by-sequence": 0, "by-head": 1, "hybrid": 2}


def shardmap_worker_for(mode, heads, workers, seq, head) -> int:
    out = C.c_int()
    _check(_lib.orc_shardmap_worker_for(SHARD_MODES[mode], heads, workers, seq, head, C.byref(out)))
    return out.value


def shardmap_head_range(mode, heads, workers, w):
    a, b = C.c_int(), C.c_int()
    _check(_lib.orc_shardmap_head_range(SHARD_MODES[mode], heads, workers, w, C.byref(a), C.byref(b)))
    return a.value, b.value


# ------------------------------------------------------------- scheduler ---
def micro_batch_size(batch, interval, target_len) -> int:
    out = C.c_int()
    _check(_lib.orc_micro_batch_size(batch, interval, target_len, C.byref(out)))
    return out.value


def cold_start_schedule(batch, target_len, interval, mode="fixed-interval", horizon=0):
    m = {"fixed-interval": 0, "ramped-limit": 1}[mode]
    n = C.c_long()
    cap = horizon + 2
    buf = np.zeros(3 * cap, dtype=np.int64)
    _check(_lib.orc_cold_start_schedule(batch, target_len, interval, m, horizon,
                                        buf.ctypes.data_as(LP), cap, C.byref(n)))
    return [tuple(int(v) for v in buf[3 * i:3 * i + 3]) for i in range(n.value)]


def run_schedule(admissions, load_limit, horizon):
    a = np.asarray(admissions, dtype=np.int64).reshape(-1)
    out = np.zeros(4 * max(horizon, 1), dtype=np.int64)
    _check(_lib.orc_run_schedule(a.ctypes.data_as(LP), len(admissions), load_limit, horizon,
                                 out.ctypes.data_as(LP)))
    return out.reshape(-1, 4)[:horizon]  # (step, n_active, total_load, n_ending)


class LoadTracker:
    """LoadTracker (scheduler.hpp:58-97)."""

    def __init__(self, limit):
        self.h = C.c_void_p()
        _check(_lib.orc_tracker_create(limit, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            _lib.orc_tracker_destroy(self.h)
            self.h = None

    def earliest_start(self, m, s):
        out = C.c_long()
        _check(_lib.orc_tracker_earliest_start(self.h, m, s, C.byref(out)))
        return out.value

    def add_micro_batch(self, start, m, s):
        out = C.c_int()
        _check(_lib.orc_tracker_add(self.h, start, m, s, C.byref(out)))
        return out.value

    def step(self):
        na, ne = C.c_int(), C.c_int()
        ending = (C.c_int * 256)()
        load = _lib.orc_tracker_step(self.h, C.byref(na), ending, 256, C.byref(ne))
        return {"n_active": na.value, "total_load": int(load), "ending": list(ending[:ne.value])}

    def recomputed_load(self, step):
        return int(_lib.orc_tracker_recomputed_load(self.h, step))

    def current_step(self):
        return int(_lib.orc_tracker_current(self.h))

    def load_limit(self):
        return int(_lib.orc_tracker_limit(self.h))

    def batches(self):
        out = []
        for i in range(_lib.orc_tracker_num_batches(self.h)):
            e, w = C.c_long(), C.c_long()
            _lib.orc_tracker_batch(self.h, i, C.byref(e), C.byref(w))
            out.append((e.value, w.value))
        return out


# ---------------------------------------------------------------- drive ----
def run_monolithic(W: Weights, batch, target_len, interval, steps, seed=0, capacity=1 << 16,
                   fmt="single", cold_start="fixed-interval", load_limit=0, record=False,
                   threads=1):
    """run_monolithic (workers.cpp:697-701) -> (transcript [(step, seq, tok)], activations)."""
    h = C.c_void_p()
    _check(_lib.orc_drive_monolithic(W.h, batch, target_len, interval, steps,
                                     {"fixed-interval": 0, "ramped-limit": 1}[cold_start],
                                     load_limit, seed, int(record), capacity, FORMATS[fmt],
                                     threads, C.byref(h)))
    try:
        n = _lib.orc_drive_count(h)
        recs = []
        st, sq, tk = C.c_long(), C.c_uint64(), C.c_int()
        for i in range(n):
            _lib.orc_drive_record(h, i, C.byref(st), C.byref(sq), C.byref(tk))
            recs.append((st.value, sq.value, tk.value))
        acts = None
        if record:
            p = _lib.orc_drive_activations(h)
            acts = np.ctypeslib.as_array(p, shape=(n * W.spec.model_dim,)).reshape(n, -1).copy()
        return recs, acts
    finally:
        _lib.orc_drive_destroy(h)


def transcript_csv(recs) -> str:
    """transcript_csv (workers.cpp:746-755)."""
    return "step,seq_id,token_id\n" + "".join(f"{s},{q},{t}\n" for s, q, t in recs)


# -------------------------------------------------------------- baselines ---
def bench_attend(spec: Spec, batch, seq_len, fmt="half", threads=1, reps=3) -> float:
    out = C.c_double()
    _check(_lib.orc_bench_attend(C.byref(spec), batch, seq_len, FORMATS[fmt], threads, reps,
                                 C.byref(out)))
    return out.value


def bench_dense(spec: Spec, batch, threads=1, reps=3) -> float:
    out = C.c_double()
    _check(_lib.orc_bench_dense(C.byref(spec), batch, threads, reps, C.byref(out)))
    return out.value
