"""SDWP wire protocol restated in Python (TEST INFRASTRUCTURE ONLY).

The reference's frame and payload codecs (proj/src/transport.cpp:105-301,
proj/include/splitdecode/transport.hpp) as the client side of the tests
that drive the product's B200 attention worker (sd_rworker_*). Pinned to
the reference's own byte-level tests (tests/test_oracle_sdwp.py:
test_transport.cpp:58-124). Little-endian throughout:

    frame = b"SDWP" | version u8 | msg_type u8 | payload_len u32 | payload
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"SDWP"
VERSION = 1
HEADER = 10
MAX_PAYLOAD = 64 << 20
HELLO, CONFIG, QKV_BATCH, O_BATCH, DROP_SEQ, SHUTDOWN, ERROR = range(1, 8)
ERR_BAD_VERSION, ERR_UNKNOWN_TYPE, ERR_MALFORMED, ERR_CAPACITY, ERR_UNKNOWN_SEQ, ERR_INTERNAL = range(1, 7)


def encode_frame(msg_type: int, payload: bytes = b"", version: int = VERSION) -> bytes:
    """encode_frame (transport.cpp:105-117)."""
    if len(payload) > MAX_PAYLOAD:
        raise ValueError("payload exceeds the frame size limit")
    return MAGIC + struct.pack("<BBI", version, msg_type, len(payload)) + payload


class FrameDecoder:
    """FrameDecoder::feed / poll (transport.cpp:119-147): complete frames, then
    "more" or exactly one "fatal"."""

    def __init__(self):
        self.buf = b""
        self.fatal = False
        self.error = ""

    def feed(self, data: bytes):
        self.buf += data

    def poll(self):
        if self.fatal:
            return "fatal", None
        if len(self.buf) < HEADER:
            return "more", None
        if self.buf[:4] != MAGIC:
            self.fatal, self.error = True, "bad magic"
            return "fatal", None
        version, msg_type, n = struct.unpack("<BBI", self.buf[4:10])
        if n > MAX_PAYLOAD:
            self.fatal, self.error = True, f"frame length {n} exceeds the limit"
            return "fatal", None
        if len(self.buf) < HEADER + n:
            return "more", None
        payload = self.buf[HEADER:HEADER + n]
        self.buf = self.buf[HEADER + n:]
        return "frame", (version, msg_type, payload)


def frames(data: bytes):
    """All complete frames of a byte string, as (version, type, payload)."""
    d = FrameDecoder()
    d.feed(data)
    out = []
    while True:
        st, f = d.poll()
        if st != "frame":
            return out, st
        out.append(f)


def _vec(x, precision):
    x = np.ascontiguousarray(x, np.float32)
    return x.astype("<f4").tobytes() if precision == "single" else x.astype("<f2").tobytes()


def encode_qkv(layer, step, head_start, head_count, seqs, positions, q, k, v, precision="single") -> bytes:
    """encode_qkv_payload (transport.cpp:163-181): prefix layer u16 | step u32 |
    count u32 | head_start u16 | head_count u16, then seq u64 | position u32 |
    q | k | v per record (fp32, or IEEE half RNE under "half")."""
    out = [struct.pack("<HIIHH", layer, step, len(seqs), head_start, head_count)]
    for i, s in enumerate(seqs):
        out.append(struct.pack("<QI", int(s), int(positions[i])))
        out += [_vec(q[i], precision), _vec(k[i], precision), _vec(v[i], precision)]
    return b"".join(out)


def decode_o(payload: bytes, width: int, precision="single"):
    """decode_o_payload (transport.cpp:224-247) -> (layer, step, head_start,
    head_count, seqs, o [n][width])."""
    layer, step, count, h0, hc = struct.unpack("<HIIHH", payload[:14])
    es = 4 if precision == "single" else 2
    rec = 8 + width * es
    if len(payload) - 14 != count * rec:
        raise ValueError("o batch: payload size does not match count")
    seqs, rows = [], []
    for i in range(count):
        b = payload[14 + i * rec:14 + (i + 1) * rec]
        seqs.append(struct.unpack("<Q", b[:8])[0])
        rows.append(np.frombuffer(b[8:], "<f4" if es == 4 else "<f2").astype(np.float32))
    return layer, step, h0, hc, seqs, np.array(rows, np.float32).reshape(count, width)


def encode_drop(seqs) -> bytes:
    """encode_drop_payload (transport.cpp:249-255)."""
    return struct.pack("<I", len(seqs)) + b"".join(struct.pack("<Q", int(s)) for s in seqs)


def decode_error(payload: bytes):
    """decode_error_payload (transport.cpp:276-287) -> (code, message)."""
    code, n = struct.unpack("<HI", payload[:6])
    if len(payload) - 6 != n:
        raise ValueError("error payload truncated")
    return code, payload[6:].decode()


def config_payload(num_layers, model_dim, num_heads, mlp_dim, vocab_size, head_start, head_count,
                   wire_precision="single", num_kv_heads=None) -> bytes:
    """The CONFIG JSON DistributedComputation sends (workers.cpp:292-301)."""
    import json
    model = {"num_layers": num_layers, "model_dim": model_dim, "num_heads": num_heads,
             "head_dim": model_dim // num_heads, "mlp_dim": mlp_dim, "vocab_size": vocab_size}
    if num_kv_heads:
        model["num_kv_heads"] = num_kv_heads
    return json.dumps({"model": model, "head_start": head_start, "head_count": head_count,
                       "wire_precision": wire_precision}).encode()
