"""SDWP (the reference's S<->R wire protocol, transport.cpp:105-301) and the
B200 attention worker that speaks it (AttentionWorkerSession,
workers.cpp:40-214).

The oracle's restated codec (oracle/sdwp.py) is pinned to the reference's
byte-level tests (test_transport.cpp:58-124); the product's worker session is
then driven with frames the oracle encodes: host-only message handling on
CPU, and on the GPU the QKV_BATCH -> O_BATCH path against the oracle's
KvShard (identical tokens of work, attention outputs <= 1e-5), typed errors,
DROP_SEQ, half-precision wire, and the TCP service loop."""
import os
import struct
import threading

import numpy as np
import pytest


@pytest.fixture(scope="module")
def w():
    import sdwp
    return sdwp


# ----------------------------------------------------- oracle codec pinned
def test_frame_header_layout(w):
    # test_transport.cpp:58-73
    b = w.encode_frame(w.HELLO, bytes([0xAA, 0xBB]))
    assert b == b"SDWP" + bytes([1, 1, 2, 0, 0, 0, 0xAA, 0xBB])


def test_golden_qkv_record(w):
    # test_transport.cpp:75-124: head_dim 2, one head
    got = w.encode_qkv(3, 7, 1, 1, [0x0102030405060708], [9], [[1.0, -2.0]], [[0.5, 4.0]], [[-0.25, 8.0]])
    want = bytes([3, 0, 7, 0, 0, 0, 1, 0, 0, 0, 1, 0, 1, 0, 8, 7, 6, 5, 4, 3, 2, 1, 9, 0, 0, 0])
    want += struct.pack("<6f", 1.0, -2.0, 0.5, 4.0, -0.25, 8.0)
    assert got == want and len(want) == 14 + 12 + 3 * 2 * 4


def test_decoder_split_and_fatal(w):
    # test_transport.cpp:203-255
    stream = w.encode_frame(w.HELLO) + w.encode_frame(w.DROP_SEQ, w.encode_drop([1, 2, 3]))
    for chunk in (1, 3, 7, len(stream)):
        d = w.FrameDecoder()
        out = []
        for i in range(0, len(stream), chunk):
            d.feed(stream[i:i + chunk])
            while True:
                st, f = d.poll()
                if st != "frame":
                    break
                out.append(f)
        assert [f[1] for f in out] == [w.HELLO, w.DROP_SEQ]
    bad = b"X" + w.encode_frame(w.HELLO)[1:]
    d = w.FrameDecoder()
    d.feed(bad)
    assert d.poll()[0] == "fatal" and d.error == "bad magic"


# ------------------------------------------- product session, host-only
@pytest.fixture()
def rw():
    import paper_2403_11421_b200 as sd
    h = sd.RWorker(1 << 12, "single", 0)
    yield h
    h.close()


def test_worker_hello_errors_and_split_feeding(w, rw):
    """HELLO is echoed; a bad version, an unknown type and O_BATCH at the
    worker are ERROR replies (the connection survives); QKV before CONFIG is
    malformed; bytes may arrive split anywhere (workers.cpp:40-160)."""
    out = b""
    stream = (w.encode_frame(w.HELLO) + w.encode_frame(w.HELLO, version=9) + w.encode_frame(200)
              + w.encode_frame(w.O_BATCH) + w.encode_frame(w.QKV_BATCH, w.encode_qkv(0, 0, 0, 1, [], [], [], [], [])))
    for i in range(len(stream)):
        out += rw.feed(stream[i:i + 1])
    fr, st = w.frames(out)
    assert st == "more" and [f[1] for f in fr] == [w.HELLO, w.ERROR, w.ERROR, w.ERROR, w.ERROR]
    codes = [w.decode_error(f[2]) for f in fr[1:]]
    assert codes[0][0] == w.ERR_BAD_VERSION and "version 9" in codes[0][1]
    assert codes[1] == (w.ERR_UNKNOWN_TYPE, "unknown message type 200")
    assert codes[2] == (w.ERR_UNKNOWN_TYPE, "unexpected O_BATCH at the worker")
    assert codes[3] == (w.ERR_MALFORMED, "QKV before CONFIG")
    # DROP before CONFIG: no reply; SHUTDOWN: stats JSON and the session ends
    assert rw.feed(w.encode_frame(w.DROP_SEQ, w.encode_drop([5]))) == b""
    fr, _ = w.frames(rw.feed(w.encode_frame(w.SHUTDOWN)))
    import json
    stats = json.loads(fr[0][2])
    assert fr[0][1] == w.SHUTDOWN and set(stats) == {"busy_seconds", "drop_warnings", "idle_seconds",
                                                      "tokens_processed"}
    assert rw.shutdown_requested()


def test_worker_bad_magic_is_fatal(w, rw):
    import paper_2403_11421_b200 as sd
    with pytest.raises(sd.ProtocolError, match="bad magic"):
        rw.feed(b"XDWP" + bytes(6))


def test_worker_bad_config_is_an_error_reply(w, rw):
    fr, _ = w.frames(rw.feed(w.encode_frame(w.CONFIG, b'{"model": 3}')))
    code, msg = w.decode_error(fr[0][2])
    assert code == w.ERR_MALFORMED and msg.startswith("bad config")


# ------------------------------------------------------------- GPU path
def _session(w, sd, fmt, precision, spec=(2, 64, 4, 256, 128), h0=0, hc=4, cap=1 << 12):
    rw = sd.RWorker(cap, fmt, 0)
    fr, _ = w.frames(rw.feed(w.encode_frame(w.CONFIG, w.config_payload(*spec, h0, hc, precision))))
    assert fr[0][1] == w.CONFIG, w.decode_error(fr[0][2])
    return rw, fr[0][2]


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["single", "half", "int8", "int4"])
@pytest.mark.parametrize("precision", ["single", "half"])
def test_worker_qkv_batches_match_oracle_kvshard(w, oracle, fmt, precision):
    """Several steps x layers of QKV_BATCH frames (new sequences, growing
    positions, ragged membership) through the B200 worker: every O_BATCH row
    equals the oracle KvShard's attend on the same (wire-rounded) inputs
    within 1e-5, records in request order; the CONFIG ack is the
    reference's JSON (workers.cpp:63-84)."""
    import json
    import paper_2403_11421_b200 as sd
    rw, ack = _session(w, sd, fmt, precision)
    assert json.loads(ack) == {"capacity_tokens": 1 << 12, "ok": True, "storage_format": fmt, "width": 64}
    assert ack == json.dumps(json.loads(ack), separators=(",", ":"), sort_keys=True).encode()
    okv = oracle.KvShard(oracle.make_spec(2, 64, 4, 256, 128), 0, 4, 1 << 12, fmt)
    rng = np.random.default_rng(5)
    pos = {}
    worst = 0.0
    for step in range(6):
        seqs = [s for s in range(1, 9) if s <= 3 + step and (s + step) % 5]
        for layer in range(2):
            P = [pos.get((s, layer), 0) for s in seqs]
            q, k, v = (rng.uniform(-1, 1, (len(seqs), 64)).astype(np.float32) for _ in range(3))
            if precision == "half":  # the wire carries fp16: the worker sees the rounded values
                q, k, v = (x.astype(np.float16).astype(np.float32) for x in (q, k, v))
            frame = w.encode_frame(w.QKV_BATCH, w.encode_qkv(layer, step, 0, 4, seqs, P, q, k, v, precision))
            fr, _ = w.frames(rw.feed(frame))
            assert fr[0][1] == w.O_BATCH, w.decode_error(fr[0][2])
            ly, st, h0, hc, oseqs, o = w.decode_o(fr[0][2], 64, precision)
            assert (ly, st, h0, hc, oseqs) == (layer, step, 0, 4, seqs)
            okv.append_request(layer, seqs, P, k, v)
            ref = okv.attend(layer, seqs, q)
            if precision == "half":
                ref = ref.astype(np.float16).astype(np.float32)
                worst = max(worst, float(np.abs(o - ref).max() / 2.0**-10))  # one half ulp at |x| < 1
            else:
                worst = max(worst, float(np.abs(o - ref).max() / 1e-5))
            for s in seqs:
                pos[(s, layer)] = pos.get((s, layer), 0) + 1
        if step == 3:  # DROP_SEQ is fire-and-forget; the worker forgets the sequence
            assert rw.feed(w.encode_frame(w.DROP_SEQ, w.encode_drop([2, 99]))) == b""
            okv.drop_sequence(2)
            okv.drop_sequence(99)
            for layer in range(2):
                pos.pop((2, layer), None)
    assert worst <= 1.0
    rw.close()


@pytest.mark.gpu
def test_worker_typed_errors(w):
    """CapacityError -> code 4, a wrong first position -> UnknownSequence 5,
    a foreign head range -> malformed 3 (workers.cpp:133-140)."""
    import paper_2403_11421_b200 as sd
    rw, _ = _session(w, sd, "single", "single", cap=2)
    one = np.zeros((1, 64), np.float32)

    def send(layer, seqs, P, h0=0):
        fr, _ = w.frames(rw.feed(w.encode_frame(w.QKV_BATCH, w.encode_qkv(
            layer, 0, h0, 4, seqs, P, np.repeat(one, len(seqs), 0), np.repeat(one, len(seqs), 0),
            np.repeat(one, len(seqs), 0)))))
        return fr[0]

    assert send(0, [1], [3])[1] == w.ERROR and w.decode_error(send(0, [1], [3])[2])[0] == w.ERR_UNKNOWN_SEQ
    assert send(0, [1], [0])[1] == w.O_BATCH
    assert send(0, [2], [0])[1] == w.O_BATCH
    assert send(0, [2], [0], h0=1)[1] == w.ERROR
    r = send(0, [3], [0])  # 2-token capacity x 2 layers is full
    assert r[1] == w.ERROR and w.decode_error(r[2])[0] == w.ERR_CAPACITY


@pytest.mark.gpu
def test_worker_serves_over_tcp(w, oracle, tmp_path):
    """serve_attention_worker (workers.cpp:162-214) in this process: a socket
    client (the dense side) runs HELLO, CONFIG, QKV_BATCH, SHUTDOWN."""
    import socket
    import time
    import paper_2403_11421_b200 as sd
    port_file = str(tmp_path / "port")
    t = threading.Thread(target=sd.serve_rworker, args=("127.0.0.1:0", 1 << 12, "half", 0, port_file, True),
                         daemon=True)
    t.start()
    for _ in range(200):
        if os.path.exists(port_file) and open(port_file).read().strip():
            break
        time.sleep(0.05)
    port = int(open(port_file).read())
    c = socket.create_connection(("127.0.0.1", port), timeout=30)
    seqs, P = [11, 12, 13], [0, 0, 0]
    rng = np.random.default_rng(1)
    q, k, v = (rng.uniform(-1, 1, (3, 64)).astype(np.float32) for _ in range(3))
    c.sendall(w.encode_frame(w.HELLO) + w.encode_frame(w.CONFIG, w.config_payload(2, 64, 4, 256, 128, 0, 4))
              + w.encode_frame(w.QKV_BATCH, w.encode_qkv(0, 0, 0, 4, seqs, P, q, k, v)) + w.encode_frame(w.SHUTDOWN))
    data = b""
    while True:
        fr, _ = w.frames(data)
        if len(fr) == 4:
            break
        chunk = c.recv(1 << 16)
        assert chunk, "connection closed early"
        data += chunk
    c.close()
    t.join(timeout=30)
    assert [f[1] for f in fr] == [w.HELLO, w.CONFIG, w.O_BATCH, w.SHUTDOWN]
    okv = oracle.KvShard(oracle.make_spec(2, 64, 4, 256, 128), 0, 4, 1 << 12, "half")
    okv.append_request(0, seqs, P, k, v)
    _, _, _, _, oseqs, o = w.decode_o(fr[2][2], 64)
    assert oseqs == seqs and np.abs(o - okv.attend(0, seqs, q)).max() <= 2e-5


# ------------------------------------------ the `serve` drop-in binary
RWORKER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2403_11421_b200",
                       "sd_rworker")


def test_rworker_cli_rejects_bad_options():
    """The reference CLI's argument errors (splitdecode_main.cpp serve:
    --capacity required, --storage single|half|int8): exit 2, no socket."""
    import subprocess
    assert os.access(RWORKER, os.X_OK), "sd_rworker not built (make -C paper_2403_11421_b200/csrc)"
    for args, msg in ((["serve"], "usage"), (["serve", "--capacity", "16", "--storage", "fp8"], "unknown kv storage"),
                      (["serve", "--capacity"], "needs a value"), (["bogus"], "usage")):
        r = subprocess.run([RWORKER, *args], capture_output=True, text=True, timeout=60)
        assert r.returncode == 2 and msg in r.stderr, (args, r.stderr)


def _start_rworker(tmp_path, *extra):
    import subprocess
    import time
    port_file = str(tmp_path / "port")
    p = subprocess.Popen([RWORKER, "serve", "--listen", "127.0.0.1:0", "--port-file", port_file, "--once", *extra],
                         stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    for _ in range(1200):
        if os.path.exists(port_file) and open(port_file).read().strip():
            return p, int(open(port_file).read())
        if p.poll() is not None:
            break
        time.sleep(0.05)
    p.kill()
    raise AssertionError("sd_rworker did not come up: " + p.communicate()[1])


@pytest.mark.gpu
@pytest.mark.parametrize("storage", ["half", "int8", "int4"])
def test_rworker_binary_serves_a_session(w, oracle, tmp_path, storage):
    """`sd_rworker serve --once` as its own process: the dense side connects
    over TCP, runs HELLO / CONFIG / two steps of QKV_BATCH / SHUTDOWN, gets
    the oracle KvShard's outputs back, and the worker exits 0."""
    import json
    import socket
    p, port = _start_rworker(tmp_path, "--capacity", "4096", "--storage", storage)
    try:
        c = socket.create_connection(("127.0.0.1", port), timeout=60)
        okv = oracle.KvShard(oracle.make_spec(2, 64, 4, 256, 128), 0, 4, 4096, storage)
        rng = np.random.default_rng(3)
        seqs = [21, 22, 23, 24]
        c.sendall(w.encode_frame(w.HELLO) + w.encode_frame(w.CONFIG, w.config_payload(2, 64, 4, 256, 128, 0, 4)))
        sent, want = [], []
        for step in range(2):
            for layer in range(2):
                q, k, v = (rng.uniform(-1, 1, (4, 64)).astype(np.float32) for _ in range(3))
                sent.append(w.encode_frame(w.QKV_BATCH, w.encode_qkv(layer, step, 0, 4, seqs, [step] * 4, q, k, v)))
                okv.append_request(layer, seqs, [step] * 4, k, v)
                want.append(okv.attend(layer, seqs, q))
        c.sendall(b"".join(sent) + w.encode_frame(w.SHUTDOWN))
        data = b""
        while True:
            fr, _ = w.frames(data)
            if len(fr) == 7:
                break
            chunk = c.recv(1 << 16)
            assert chunk, "connection closed early"
            data += chunk
        c.close()
        assert p.wait(timeout=60) == 0, p.communicate()[1]
    finally:
        if p.poll() is None:
            p.kill()
    assert [f[1] for f in fr] == [w.HELLO, w.CONFIG] + [w.O_BATCH] * 4 + [w.SHUTDOWN]
    assert json.loads(fr[1][2])["storage_format"] == storage
    for f, ref in zip(fr[2:6], want):
        assert np.abs(w.decode_o(f[2], 64)[5] - ref).max() <= 2e-5
    assert json.loads(fr[6][2])["tokens_processed"] == 4 * 2 * 2


@pytest.mark.gpu
def test_rworker_binary_receive_timeout(w, tmp_path):
    """--timeout (ServeOptions::recv_timeout_seconds): an idle connection
    ends its session; with --once the worker then exits 0."""
    import socket
    import time
    p, port = _start_rworker(tmp_path, "--capacity", "64", "--timeout", "1")
    try:
        c = socket.create_connection(("127.0.0.1", port), timeout=60)
        c.sendall(w.encode_frame(w.HELLO))
        t0 = time.time()
        assert p.wait(timeout=60) == 0
        assert time.time() - t0 < 30 and "timed out" in p.communicate()[1]
        c.close()
    finally:
        if p.poll() is None:
            p.kill()
