"""CPU-side checks of the C-ABI library: it loads, exports every function
include/sd_abi.h declares, and its host-only logic (spec validation,
ShardMap, scheduler) matches the oracle. No kernels are launched."""
import collections
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sd_abi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2403_11421_b200 as sd
    names = _declared()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(sd.lib, n)]
    assert not missing, missing
    assert sd.lib.sd_abi_version() == 1


def test_every_tuning_switch_is_known_and_documented():
    """sd_tune accepts each switch the Python mirror restores (api._TUNED)
    and sd_abi.h documents it; an unknown name is a ConfigError."""
    import paper_2403_11421_b200 as sd
    from paper_2403_11421_b200 import api
    doc = open(os.path.join(ROOT, "include", "sd_abi.h")).read()
    for name, default in api._TUNED.items():
        sd.tune(name, default)
        assert f'"{name}"' in doc, name
    with pytest.raises(sd.ConfigError):
        sd.tune("no_such_switch", 1)


def test_spec_and_errors_match_reference():
    import paper_2403_11421_b200 as sd
    s = sd.make_model_spec(2, 64, 4, 256, 128)
    assert (s.head_dim, s.num_kv_heads) == (16, 4)
    assert sd.make_model_spec(32, 4096, 32, 11008, 32000).head_dim == 128
    with pytest.raises(sd.ConfigError, match="not divisible"):
        sd.make_model_spec(2, 63, 4, 256, 128)
    with pytest.raises(sd.ConfigError):
        sd.make_model_spec(0, 64, 4, 256, 128)


def test_kv_format_validation_before_any_device_work():
    """Storage formats: unknown ones and int4 over an odd head_dim are
    config errors, raised before the store touches a device."""
    import paper_2403_11421_b200 as sd
    odd = sd.make_model_spec(1, 12, 4, 8, 8)  # head_dim 3
    with pytest.raises(sd.ConfigError, match="even head_dim"):
        sd.KvShard(odd, 0, 4, 8, "int4")
    with pytest.raises(KeyError):
        sd.KvShard(odd, 0, 4, 8, "int2")


def test_mix64_prompt_tokens_match_oracle(oracle):
    import paper_2403_11421_b200 as sd
    for x in [0, 1, 42, 2**63 + 5, 2**64 - 1]:
        assert sd.mix64(x) == oracle.mix64(x)
    for seq in range(1, 300):
        assert sd.prompt_token(7, seq, 32000) == oracle.prompt_token(7, seq, 32000)


def test_shardmap_bit_exact_vs_oracle(oracle):
    import paper_2403_11421_b200 as sd
    for mode in ("by-sequence", "by-head", "hybrid"):
        for heads, workers in ((8, 1), (8, 2), (8, 4), (7, 3), (32, 8), (40, 8)):
            if mode == "by-head" and workers > heads:
                continue
            m = sd.ShardMap(mode, heads, workers)
            for w in range(workers):
                assert m.head_range(w) == oracle.shardmap_head_range(mode, heads, workers, w)
            for seq in range(1, 200):
                for h in (0, heads // 2, heads - 1):
                    assert m.worker_for(seq, h) == oracle.shardmap_worker_for(mode, heads, workers, seq, h)
    # proj/tests/test_transport.cpp:360-371
    c = collections.Counter(sd.ShardMap("by-sequence", 8, 4).worker_for(q, 0) for q in range(1, 1001))
    assert all(230 <= c[i] <= 270 for i in range(4))
    with pytest.raises(sd.ConfigError):
        sd.ShardMap("by-head", 2, 4)


def test_scheduler_matches_oracle(oracle):
    import paper_2403_11421_b200 as sd
    for b, s, f in ((6, 6, 2), (7, 10, 3), (32, 128, 4), (8, 32, 8), (1024, 1024, 16)):
        assert sd.micro_batch_size(b, f, s) == oracle.micro_batch_size(b, f, s)
        for mode in ("fixed-interval", "ramped-limit"):
            assert sd.cold_start_schedule(b, s, f, mode, 3 * s) == \
                oracle.cold_start_schedule(b, s, f, mode, 3 * s)
    with pytest.raises(sd.AdmissionError, match="interval too short"):
        sd.micro_batch_size(4, 2, 16)
