"""The planner's measured inputs on the GPU (sd_bench_dense_block,
sd_bench_attention_per_token, sd_kv_capacity_tokens) feeding the planner."""
import pytest

import paper_2403_11421_b200 as sd
from paper_2403_11421_b200 import planner as pl

pytestmark = pytest.mark.gpu


def test_measured_profile_plans():
    spec = sd.make_model_spec(1, 512, 4, 1024, 1024, 2)
    w = sd.DeviceWeights(spec, None, "bf16", 0, seed=0)
    table = pl.bench_dense_block(w, [1, 16, 128, 512], reps=3)
    w.close()
    assert [b for b, _ in table] == [1, 16, 128, 512]
    assert all(t > 0 for _, t in table)
    # per-token cost falls with the batch (the reason for the paper's large B)
    assert table[-1][1] / 512 < table[0][1]
    r = pl.bench_attention_per_token(spec, "half", batch=64, seq_len=256, reps=3)
    assert 0 < r < 1e-3
    cap = pl.kv_capacity_tokens(sd.make_model_spec(32, 512, 4, 1024, 1024, 2), "half")
    assert cap > 1000
    prof = pl.PerfProfile(table, r, cap, "b200-test")
    res = pl.plan(prof, pl.PlanRequest(num_layers=32, target_len=1024))
    assert res.batch_size in (1, 16, 128, 512) and res.worker_count >= 1


def test_bench_errors():
    spec = sd.make_model_spec(1, 512, 4, 1024, 1024, 2)
    w = sd.DeviceWeights(spec, None, "bf16", 0, seed=0)
    with pytest.raises(sd.ConfigError):
        pl.bench_dense_block(w, [16, 1], reps=1)
    w.close()
    with pytest.raises(sd.ConfigError):
        pl.bench_attention_per_token(spec, "half", batch=0, seq_len=16, reps=1)
