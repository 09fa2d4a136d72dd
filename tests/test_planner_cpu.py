"""The planner (Eq. 7-11) behind the C ABI against the reference's own planner
tests (proj/tests/test_planner.cpp): the same profiles, requests and known
answers. Host only."""
import json
import math
import os

import pytest

import paper_2403_11421_b200 as sd
from paper_2403_11421_b200 import planner as pl

HERE = os.path.dirname(os.path.abspath(__file__))


def simple_profile():  # test_planner.cpp:17-24
    return pl.PerfProfile([(1, 1e-3), (8, 1.5e-3), (64, 4e-3), (256, 10e-3), (512, 18e-3)], 1e-6, 1 << 20, "synthetic")


def test_block_seconds_interpolates_and_refuses_extrapolation():  # :28-36
    p = simple_profile()
    assert pl.block_seconds(p, 8) == pytest.approx(1.5e-3)
    assert pl.block_seconds(p, 36) == pytest.approx(2.75e-3)
    with pytest.raises(sd.ConfigError, match="below"):
        pl.block_seconds(p, 0)
    with pytest.raises(sd.ConfigError, match="extrapolation"):
        pl.block_seconds(p, 1024)


def test_efficiency_is_b_over_t():  # :38-43
    p = simple_profile()
    assert pl.batch_efficiency(p, 1) == pytest.approx(1000.0)
    p = pl.PerfProfile([(1, 1e-3), (1024, 1024 / 144632.768)], 1e-6, 1 << 20)
    assert pl.batch_efficiency(p, 1024) == pytest.approx(144632.768, rel=1e-4)


@pytest.mark.parametrize("table,r,c", [
    ([], 1e-6, 1),
    ([(8, 1e-3), (8, 2e-3)], 1e-6, 1),
    ([(1, 1e-3), (8, -1.0)], 1e-6, 1),
    ([(1, 1e-3)], 0.0, 1),
    ([(1, 1e-3)], 1e-6, 0),
])
def test_profile_validation(table, r, c):  # :45-55
    with pytest.raises(sd.ConfigError):
        pl.plan(pl.PerfProfile(table, r, c), pl.PlanRequest(1, 1))


def test_profile_json_round_trip():  # :57-65 (the reference's JSON shape)
    p = simple_profile()
    assert pl.PerfProfile.from_json(json.loads(json.dumps(p.to_json()))) == p


def test_latency_budget_picks_largest_feasible_batch():  # :67-88
    p = pl.PerfProfile([(64, 3e-3), (256, 5e-3), (512, 7e-3)], 1e-6, 1 << 20)
    assert pl.plan_batch_size(p, pl.PlanRequest(32, 1024, latency_budget=400.0)) == 256
    assert pl.plan_batch_size(p, pl.PlanRequest(32, 1024, latency_budget=1e9)) == 512
    with pytest.raises(sd.InfeasiblePlanError) as e:
        pl.plan_batch_size(p, pl.PlanRequest(32, 1024, latency_budget=1.0))
    assert e.value.tightest_batch == 64
    with pytest.raises(sd.ConfigError):
        pl.plan_batch_size(p, pl.PlanRequest(32, 1024, latency_budget=0.0))


def test_knee_rule():  # :90-102
    p = pl.PerfProfile([(1, 1e-3), (8, 2e-3), (64, 8e-3), (128, 128.0 / 8400.0)], 1e-6, 1 << 20)
    assert pl.plan_batch_size(p, pl.PlanRequest(1, 1)) == 64
    p = pl.PerfProfile([(1, 1e-3), (8, 2e-3), (64, 8e-3)], 1e-6, 1 << 20)
    assert pl.plan_batch_size(p, pl.PlanRequest(1, 1)) == 64


def test_worker_count_is_ceiling():  # :104-114
    p = pl.PerfProfile([(100, 5e-3)], 1e-5, 1 << 20)
    w, est = pl.plan_worker_count(p, 100, 100)
    assert est == pytest.approx(10.0) and w == 10
    p = pl.PerfProfile([(100, 5e-3)], 1e-12, 1 << 20)
    assert pl.plan_worker_count(p, 100, 100)[0] == 1


def test_memory_check():  # :116-123
    assert pl.check_memory(1024, 1024, 1 << 20, 1)[0]
    assert pl.check_memory(1024, 1024, 524288, 1)[0]
    ok, minw = pl.check_memory(1024, 1024, 1000, 1)
    assert not ok and minw == 525


def test_plan_composes_constraints():  # :125-153
    p = simple_profile()
    r = pl.plan(p, pl.PlanRequest(2, 64))
    assert r.binding_constraint == "efficiency-knee" and r.worker_count >= 1
    assert r.predicted_seq_seconds == pytest.approx(2.0 * 2 * 64 * pl.block_seconds(p, r.batch_size))
    p.capacity_c = 64
    r = pl.plan(p, pl.PlanRequest(2, 64))
    assert r.binding_constraint == "memory"
    assert r.batch_size * 64 / 2.0 <= p.capacity_c * r.worker_count
    p = simple_profile()
    r = pl.plan(p, pl.PlanRequest(2, 64, latency_budget=2.0 * 2 * 64 * 4e-3 + 1e-9))
    assert r.binding_constraint == "latency" and r.batch_size == 64


def test_reference_two_worker_operating_point():  # :155-180
    measured, workers = 8.12e-3, 2
    p = pl.PerfProfile([(1024, 7.08e-3)], measured * workers / (1024.0 * 1024.0 / 2.0), 1 << 20, "reference")
    stage, res, ok = pl.check_balance(p, 1024, 1024, 2)
    assert stage == pytest.approx(8.12e-3, rel=1e-9)
    assert res == pytest.approx((8.12 - 7.08) / 7.08, rel=1e-6)
    assert ok
    r = pl.plan(p, pl.PlanRequest(32, 1024))
    assert r.worker_count == 3
    assert r.worker_estimate == pytest.approx(8.12 * 2 / 7.08, rel=1e-6)


def _units(seed):
    state = seed
    while True:
        state = sd.mix64(state)
        yield state, (state >> 11) * 2.0 ** -53


def test_brute_force_maximal_batch_minimal_workers():  # :182-229
    it = _units(77)
    for _ in range(200):
        t = 0.5e-3 + next(it)[1] * 1e-3
        table = []
        for b in (1, 2, 4, 8, 16, 32, 64):
            table.append((b, t))
            t *= 1.2 + next(it)[1]
        r = 1e-7 + next(it)[1] * 1e-5
        p = pl.PerfProfile(table, r, 1 << 24)
        state, _ = next(it)  # the reference reads `state` after the last draw
        # (re-derive layers/len from the state after the r draw, as the reference does)
        layers = 1 + state % 8
        tlen = 16 + state % 512
        p_state, u = next(it)
        budget = 2.0 * layers * tlen * pl.block_seconds(p, 8) * (0.5 + u * 4.0)
        req = pl.PlanRequest(int(layers), int(tlen), latency_budget=budget)
        expected = max([b for b, tb in table if 2.0 * layers * tlen * tb <= budget], default=-1)
        if expected < 0:
            with pytest.raises(sd.InfeasiblePlanError):
                pl.plan_batch_size(p, req)
            continue
        got = pl.plan_batch_size(p, req)
        assert got == expected
        w, _ = pl.plan_worker_count(p, got, int(tlen))
        tb = pl.block_seconds(p, got)
        minimal = 1
        while got * tlen * r / (2.0 * minimal) > tb:
            minimal += 1
        assert w == max(1, minimal)


def test_plans_satisfy_latency_and_memory():  # :231-268
    it = _units(404)
    planned = 0
    for _ in range(1000):
        t = 1e-4 + next(it)[1] * 1e-2
        table = []
        for b in (1, 4, 16, 64, 256):
            table.append((b, t))
            t *= 1.1 + 2.0 * next(it)[1]
        r = 1e-8 + next(it)[1] * 1e-4
        cap = 1 + int(next(it)[1] * (1 << 22))
        state, _ = next(it)
        layers = 1 + state % 48
        tlen = 1 + sd.mix64(state) % 2048
        budget = None
        if next(it)[1] < 0.7:
            budget = (0.05 + next(it)[1] * 4.0) * 2.0 * layers * tlen * table[-1][1]
        try:
            res = pl.plan(pl.PerfProfile(table, r, cap), pl.PlanRequest(int(layers), int(tlen), latency_budget=budget))
        except sd.InfeasiblePlanError:
            continue
        if budget:
            assert res.predicted_seq_seconds <= budget * (1 + 1e-12)
        assert res.batch_size * tlen / 2.0 <= cap * res.worker_count
        planned += 1
    assert planned > 400


def test_workers_monotone_in_target_length():  # :270-278
    p = simple_profile()
    last = 0
    s = 16
    while s <= 4096:
        w, _ = pl.plan_worker_count(p, 64, s)
        assert w >= last
        last = w
        s *= 2


def test_machine_local_fixture():  # :280-320, on the reference's fixture profile
    p = pl.PerfProfile.from_json(json.load(open(os.path.join(HERE, "golden", "perf_profile_local.json"))))
    assert p.machine_tag
    last = 0
    for b, _ in p.t_table:
        e = pl.batch_efficiency(p, b)
        assert e > last
        last = e
    batch = p.t_table[-1][0]
    t = pl.block_seconds(p, batch)
    target_len = max(1, int(math.floor(2.0 * 4 * t / (batch * p.r_per_token))))
    r = pl.plan(p, pl.PlanRequest(2, target_len, candidate_batches=[batch]))
    assert r.batch_size == batch and r.balance_residual <= 0.15 and r.balanced
