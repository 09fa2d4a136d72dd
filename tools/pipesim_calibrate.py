"""Calibrate the reference's pipeline simulator against measured B200 steps.

pipesim (proj/src/pipesim.cpp:45-130) models a decode step as
  sequential:  s + r + tx
  pipelined:   max(s, r) + exposed * tx      (after the first busy step)
with s = num_layers * T(B) (block_seconds over the measured T(B) table,
planner.cpp:48-68), r = load * R / workers * skew (make_linear_model /
build_latency_model) and tx the exchange. This tool feeds it the B200
planner inputs (a perf profile written by tools/plan_b200.py: T(B) and R
measured with the reference's definitions) and compares its predictions with
decode steps measured by bench.py (JSON lines), per topology:

  python tools/pipesim_calibrate.py PROFILE.json MEASURED.json [out.json]

MEASURED.json: {"cases": [{"name", "batch", "context", "layers", "workers",
"skew", "pipelined", "tx_ms", "measured_ms"}, ...]}.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11421_b200 import planner as pl  # noqa: E402


def simulate_step(T, R, batch, context, layers, workers, skew, pipelined, tx, exposed=0.5):
    """One steady decode step of pipesim's simulate() (pipesim.cpp:80-130)."""
    s = layers * T
    load = batch * (context + 1)  # positions attended per layer (the new one included)
    r = layers * load * R / workers * skew
    step = max(s, r) + exposed * tx if pipelined else s + r + tx
    return s, r, step


def main():
    prof_doc = json.load(open(sys.argv[1]))["profile"]
    cases = json.load(open(sys.argv[2]))["cases"]
    prof = pl.PerfProfile([(row["batch_size"], row["seconds_per_block"]) for row in prof_doc["t_table"]],
                          prof_doc["r_per_token"], prof_doc["capacity_c"], prof_doc.get("machine_tag", ""))
    rows = []
    for c in cases:
        T = pl.block_seconds(prof, c["batch"])
        s, r, step = simulate_step(T, prof.r_per_token, c["batch"], c["context"], c["layers"], c["workers"],
                                   c.get("skew", 1.0), c["pipelined"], c.get("tx_ms", 0.0) / 1e3)
        rows.append({**c, "model_s_ms": s * 1e3, "model_r_ms": r * 1e3, "model_step_ms": step * 1e3,
                     "measured_over_model": c["measured_ms"] / (step * 1e3)})
        print(f"{c['name']:46s} model s {s*1e3:7.2f} r {r*1e3:7.2f} step {step*1e3:7.2f} ms | "
              f"measured {c['measured_ms']:7.2f} ms  ({c['measured_ms'] / (step * 1e3):.2f}x)")
    if len(sys.argv) > 3:
        json.dump({"profile": sys.argv[1], "model": "pipesim.cpp:80-130 with B200 T(B), R", "rows": rows},
                  open(sys.argv[3], "w"), indent=1)


if __name__ == "__main__":
    main()
