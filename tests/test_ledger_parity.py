"""The executor's logical memory ledger against the reference simulator's, bit for bit (no GPU).

SURVEY §8a row 12 / north star: "peak-memory accounting and tensor liveness must be bit-exact".
The executor books every forward-template tensor it physically produces or drops (and the
backward / embedding / head bytes by the same rules) on the plan clock; given the simulator's pass
start times for its stage (exec.ledger_pass_start_us, from lynx_plan_simulate_timelines) its
ledger trace and peak must equal simulate()'s memory_traces / memory_peaks entry exactly — times
and byte counts as exact rationals. Checked here in dry-run mode (the executor's full launch
program, no device) against:
  * the reference's own simulate() (oracle/_ref, unmodified sources) where it is built, and
  * this repo's native simulator (always),
over TP = 1 and TP-template plans (critical-path, window and stall-fill recompute), Megatron full
and selective baselines and multi-stage pipelines. The same check runs on the B200 in
tests/test_executor_gpu.py (real step).
"""
import json

import pytest

from paper_2406_08756_b200 import executor as ex
from paper_2406_08756_b200 import gpt_profile as gp
from paper_2406_08756_b200 import planner


def tiny(**kw):
    base = dict(name="gpt-tiny", n_layers=4, hidden=512, heads=8, seq=256, micro_batch=2, vocab=50304, tp=1, pp=1,
                n_microbatches=2, dropout=0.1)
    base.update(kw)
    return gp.GPTConfig(**base)


def static_bytes(c):
    return gp.BYTES_PER_PARAM_STATIC * c.params() // c.tp


CASES = {
    "tp1_full": (tiny(), "full"),
    "tp1_heu_tight": (tiny(mem_budget_bytes=static_bytes(tiny()) + 24 * 2**20), "heu"),
    "tp1_selective": (tiny(), "selective"),
    "tp_template_window": (tiny(tp_template=True, mem_budget_bytes=static_bytes(tiny()) + 22 * 2**20), "heu"),
    "tp2_heu": (tiny(tp=2, mem_budget_bytes=static_bytes(tiny(tp=2)) + 8 * 2**20), "heu"),
    "tp2pp2_heu": (tiny(tp=2, pp=2, n_microbatches=4, mem_budget_bytes=static_bytes(tiny(tp=2)) // 2 + 4 * 2**20),
                   "heu"),
    "pp4_full": (tiny(pp=4, n_microbatches=8), "full"),
    "1.3b_tp2pp4_24gb": (gp.GPTConfig(**{**gp.CONFIGS["1.3b"].__dict__, "mem_budget_bytes": 24_000_000_000}), "heu"),
    "7b_tp2pp4_80gb": (gp.GPTConfig(**{**gp.CONFIGS["7b"].__dict__, "mem_budget_bytes": 80_000_000_000}), "heu"),
    "13b_tp4pp2_40gb": (gp.GPTConfig(**{**gp.CONFIGS["13b"].__dict__, "mem_budget_bytes": 40_000_000_000}), "heu"),
}


def executor_ledgers(c, text, plans, sim):
    out = []
    layers = plans[0]["layers_per_stage"]
    for s in range(c.pp):
        cfg = ex.make_config(c, layers, exec_opts={"dry_run": True, "ledger_pass_start_us": sim["pass_start_us"][s]})
        e = ex.Executor(text, plans[s]["timeline"], cfg)
        try:
            e.step(None, None)
            out.append(e.report()["ledger"])
        finally:
            e.close()
    return out


@pytest.mark.parametrize("name", list(CASES))
def test_executor_ledger_equals_simulator(name):
    c, baseline = CASES[name]
    text = gp.profile_text(c)
    plans = [ex.plan_for(text, s, baseline) for s in range(c.pp)]
    layers = plans[0]["layers_per_stage"]
    timelines = [p["timeline"] for p in plans]
    sim = planner.simulate_timelines_text(text, layers, timelines)
    kinds = {it["host"] for p in plans for it in p["timeline"]["items"]}
    led = executor_ledgers(c, text, plans, sim)
    for s in range(c.pp):
        assert led[s]["plan_clock"] == "simulator"
        assert led[s]["memory_trace"] == sim["memory_traces"][s], (name, s)
        assert led[s]["memory_peak_bytes"] == sim["memory_peaks"][s], (name, s)
    from oracle import ref as oref
    if oref.available():
        ref = oref.RefLib().simulate_timelines(text, layers, timelines)
        for s in range(c.pp):
            assert led[s]["memory_trace"] == ref["memory_traces"][s], (name, s)
            assert led[s]["memory_peak_bytes"] == ref["memory_peaks"][s], (name, s)
    if name in ("tp_template_window", "tp2_heu"):
        assert "window" in kinds


@pytest.mark.parametrize("name", ["1.3b_tp2pp4_24gb", "7b_tp2pp4_80gb"])
def test_all_three_hosts_are_covered(name):
    c, baseline = CASES[name]
    text = gp.profile_text(c)
    kinds = {it["host"] for s in range(c.pp) for it in ex.plan_for(text, s, baseline)["timeline"]["items"]}
    assert {"window", "critical", "stall"} <= kinds


def test_ledger_clock_needs_one_start_per_pass():
    c, baseline = CASES["tp1_full"]
    text = gp.profile_text(c)
    plan = ex.plan_for(text, 0, baseline)
    cfg = ex.make_config(c, plan["layers_per_stage"], exec_opts={"dry_run": True, "ledger_pass_start_us": ["0"]})
    with pytest.raises(ex.LynxError) as err:
        ex.Executor(text, plan["timeline"], cfg)
    assert err.value.code == 1


# simreport.schema.json (proj/schemas/simreport.schema.json) restated: required keys, no extra keys,
# string-valued quantities, event kinds. Used on the GPU box, where /root/reference does not exist.
SIMREPORT_KEYS = {"iteration_us", "per_stage", "breakdown", "memory_peaks", "timeline"}
STAGE_KEYS = {"busy_us", "comm_us", "stall_us", "recompute_on_demand_us", "recompute_overlapped_us"}
BREAKDOWN_KEYS = {"no_recompute", "overlapped", "on_demand"}
EVENT_KINDS = {"fwd", "bwd", "comm_fwd", "comm_bwd", "recompute", "stall_recompute", "p2p", "stall"}


def check_simreport_shape(doc: dict):
    assert set(doc) == SIMREPORT_KEYS
    assert isinstance(doc["iteration_us"], str)
    for st in doc["per_stage"]:
        assert set(st) == STAGE_KEYS and all(isinstance(v, str) for v in st.values())
    for b in doc["breakdown"]:
        assert set(b) == BREAKDOWN_KEYS and all(isinstance(v, str) for v in b.values())
    assert all(isinstance(p, str) for p in doc["memory_peaks"])
    for ev in doc["timeline"]:
        assert {"stage", "microbatch", "kind", "start_us", "end_us", "overlapped"} <= set(ev)
        assert set(ev) <= {"stage", "microbatch", "kind", "op_id", "start_us", "end_us", "overlapped"}
        assert ev["kind"] in EVENT_KINDS and isinstance(ev["overlapped"], bool)


def test_executor_simreport_validates_against_reference_schema():
    import os
    c, baseline = CASES["tp_template_window"]
    text = gp.profile_text(c)
    plan = ex.plan_for(text, 0, baseline)
    e = ex.Executor(text, plan["timeline"], ex.make_config(c, plan["layers_per_stage"], exec_opts={"dry_run": True}))
    try:
        e.step(None, None)
        doc = e.simreport()
    finally:
        e.close()
    check_simreport_shape(doc)
    path = "/root/reference/proj/schemas/simreport.schema.json"
    if os.path.exists(path):
        import jsonschema
        jsonschema.validate(doc, json.load(open(path)))
    # the native simulator's report passes the same restated check (the restatement is not vacuous)
    sim = planner.simulate_timelines_text(text, plan["layers_per_stage"], [plan["timeline"]])
    check_simreport_shape(sim["report"])
