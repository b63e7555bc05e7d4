"""OPT plans through an external MILP solver (paper_2406_08756_b200/opt_milp.py).

- On a full stage the exported program is the reference's OPT model: HiGHS reaches the same
  optimal cost as the native branch-and-bound (itself byte-identical to the reference's
  optsched, tests/test_planner_parity.py).
- The native exact checker (check_schedule, optsched.cpp:245-338) rejects a schedule that breaks
  the budget, whatever produced it.
- A layer slice solved with HiGHS and replicated over a 1.3B pipeline stage fits the stage's
  budget under the native simulator's ledger.
- On a B200 the executor replays an OPT-slice timeline (window and critical-path items) with
  recomputed tensors bit-identical to the forward ones, and loss / gradients bit-identical to
  retain-all.
"""
import json
from fractions import Fraction

import numpy as np
import pytest

pytest.importorskip("scipy.optimize")

SMALL_OPT = {"model": {"name": "opt-small", "n_layers": 2, "static_bytes": 4, "layer": {"ops": [
    {"id": 0, "name": "a", "kind": "compute", "time_us": 2, "out_bytes": 4, "deps": []},
    {"id": 1, "name": "g", "kind": "comm", "time_us": 3, "out_bytes": 2, "deps": [0]},
    {"id": 2, "name": "ck", "kind": "compute", "time_us": "3/2", "out_bytes": 2, "deps": [1]},
    {"id": 3, "name": "d", "kind": "compute", "time_us": 2, "out_bytes": 1, "deps": [0, 2]}],
    "fwd_comm_ids": [], "bwd_comm_ids": [], "checkpoint_id": 2}},
    "hardware": {"mem_budget_bytes": 14, "comm_scale": 1},
    "pipeline": {"n_stages": 2, "n_microbatches": 2}}


def tiny_tp(extra_mib: int):
    from paper_2406_08756_b200 import gpt_profile as gp
    base = dict(name="gpt-tiny-tp", n_layers=4, hidden=512, heads=8, seq=256, micro_batch=2, vocab=50304, tp=1,
                pp=1, n_microbatches=2, dropout=0.1, tp_template=True)
    static = gp.BYTES_PER_PARAM_STATIC * gp.GPTConfig(**base).params()
    return gp.GPTConfig(**{**base, "mem_budget_bytes": static + extra_mib * 2**20}), gp.GPTConfig(**base)


@pytest.mark.parametrize("stage", [0, 1])
def test_full_stage_highs_matches_native_bnb(stage):
    from paper_2406_08756_b200 import opt_milp
    from paper_2406_08756_b200 import planner as pl
    text = json.dumps(SMALL_OPT)
    native = json.loads(pl.schedule_text(text, "opt", stage, None, 2000)[0])
    r = opt_milp.solve_stage(text, stage, None, slice_layers=0, time_limit_s=30)
    assert native["status"] == r["status"] == "optimal"
    assert Fraction(r["cost_us"]) == Fraction(native["objective_us"])
    assert r["n_recompute"] == len(native["recompute"])


def test_exact_checker_rejects_an_over_budget_schedule():
    from paper_2406_08756_b200 import planner as pl
    text = json.dumps(SMALL_OPT)
    m = pl.opt_export_text(text, 0)
    n = m["n_ops"]
    keep_all = {"keep": [[t, i] for t in range(1, n) for i in range(t)], "recompute": []}
    out, st = pl.opt_timeline_text(text, 0, keep_all)
    assert st == 1 and "BudgetViolation" in out["issues"] and "timeline" not in out


def test_export_is_well_formed():
    from paper_2406_08756_b200 import planner as pl
    c, _ = tiny_tp(22)
    from paper_2406_08756_b200 import gpt_profile as gp
    m = pl.opt_export_text(gp.profile_text(c), 0, [4], 1)
    n, rows = m["n_vars"], m["n_rows"]
    assert len(m["lo"]) == len(m["hi"]) == len(m["integer"]) == n
    assert len(m["row"]) == len(m["col"]) == len(m["val"]) and len(m["sense"]) == len(m["rhs"]) == rows
    assert max(m["row"]) < rows and max(m["col"]) < n
    assert len(m["R"]) == len(m["S"]) == m["n_ops"]
    assert all(len(m["R"][t]) == t + 1 and len(m["S"][t]) == t for t in range(m["n_ops"]))
    # the replication rows: one Y variable, one retained_t row per phase
    assert sum(1 for k in m["integer"] if k == 0) > m["n_ops"]


def test_slice_plan_fits_a_pipeline_stage():
    """1.3B TP2xPP4 (estimated times): the last stage's OPT slice, replicated, fits its budget."""
    from paper_2406_08756_b200 import gpt_profile as gp
    from paper_2406_08756_b200 import opt_milp
    from paper_2406_08756_b200 import planner as pl
    text = gp.profile_text(gp.CONFIGS["1.3b"])
    part = json.loads(pl.partition_text(text))["layers_per_stage"]
    stage = len(part) - 1
    r = opt_milp.plan_stage(text, stage, part, slice_layers=1, time_limit_s=60)
    budget = json.loads(text)["hardware"]["mem_budget_bytes"]
    assert r["stage_peak_bytes"] <= budget
    items = r["timeline"]["items"]
    retained = r["timeline"]["plan"]["retained"]
    assert items and all(not retained[it["op"]] for it in items)  # only discarded ops are regenerated
    assert {it["owner_layer"] for it in items} <= set(range(part[stage]))
    assert r["n_overlapped"] >= 1  # OPT hides recomputation in the all-reduce windows


@pytest.mark.gpu
def test_opt_slice_timeline_replays_bit_identical(cuda):
    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    from paper_2406_08756_b200 import opt_milp
    tight, loose = tiny_tp(22)
    text = gp.profile_text(tight)
    r = opt_milp.plan_stage(text, 0, [4], slice_layers=1, time_limit_s=60)
    tl = r["timeline"]
    assert tl["items"] and {it["host"] for it in tl["items"]} >= {"window"}

    def run(c, timeline):
        t = gp.profile_text(c)
        e = ex.Executor(t, timeline, ex.make_config(c, [c.n_layers], exec_opts={"check_recompute": True}))
        tok, lab = ex.synthetic_batch(c)
        loss = e.step(tok, lab)
        shapes = ex.param_shapes(c, c.n_layers, True, True)
        grads = {k: e.get("grad:" + k, int(np.prod(s))) for k, s in shapes.items()}
        rep = e.report()
        e.close()
        return loss, grads, rep

    l_opt, g_opt, rep = run(tight, tl)
    assert rep["recompute_launches"] == len(tl["items"])
    assert rep["recompute_checked"] > 0 and rep["recompute_mismatch_words"] == 0
    keep = ex.plan_for(gp.profile_text(loose), 0, "retain_all")["timeline"]
    l_keep, g_keep, _ = run(loose, keep)
    assert l_opt == l_keep
    for k in g_keep:
        assert np.array_equal(g_keep[k], g_opt[k]), k
