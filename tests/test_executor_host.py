"""Executor host logic without a GPU: dry-run launch programs for TP/PP configurations.

The multi-GPU path cannot run in this round (one B200 per call), so these CPU
tests build every rank's launch program in dry-run mode and check that the
collectives are consistent: both TP ranks of a stage issue the same all-reduce
sequence (same sizes, same order — recomputed all-reduces included), and every
pipeline send has a matching receive of the same size, in the same order, on
the same communicator. Activations and gradients travel on separate
communicators whose per-direction sequences are monotone in the microbatch, so
1F1B cannot deadlock.
"""
import json

import pytest

from paper_2406_08756_b200 import executor as ex
from paper_2406_08756_b200 import gpt_profile as gp


def dry_programs(c: gp.GPTConfig, budget: int | None = None):
    if budget:
        c = gp.GPTConfig(**{**c.__dict__, "mem_budget_bytes": budget})
    text = gp.profile_text(c)
    progs = {}
    plans = [ex.plan_for(text, s) for s in range(c.pp)]
    layers = plans[0]["layers_per_stage"]
    for s in range(c.pp):
        for r in range(c.tp):
            cfg = ex.make_config(c, layers, tp_rank=r, exec_opts={"dry_run": True})
            e = ex.Executor(text, plans[s]["timeline"], cfg)
            e.step(None, None)
            progs[(s, r)] = e.program()
            e.close()
    return progs, plans


@pytest.mark.parametrize("key,budget", [("1.3b", None), ("1.3b", 24_000_000_000), ("7b", None), ("13b", 40_000_000_000)])
def test_tp_allreduce_sequences_match(key, budget):
    c = gp.CONFIGS[key]
    progs, plans = dry_programs(c, budget)
    for s in range(c.pp):
        seqs = [[(o["kind"], o["bytes"], o["what"]) for o in progs[(s, r)] if o["comm"] == "tp"] for r in range(c.tp)]
        assert all(q == seqs[0] for q in seqs)
        # two forward and two backward all-reduces per layer per microbatch (+ phase-5 recomputes)
        n_layers = plans[0]["layers_per_stage"][s]
        assert len(seqs[0]) >= 4 * n_layers * c.n_microbatches


@pytest.mark.parametrize("key", ["1.3b", "7b", "13b"])
def test_pipeline_sends_match_receives(key):
    c = gp.CONFIGS[key]
    progs, _ = dry_programs(c)
    for comm, direction in [("pp_act", +1), ("pp_grad", -1)]:
        for r in range(c.tp):
            for s in range(c.pp):
                peer = s + direction
                if not 0 <= peer < c.pp:
                    continue
                sends = [(o["bytes"], o["what"]) for o in progs[(s, r)] if o["comm"] == comm and o["kind"] == "send"]
                recvs = [(o["bytes"], o["what"]) for o in progs[(peer, r)]
                         if o["comm"] == comm and o["kind"] == "recv" and o["peer"] == s]
                assert sends == recvs and len(sends) == c.n_microbatches
                mbs = [int(w.split("mb")[1]) for _, w in sends]
                assert mbs == sorted(mbs)  # monotone per direction: no 1F1B cycle


def test_single_gpu_program_has_no_collectives():
    c = gp.CONFIGS["tiny"]
    progs, _ = dry_programs(c)
    assert progs[(0, 0)] == []


def test_executor_rejects_foreign_templates():
    from paper_2406_08756_b200._native import LynxError
    c = gp.CONFIGS["tiny"]
    text = json.loads(gp.profile_text(c))
    text["model"]["layer"]["ops"][1]["name"] = "mystery"
    t = json.dumps(text)
    plan = ex.plan_for(t, 0)
    with pytest.raises(LynxError):
        ex.Executor(t, plan["timeline"], ex.make_config(c, plan["layers_per_stage"], exec_opts={"dry_run": True}))


def test_comm_standin_stage_program():
    """exec.comm_standin_us (tools/emulate_stage.py): one TP rank of a TP2 stage runs alone with
    stand-in all-reduces; its launch program keeps the TP rank's all-reduce sequence (same windows)
    and the PP transfers become synthetic. Without a stand-in, or outside a standalone stage, it is
    rejected."""
    from paper_2406_08756_b200._native import LynxError
    c = gp.CONFIGS["1.3b"]
    progs, plans = dry_programs(c)
    text = gp.profile_text(c)
    layers = plans[0]["layers_per_stage"]
    for s in (0, c.pp - 1):
        opts = {"dry_run": True, "standalone_stage": True, "comm_standin_us": 500.0}
        e = ex.Executor(text, plans[s]["timeline"], ex.make_config(c, layers, exec_opts=opts))
        e.step(None, None)
        prog = e.program()
        e.close()
        assert prog == progs[(s, 0)] and any(o["comm"] == "tp" for o in prog)
    for opts in ({"dry_run": True, "standalone_stage": True},
                 {"dry_run": True, "comm_standin_us": 500.0}):
        with pytest.raises(LynxError):
            ex.Executor(text, plans[0]["timeline"], ex.make_config(c, layers, exec_opts=opts))


def test_bench_op_times_replay_reproduces_the_measured_plan(tmp_path):
    """`bench.py --op-times` (used for ncu launch lists): the committed bench line's operator times
    give back the plan that line ran (same S, phases and exact peak bytes), and a flat map loads too."""
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import bench
    line_path = root / "profiles" / "r01_bench_n1.json"
    line = json.loads(line_path.read_text())
    times = bench.load_op_times(str(line_path))
    flat = tmp_path / "times.json"
    flat.write_text(json.dumps(line["recompute"]["op_times_us"]))
    assert bench.load_op_times(str(flat)) == times
    import argparse
    c = bench.config_for(1, argparse.Namespace(gpus=1, model="7b", micro_batch=0, microbatches=0, plan="heu"))
    c.mem_budget_bytes = line["memory"]["ledger_budget_bytes"]
    plans, _ = bench.plan_all(c, gp.profile_text(c, times=times), "heu")
    got = json.loads(plans[0]["plan_json"])
    want = line["recompute"]["plan"]
    assert (got["S"], got["phase_assignment"], got["peak_bytes"]) == (want["S"], want["phase_assignment"],
                                                                       want["peak_bytes"])


def test_non_causal_timeline_is_rejected_at_create():
    """A timeline whose regeneration of a tensor comes after that tensor's consumer is rejected when the
    executor is created (InconsistentPlan, the reference's exit code 2), not in the middle of a step."""
    import copy
    c = gp.GPTConfig("gpt-tiny", 4, 512, 8, 256, 2, 50304, 1, 1, 2, dropout=0.1)
    text = gp.profile_text(c)
    plan = ex.plan_for(text, 0, "full")
    tl = copy.deepcopy(plan["timeline"])
    late = None
    for it in tl["items"]:
        if it["host"] == "critical" and it["op"] == 1 and it["host_backward"]:  # qkv, consumed by attn_bwd
            it["host_elem"] = 2  # ln1_bwd's element: after attn_bwd read it
            late = it
            break
    assert late is not None
    for dry in (True, False):
        cfg = ex.make_config(c, plan["layers_per_stage"], exec_opts={"dry_run": dry})
        with pytest.raises(ex.LynxError) as err:
            ex.Executor(text, tl, cfg)
        assert err.value.code == 2 and "InconsistentPlan" in str(err.value)
    e = ex.Executor(text, plan["timeline"], ex.make_config(c, plan["layers_per_stage"], exec_opts={"dry_run": True}))
    e.close()


def test_reference_inconsistent_plan_is_rejected_like_the_reference():
    """A HEU plan whose expansion (expand_plan_to_stage) regenerates a tensor's consumer before the tensor
    itself: the reference's own simulate() rejects it (InconsistentPlan, exit code 2) and so does
    lynx_rt_create — the same plan, the same verdict. (TP4·PP2 tiny GPT, budget static/2 + 8 MiB: ln1 of
    (mb 1, layer 1) is regenerated in F(2) but its consumer qkv in B(0), which runs first.)"""
    from paper_2406_08756_b200 import planner
    base = dict(name="t", n_layers=4, hidden=512, heads=8, seq=256, micro_batch=2, vocab=50688, tp=4, pp=2,
                n_microbatches=4, dropout=0.1)
    static = gp.BYTES_PER_PARAM_STATIC * gp.GPTConfig(**base).params() // 4
    c = gp.GPTConfig(**{**base, "mem_budget_bytes": static // 2 + 8 * 2**20})
    text = gp.profile_text(c)
    plans = [ex.plan_for(text, s) for s in range(2)]
    with pytest.raises(ex.LynxError) as ref_err:
        planner.simulate_timelines_text(text, plans[0]["layers_per_stage"], [p["timeline"] for p in plans])
    with pytest.raises(ex.LynxError) as ours:
        ex.Executor(text, plans[0]["timeline"], ex.make_config(c, plans[0]["layers_per_stage"],
                                                               exec_opts={"dry_run": True}))
    assert ref_err.value.code == ours.value.code == 2
    from oracle import ref as oref
    if oref.available():
        with pytest.raises(RuntimeError):
            oref.RefLib().simulate_timelines(text, plans[0]["layers_per_stage"], [p["timeline"] for p in plans])


def test_tp_fused_keeps_the_collective_program_and_rejects_what_it_cannot_run():
    c = gp.GPTConfig("t", 4, 512, 8, 256, 2, 50432, tp=2, pp=2, n_microbatches=4, dropout=0.1,
                     mem_budget_bytes=gp.BYTES_PER_PARAM_STATIC * gp.GPTConfig("t", 4, 512, 8, 256, 2, 50432,
                                                                               tp=2).params() // 4 + 8 * 2**20)
    text = gp.profile_text(c)
    plans = [ex.plan_for(text, s) for s in range(2)]
    for s in range(2):
        progs = []
        for fused in (False, True):
            cfg = ex.make_config(c, plans[0]["layers_per_stage"], exec_opts={"dry_run": True, "tp_fused": fused})
            e = ex.Executor(text, plans[s]["timeline"], cfg)
            e.step(None, None)
            progs.append(e.program())
            e.close()
        assert progs[0] == progs[1]  # same exchanges, same order: only how they run changes
    cfg = ex.make_config(c, plans[0]["layers_per_stage"],
                         exec_opts={"tp_fused": True, "standalone_stage": True, "comm_standin_us": 10})
    with pytest.raises(ex.LynxError) as err:
        ex.Executor(text, plans[0]["timeline"], cfg)
    assert err.value.code == 1
    # a plan that regenerates an all-reduce output (phase 5 on ar1) cannot run fused
    import copy
    tl = copy.deepcopy(plans[0]["timeline"])
    tl["items"].append({"owner_mb": 0, "owner_layer": 0, "op": 4, "host": "critical", "host_mb": 0,
                        "host_backward": True, "host_layer": 0, "host_window": 0, "host_elem": 0})
    with pytest.raises(ex.LynxError) as err:
        ex.Executor(text, tl, ex.make_config(c, plans[0]["layers_per_stage"],
                                             exec_opts={"dry_run": True, "tp_fused": True}))
    assert err.value.code == 1 and "tp_fused" in str(err.value)
