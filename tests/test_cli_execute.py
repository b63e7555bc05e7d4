"""`lynx_execute` (paper_2406_08756_b200/cli/lynx_execute.cpp): the compiled `lynx execute` CLI over the
C-ABI, the sibling of the reference CLI's `simulate` (proj/tools/lynx_main.cpp:200-226). On CPU it runs in
dry-run mode (the executor's full launch program, no device); the GPU test runs a real iteration."""
import json
import subprocess

import pytest

from paper_2406_08756_b200 import build as B
from paper_2406_08756_b200 import executor as ex
from paper_2406_08756_b200 import gpt_profile as gp
from paper_2406_08756_b200 import planner


def _files(tmp_path, exec_opts):
    c = gp.GPTConfig("gpt-tiny", 4, 512, 8, 256, 2, 50304, 1, 1, 2, dropout=0.1, tp_template=True,
                     mem_budget_bytes=gp.BYTES_PER_PARAM_STATIC * gp.GPTConfig("t", 4, 512, 8, 256, 2).params()
                     + 22 * 2**20)
    text = gp.profile_text(c)
    (tmp_path / "p.json").write_text(text)
    (tmp_path / "c.json").write_text(json.dumps(ex.make_config(c, [4], exec_opts=exec_opts)))
    return c, text


def run(tmp_path, *args):
    if not B.CLI.exists():
        pytest.skip("lynx_execute not built")
    import os
    env = {k: v for k, v in os.environ.items() if k != "NCCL_DEBUG"}
    r = subprocess.run([str(B.CLI), str(tmp_path / "p.json"), str(tmp_path / "c.json"), *args],
                       capture_output=True, text=True, timeout=300, env=env)
    return r.returncode, r.stdout, r.stderr


def test_cli_dry_run_report_and_ledger(tmp_path):
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0])
    from test_ledger_parity import check_simreport_shape
    c, text = _files(tmp_path, {"dry_run": True})
    rc, out, err = run(tmp_path, "--mode", "heu", "--format", "json")
    assert rc == 0, err
    check_simreport_shape(json.loads(out))
    rc, out, err = run(tmp_path, "--mode", "heu", "--format", "stats")
    assert rc == 0, err
    stats = json.loads(out)
    plan = ex.plan_for(text, 0, "heu")
    sim = planner.simulate_timelines_text(text, plan["layers_per_stage"], [plan["timeline"]])
    assert stats["ledger"]["memory_trace"] == sim["memory_traces"][0]  # back-to-back clock = PP1 simulator clock
    assert stats["recompute_launches"] == len(plan["timeline"]["items"]) > 0  # every plan item issued


def test_cli_exit_codes(tmp_path):
    _files(tmp_path, {"dry_run": True})
    assert run(tmp_path, "--mode", "bogus")[0] == 1
    (tmp_path / "p.json").write_text("{not json")
    assert run(tmp_path)[0] == 2


@pytest.mark.gpu
def test_cli_runs_a_real_iteration(tmp_path, cuda):
    _files(tmp_path, {"trace": True, "reserve_pool": False})
    rc, _, err = run(tmp_path, "--mode", "heu", "--steps", "2", "--format", "csv", "--out", str(tmp_path / "t.csv"))
    assert rc == 0, err
    lines = (tmp_path / "t.csv").read_text().splitlines()  # stdout may carry NCCL's banner
    assert lines[0] == "stage,microbatch,kind,op_id,start_us,end_us,overlapped"
    kinds = {ln.split(",")[2] for ln in lines[1:]}
    assert {"fwd", "bwd", "comm_fwd", "recompute"} <= kinds
