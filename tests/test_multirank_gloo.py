"""The N > 1 path with real processes: world_size-2 `gloo` runs on CPU.

One process per rank, as `bench.py` runs under torchrun. Each rank
- takes the operator times rank 0 measured through `broadcast_object_list` (the bench's
  flow) and plans from the same profile document: every rank must hold identical plans;
- builds its own launch program with the executor in dry-run mode (the C-ABI, no GPU), and
- replays that program's collectives over gloo in program order: TP all-reduces on the TP
  group, pipeline sends / receives with one tag per communicator (activations, gradients),
  with each message sized from the program's byte count.
A mismatch in order, size or pairing between ranks makes gloo fail (size mismatch) or hang
(caught by the process-group timeout), so a passing run shows that the ranks' programs are
consistent end to end — the property the NCCL path on 8 x B200 relies on.
"""
import datetime
import hashlib
import json
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

TAG = {"pp_act": 1, "pp_grad": 2}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, cfg_kw: dict, out_dir: str) -> None:
    from fractions import Fraction

    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=60))
    c = gp.GPTConfig(**cfg_kw)
    # rank 0 "measures" (here: the analytic estimate, perturbed so the document is rank-0 specific)
    obj = [{k: str(v * Fraction(1001, 1000)) for k, v in gp.estimate_times(c).items()} if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    times = {k: Fraction(v) for k, v in obj[0].items()}
    text = gp.profile_text(c, times=times)
    plans = [ex.plan_for(text, s) for s in range(c.pp)]
    digest = hashlib.sha256(json.dumps([p["plan_json"] for p in plans]).encode()).hexdigest()
    digests = [None] * world
    dist.all_gather_object(digests, digest)
    assert len(set(digests)) == 1, "ranks planned differently"

    stage, tp_rank = rank // c.tp, rank % c.tp
    cfg = ex.make_config(c, plans[0]["layers_per_stage"], tp_rank=tp_rank, world_rank=rank, world_size=world,
                         exec_opts={"dry_run": True})
    e = ex.Executor(text, plans[stage]["timeline"], cfg)
    e.step(None, None)
    program = e.program()
    e.close()

    tp_groups = [dist.new_group([s * c.tp + r for r in range(c.tp)]) for s in range(c.pp)]
    works, n_ops = [], {"allreduce": 0, "send": 0, "recv": 0}
    for op in program:
        n = max(1, op["bytes"] // (1 << 20))  # one fp32 per MiB keeps the messages small but size-checked
        buf = torch.full((n,), float(rank + 1))
        if op["kind"] == "allreduce":
            works.append(dist.all_reduce(buf, group=tp_groups[stage], async_op=True))
        else:
            peer = op["peer"] * c.tp + tp_rank  # peer stage -> global rank (same TP rank)
            fn = dist.isend if op["kind"] == "send" else dist.irecv
            works.append(fn(buf, peer, tag=TAG[op["comm"]]))
        n_ops[op["kind"]] += 1
    for w in works:
        w.wait()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"ops": n_ops, "digest": digest}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,kw", [
    ("tp2", dict(tp=2, pp=1, n_microbatches=2)),
    ("tp2_vocab_parallel", dict(tp=2, pp=1, n_microbatches=2, vocab=50432)),
    ("pp2", dict(tp=1, pp=2, n_microbatches=4)),
])
def test_two_rank_programs_replay_over_gloo(tmp_path, name, kw):
    from paper_2406_08756_b200 import gpt_profile as gp
    base = gp.CONFIGS["1.3b"].__dict__.copy()
    base.update(kw, n_layers=4, mem_budget_bytes=24_000_000_000)
    mp.spawn(_worker, args=(2, _free_port(), base, str(tmp_path)), nprocs=2, join=True)
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(2)]
    assert res[0]["digest"] == res[1]["digest"]
    if kw["tp"] == 2:  # both TP ranks issue the same all-reduces (fwd + bwd windows, recomputed ones included)
        assert res[0]["ops"]["allreduce"] == res[1]["ops"]["allreduce"] >= 4 * 4 * kw["n_microbatches"]
    else:  # stage 0 sends every activation the last stage receives, and the gradients back
        assert res[0]["ops"]["send"] == res[1]["ops"]["recv"] == kw["n_microbatches"]
        assert res[1]["ops"]["send"] == res[0]["ops"]["recv"] == kw["n_microbatches"]
