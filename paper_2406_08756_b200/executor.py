"""Python handle on the B200 executor C-ABI (include/lynx_rt.h, `lynx_rt_*`).

The executor replaces the reference's CPU `simulate()` for one pipeline stage
on one TP rank: it consumes the same profile and the same
StageRecomputeTimeline (from `planner.stage_plan_text`) and runs the real
training step on the GPU. This wrapper only marshals arguments; all work
happens in `_lib/liblynx_b200.so`.
"""
from __future__ import annotations

import ctypes
import json

import numpy as np

from . import gpt_profile as gp
from . import planner
from ._native import LynxError, lib

_c = ctypes
_SIGS = {
    "lynx_rt_create": (_c.c_int, [_c.c_char_p, _c.c_char_p, _c.c_char_p, _c.POINTER(_c.c_void_p)]),
    "lynx_rt_step": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.POINTER(_c.c_float)]),
    "lynx_rt_report_json": (_c.c_void_p, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "lynx_rt_stats_json": (_c.c_void_p, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "lynx_rt_trace": (_c.c_void_p, [_c.c_void_p, _c.c_int, _c.POINTER(_c.c_int)]),
    "lynx_rt_program_json": (_c.c_void_p, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "lynx_rt_get_tensor": (_c.c_int, [_c.c_void_p, _c.c_char_p, _c.c_void_p, _c.c_size_t]),
    "lynx_rt_set_tensor": (_c.c_int, [_c.c_void_p, _c.c_char_p, _c.c_void_p, _c.c_size_t]),
    "lynx_rt_nccl_unique_id": (_c.c_int, [_c.c_char_p, _c.c_size_t]),
    "lynx_rt_destroy": (None, [_c.c_void_p]),
    "lynx_free": (None, [_c.c_void_p]),
}
_bound = False


def _lib():
    global _bound
    l = lib()
    if not _bound:
        for n, (r, a) in _SIGS.items():
            f = getattr(l, n)
            f.restype = r
            f.argtypes = a
        _bound = True
    return l


def _check(code: int):
    if code:
        raise LynxError(code, _lib().lynx_last_error().decode(errors="replace"))


def _take(ptr, st) -> str:
    if not ptr:
        raise LynxError(st.value, _lib().lynx_last_error().decode(errors="replace"))
    try:
        return _c.cast(ptr, _c.c_char_p).value.decode()
    finally:
        _lib().lynx_free(ptr)


def nccl_unique_id() -> str:
    buf = _c.create_string_buffer(512)
    _check(_lib().lynx_rt_nccl_unique_id(buf, 512))
    return buf.value.decode()


class Executor:
    def __init__(self, profile_text: str, timeline: dict, config: dict):
        self._h = _c.c_void_p()
        self.config = config
        self.profile_text = profile_text
        self.timeline = timeline
        _check(_lib().lynx_rt_create(profile_text.encode(), json.dumps(timeline).encode(),
                                     json.dumps(config).encode(), _c.byref(self._h)))

    def close(self):
        if self._h:
            _lib().lynx_rt_destroy(self._h)
            self._h = _c.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, tokens: np.ndarray | None, labels: np.ndarray | None) -> float:
        loss = _c.c_float(0.0)
        t = None if tokens is None else np.ascontiguousarray(tokens, dtype=np.int32)
        y = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
        _check(_lib().lynx_rt_step(self._h, None if t is None else t.ctypes.data, None if y is None else y.ctypes.data,
                                   _c.byref(loss)))
        return float(loss.value)

    def report(self) -> dict:
        """Executor counters of the last step (lynx_rt_stats_json), incl. the logical ledger."""
        st = _c.c_int(0)
        return json.loads(_take(_lib().lynx_rt_stats_json(self._h, _c.byref(st)), st))

    def simreport(self) -> dict:
        """The last step's measured report in simreport.schema.json shape (lynx_rt_report_json)."""
        st = _c.c_int(0)
        return json.loads(_take(_lib().lynx_rt_report_json(self._h, _c.byref(st)), st))

    def trace(self, fmt: str = "chrome") -> str:
        st = _c.c_int(0)
        return _take(_lib().lynx_rt_trace(self._h, 0 if fmt == "chrome" else 1, _c.byref(st)), st)

    def program(self) -> list:
        st = _c.c_int(0)
        return json.loads(_take(_lib().lynx_rt_program_json(self._h, _c.byref(st)), st))

    def get(self, name: str, n: int) -> np.ndarray:
        """Parameter (bf16 -> float32 array) or gradient ("grad:<name>", fp32) with n elements."""
        if name.startswith("grad:"):
            out = np.empty(n, dtype=np.float32)
            _check(_lib().lynx_rt_get_tensor(self._h, name.encode(), out.ctypes.data, out.nbytes))
            return out
        raw = np.empty(n, dtype=np.uint16)
        _check(_lib().lynx_rt_get_tensor(self._h, name.encode(), raw.ctypes.data, raw.nbytes))
        return (raw.astype(np.uint32) << 16).view(np.float32)

    def set(self, name: str, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float32)
        _check(_lib().lynx_rt_set_tensor(self._h, name.encode(), v.ctypes.data, v.nbytes))


def make_config(c: gp.GPTConfig, layers_per_stage, *, tp_rank=0, world_rank=0, world_size=1, nccl_id="",
                loopback: str = "", train: dict | None = None, exec_opts: dict | None = None) -> dict:
    par = {"tp": c.tp, "tp_rank": tp_rank, "world_rank": world_rank, "world_size": world_size, "nccl_id": nccl_id}
    if loopback:
        par["loopback"] = loopback
    return {
        "model": {"hidden": c.hidden, "heads": c.heads, "seq": c.seq, "micro_batch": c.micro_batch,
                  "vocab": c.vocab},
        "layers_per_stage": list(layers_per_stage),
        "parallel": par,
        "train": {"dropout": c.dropout, "seed": 42, "lr": 1e-4, "beta1": 0.9, "beta2": 0.95, "eps": 1e-8,
                  "weight_decay": 0.1, "init_std": 0.02, **(train or {})},
        "exec": dict(exec_opts or {}),
    }


def plan_for(profile_text: str, stage: int, baseline: str = "heu", layers_per_stage=None) -> dict:
    """Stage plan through the native planner: {plan_json, timeline, period_us, layers_per_stage}."""
    return planner.stage_plan_text(profile_text, stage, layers_per_stage, baseline)


def param_shapes(c: gp.GPTConfig, layers: int, first: bool, last: bool) -> dict[str, tuple]:
    """Per-rank parameter shapes in the executor's layout (runtime/params.cpp)."""
    h, hp = c.hidden, c.hidden // c.tp
    d: dict[str, tuple] = {}
    if first:
        d["wte"] = (c.vocab, h)
        d["wpe"] = (c.seq, h)
    for l in range(layers):
        p = f"l{l}."
        d.update({p + "ln1_g": (h,), p + "ln1_b": (h,), p + "w_qkv": (3 * hp, h), p + "b_qkv": (3 * hp,),
                  p + "w_proj": (h, hp), p + "b_proj": (h,), p + "ln2_g": (h,), p + "ln2_b": (h,),
                  p + "w_fc1": (4 * hp, h), p + "b_fc1": (4 * hp,), p + "w_fc2": (h, 4 * hp), p + "b_fc2": (h,)})
    if last:
        d["lnf_g"] = (h,)
        d["lnf_b"] = (h,)
        d["w_head"] = (c.vocab // c.tp if c.vocab_parallel else c.vocab, h)
    return d


def synthetic_batch(c: gp.GPTConfig, seed: int = 1234) -> tuple[np.ndarray, np.ndarray]:
    """Tokens uniform in [0, 50257) (GPT-2 vocabulary; the model vocab is padded to a multiple of 128),
    labels = next token. Shape [n_microbatches * micro_batch * seq]."""
    rng = np.random.default_rng(seed)
    seqs = rng.integers(0, min(50257, c.vocab), size=(c.n_microbatches * c.micro_batch, c.seq + 1), dtype=np.int64)
    return seqs[:, :-1].astype(np.int32).ravel(), seqs[:, 1:].astype(np.int32).ravel()


class LoopbackGrid:
    """Every (stage, TP rank) executor of a TP x PP configuration inside this process, on one GPU.

    The ranks talk through the executor's in-process loopback Comms (runtime/comm.hpp:
    parallel.loopback) instead of NCCL, which cannot place two ranks on one device; each
    rank is driven by its own host thread (ctypes releases the GIL), exactly as one process
    per GPU drives it under torchrun. This is how the sharded numerics — Megatron column /
    row splits, the four TP all-reduces per layer, the 1F1B pipeline hand-off, the plan's
    window recomputes overlapping the all-reduces — are checked against the unsharded CPU
    oracle on a single B200.
    """

    _count = 0

    def __init__(self, c: gp.GPTConfig, profile_text: str, plans: list[dict], *, exec_opts: dict | None = None,
                 train: dict | None = None, stage_exec_opts: list[dict] | None = None):
        LoopbackGrid._count += 1
        name = f"grid{LoopbackGrid._count}-{id(self):x}"
        self.c = c
        self.layers = plans[0]["layers_per_stage"]
        opts = {"reserve_pool": False, **(exec_opts or {})}
        self.ranks: dict[tuple[int, int], Executor] = {}
        try:
            for s in range(c.pp):
                for r in range(c.tp):
                    cfg = make_config(c, self.layers, tp_rank=r, world_rank=s * c.tp + r, world_size=c.tp * c.pp,
                                      loopback=name, train=train,
                                      exec_opts={**opts, **(stage_exec_opts[s] if stage_exec_opts else {})})
                    self.ranks[(s, r)] = Executor(profile_text, plans[s]["timeline"], cfg)
        except Exception:
            self.close()
            raise

    def step(self, tokens: np.ndarray, labels: np.ndarray) -> dict[tuple[int, int], float]:
        """One training iteration on every rank concurrently; returns each rank's loss (last stage)."""
        import threading
        out: dict[tuple[int, int], float] = {}
        errs: list[BaseException] = []

        def run(key, e):
            try:
                s = key[0]
                out[key] = e.step(tokens if s == 0 else None, labels if s == self.c.pp - 1 else None)
            except BaseException as exc:  # noqa: BLE001 - re-raised below
                errs.append(exc)

        th = [threading.Thread(target=run, args=(k, e)) for k, e in self.ranks.items()]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        return out

    def reports(self) -> dict[tuple[int, int], dict]:
        return {k: e.report() for k, e in self.ranks.items()}

    def rank_tensors(self, grad: bool) -> dict[tuple[int, int], dict[str, np.ndarray]]:
        """Per rank: its parameters (or fp32 gradients) under GLOBAL layer names."""
        out = {}
        l0 = [sum(self.layers[:s]) for s in range(self.c.pp)]
        for (s, r), e in self.ranks.items():
            shapes = param_shapes(self.c, self.layers[s], s == 0, s == self.c.pp - 1)
            d = {}
            for k, shp in shapes.items():
                v = e.get(("grad:" if grad else "") + k, int(np.prod(shp))).reshape(shp)
                if k.startswith("l") and "." in k:
                    k = f"l{int(k[1:k.index('.')]) + l0[s]}{k[k.index('.'):]}"
                d[k] = v
            out[(s, r)] = d
        return out

    def close(self):
        for e in self.ranks.values():
            e.close()
        self.ranks = {}


# Megatron split of each per-layer tensor: (kind, axis, blocks). "rows": column-parallel output rows
# (QKV's q | k | v blocks of hp rows each, FC1's 4hp rows); "cols": row-parallel input columns.
_SPLIT = {"w_qkv": ("rows", 3), "b_qkv": ("rows", 3), "w_fc1": ("rows", 1), "b_fc1": ("rows", 1),
          "w_proj": ("cols", 1), "w_fc2": ("cols", 1)}


def unshard(per_rank: list[np.ndarray], name: str, vocab_parallel: bool = False) -> np.ndarray:
    """Reassemble one tensor from its TP-rank slices (rank order); replicated tensors come back from
    rank 0 (callers check the replicas are identical). With `vocab_parallel` the LM head is split by
    vocabulary rows."""
    base = name[name.index(".") + 1:] if name.startswith("l") and "." in name else name
    if base == "w_head" and vocab_parallel and len(per_rank) > 1:
        return np.concatenate(per_rank, axis=0)
    if base not in _SPLIT or len(per_rank) == 1:
        return per_rank[0]
    kind, blocks = _SPLIT[base]
    if kind == "cols":
        return np.concatenate(per_rank, axis=1)
    parts = [np.split(x, blocks, axis=0) for x in per_rank]  # [rank][block]
    return np.concatenate([parts[r][b] for b in range(blocks) for r in range(len(per_rank))], axis=0)


def is_tp_sharded(name: str, vocab_parallel: bool = False) -> bool:
    base = name[name.index(".") + 1:] if name.startswith("l") and "." in name else name
    return base in _SPLIT or (vocab_parallel and base == "w_head")
