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
                train: dict | None = None, exec_opts: dict | None = None) -> dict:
    return {
        "model": {"hidden": c.hidden, "heads": c.heads, "seq": c.seq, "micro_batch": c.micro_batch,
                  "vocab": c.vocab},
        "layers_per_stage": list(layers_per_stage),
        "parallel": {"tp": c.tp, "tp_rank": tp_rank, "world_rank": world_rank, "world_size": world_size,
                     "nccl_id": nccl_id},
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
        d["w_head"] = (c.vocab, h)
    return d


def synthetic_batch(c: gp.GPTConfig, seed: int = 1234) -> tuple[np.ndarray, np.ndarray]:
    """Tokens uniform in [0, 50257) (GPT-2 vocabulary; the model vocab is padded to a multiple of 128),
    labels = next token. Shape [n_microbatches * micro_batch * seq]."""
    rng = np.random.default_rng(seed)
    seqs = rng.integers(0, min(50257, c.vocab), size=(c.n_microbatches * c.micro_batch, c.seq + 1), dtype=np.int64)
    return seqs[:, :-1].astype(np.int32).ravel(), seqs[:, 1:].astype(np.int32).ravel()
