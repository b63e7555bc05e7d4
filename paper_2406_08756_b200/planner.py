"""Host planner API — the reference's `_lynx` Python module, restated.

Same functions, argument meaning and error behaviour as the reference's pybind
module (proj/bindings/module.cpp:75-95): `validate`, `schedule`, `partition`,
`simulate`, `serialize_profile`, each taking a profile *path* and returning the
same JSON text. They call the native C++ planner in `_lib/liblynx_b200.so`
through include/lynx_rt.h (`lynx_plan_*`). Text-level variants (`*_text`) take
the profile document itself, which is what the executor and the benchmarks use.
"""
from __future__ import annotations

import ctypes
import json
from pathlib import Path

from ._native import LynxError, lib

_c = ctypes
_SIGS = {
    "lynx_free": (None, [_c.c_void_p]),
    "lynx_plan_validate": (_c.c_void_p, [_c.c_char_p, _c.c_int, _c.POINTER(_c.c_int)]),
    "lynx_plan_serialize_profile": (_c.c_void_p, [_c.c_char_p, _c.c_int, _c.POINTER(_c.c_int)]),
    "lynx_plan_schedule": (_c.c_void_p, [_c.c_char_p, _c.c_char_p, _c.c_int, _c.c_void_p, _c.c_int, _c.c_longlong,
                                         _c.c_int, _c.POINTER(_c.c_int)]),
    "lynx_plan_partition": (_c.c_void_p, [_c.c_char_p, _c.c_char_p, _c.c_longlong, _c.POINTER(_c.c_int)]),
    "lynx_plan_simulate": (_c.c_void_p, [_c.c_char_p, _c.c_char_p, _c.c_void_p, _c.c_int, _c.c_char_p, _c.c_int,
                                         _c.c_int, _c.c_longlong, _c.POINTER(_c.c_int)]),
    "lynx_plan_stage": (_c.c_void_p, [_c.c_char_p, _c.c_int, _c.c_void_p, _c.c_int, _c.c_int, _c.c_longlong,
                                      _c.POINTER(_c.c_int)]),
    "lynx_plan_simulate_timelines": (_c.c_void_p, [_c.c_char_p, _c.c_void_p, _c.c_int, _c.c_char_p, _c.c_char_p,
                                                   _c.POINTER(_c.c_int)]),
    "lynx_plan_solve_heu": (_c.c_void_p, [_c.c_char_p, _c.c_int, _c.c_int, _c.c_int, _c.c_char_p, _c.c_longlong,
                                          _c.POINTER(_c.c_int)]),
    "lynx_plan_opt_export": (_c.c_void_p, [_c.c_char_p, _c.c_int, _c.c_void_p, _c.c_int, _c.c_int, _c.c_char_p,
                                           _c.POINTER(_c.c_int)]),
    "lynx_plan_opt_timeline": (_c.c_void_p, [_c.c_char_p, _c.c_int, _c.c_void_p, _c.c_int, _c.c_int, _c.c_char_p,
                                             _c.c_char_p, _c.POINTER(_c.c_int)]),
}
_bound = False


def _lib():
    global _bound
    l = lib()
    if not _bound:
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _bound = True
    return l


def _call(name: str, *args, ok_codes=(0,)) -> tuple[str, int]:
    """Returns (text, status). Raises LynxError when no document was produced."""
    l = _lib()
    st = _c.c_int(0)
    ptr = getattr(l, name)(*args, _c.byref(st))
    if not ptr:
        raise LynxError(st.value, l.lynx_last_error().decode(errors="replace"))
    try:
        text = _c.cast(ptr, _c.c_char_p).value.decode()
    finally:
        l.lynx_free(ptr)
    return text, st.value


def _b(s: str | None) -> bytes | None:
    return None if s is None else s.encode()


def _layers(layers):
    if not layers:
        return None, 0
    arr = (_c.c_int * len(layers))(*layers)
    return _c.cast(arr, _c.c_void_p), len(layers)


# ------------------------------------------------------------------ text API
def validate_text(profile: str, lenient: bool = False) -> tuple[str, int]:
    return _call("lynx_plan_validate", _b(profile), int(lenient))


def serialize_profile_text(profile: str, lenient: bool = False) -> str:
    return _call("lynx_plan_serialize_profile", _b(profile), int(lenient))[0]


def schedule_text(profile: str, mode: str = "heu", stage: int = 0, layers_per_stage=None,
                  time_limit_ms: int = 10000, emit_lp: bool = False) -> tuple[str, int]:
    lp, n = _layers(layers_per_stage)
    return _call("lynx_plan_schedule", _b(profile), _b(mode), stage, lp, n, time_limit_ms, int(emit_lp))


def partition_text(profile: str, mode: str = "heu", time_limit_ms: int = 10000) -> str:
    return _call("lynx_plan_partition", _b(profile), _b(mode), time_limit_ms)[0]


def simulate_text(profile: str, mode: str = "heu", layers_per_stage=None, p2p_us: str = "0", fmt: str = "json",
                  pybind_semantics: bool = False, time_limit_ms: int = 10000) -> str:
    lp, n = _layers(layers_per_stage)
    f = {"json": 0, "csv": 1, "chrome-trace": 2, "report": 3}[fmt]
    return _call("lynx_plan_simulate", _b(profile), _b(mode), lp, n, _b(p2p_us), f, int(pybind_semantics),
                 time_limit_ms)[0]


def stage_plan_text(profile: str, stage: int, layers_per_stage=None, baseline: str = "heu",
                    time_limit_ms: int = 10000) -> dict:
    lp, n = _layers(layers_per_stage)
    b = {"heu": 0, "full": 1, "retain_all": 2, "selective": 3}[baseline]
    return json.loads(_call("lynx_plan_stage", _b(profile), stage, lp, n, b, time_limit_ms)[0])


def simulate_timelines_text(profile: str, layers_per_stage, timelines: list, p2p_us: str = "0") -> dict:
    lp, n = _layers(layers_per_stage)
    return json.loads(_call("lynx_plan_simulate_timelines", _b(profile), lp, n, _b(json.dumps(timelines)),
                            _b(p2p_us))[0])


def solve_heu_text(profile: str, stage: int, stage_layers: int, policy: int = 0, delta_bytes: str = "0",
                   time_limit_ms: int = 10000) -> dict:
    return json.loads(_call("lynx_plan_solve_heu", _b(profile), stage, stage_layers, policy, _b(delta_bytes),
                            time_limit_ms)[0])


def opt_export_text(profile: str, stage: int, layers_per_stage=None, slice_layers: int = 0,
                    reserve_bytes: str | None = None) -> dict:
    """The OPT program of a layer slice in matrix form (include/lynx_rt.h: lynx_plan_opt_export)."""
    lp, n = _layers(layers_per_stage)
    return json.loads(_call("lynx_plan_opt_export", _b(profile), stage, lp, n, slice_layers, _b(reserve_bytes))[0])


def opt_timeline_text(profile: str, stage: int, schedule: dict, layers_per_stage=None, slice_layers: int = 0,
                      reserve_bytes: str | None = None) -> tuple[dict, int]:
    """Exact check of a solver's schedule + its replayable stage timeline (lynx_plan_opt_timeline)."""
    lp, n = _layers(layers_per_stage)
    text, st = _call("lynx_plan_opt_timeline", _b(profile), stage, lp, n, slice_layers, _b(reserve_bytes),
                     _b(json.dumps(schedule)), ok_codes=(0, 1))
    return json.loads(text), st


# ------------------------------------------------ the reference's _lynx API
def _load(path: str, lenient: bool) -> str:
    text = Path(path).read_text()
    return serialize_profile_text(text, True) if lenient else text


def validate(path: str, lenient: bool = False) -> str:
    """Empty string when well-formed, else the diagnostics report (module.cpp:66-72)."""
    return validate_text(Path(path).read_text(), lenient)[0]


def schedule(path: str, mode: str = "heu", stage: int = 0, time_limit_ms: int = 10000, lenient: bool = False) -> str:
    text = _load(path, lenient)
    return schedule_text(text, mode, stage, None, time_limit_ms)[0]


def partition(path: str, mode: str = "heu", time_limit_ms: int = 10000, lenient: bool = False) -> str:
    return partition_text(_load(path, lenient), mode, time_limit_ms)


def simulate(path: str, mode: str = "heu", layers_per_stage=(), p2p_us: str = "0", time_limit_ms: int = 10000,
             lenient: bool = False) -> str:
    return simulate_text(_load(path, lenient), mode, list(layers_per_stage), p2p_us, "json",
                         pybind_semantics=True, time_limit_ms=time_limit_ms)


def serialize_profile(path: str, lenient: bool = False) -> str:
    return serialize_profile_text(Path(path).read_text(), lenient)
