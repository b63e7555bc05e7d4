"""TEST INFRASTRUCTURE ONLY — Python handle on the parity oracle.

`oracle/_ref/` holds the reference's own, unmodified lynx_core compiled by
oracle/Makefile (Boost/GTest/CLI11 shims in oracle/shim/). Its correctness is
pinned by the reference's own suites, which all pass against this build
(`make -C oracle check pycheck`: 98 unit tests, acceptance C1-C11, Python smoke).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module; the product never does.

    RefLib      ctypes wrapper of _ref/liblynx_ref.so (oracle/ref_capi.cpp)
    ref_module  the reference's own pybind `_lynx` module (bindings/module.cpp)
    ref_cli     path of the reference CLI binary (tools/lynx_main.cpp)
"""
from __future__ import annotations

import ctypes
import importlib.util
import json
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
LIB = REF_DIR / "liblynx_ref.so"
CLI = REF_DIR / "lynx"
REFERENCE_SRC = Path("/root/reference/proj")


def available() -> bool:
    return LIB.exists()


def build(quiet: bool = True) -> bool:
    """Build the oracle when the reference sources are present (this container only)."""
    if not REFERENCE_SRC.exists():
        return available()
    r = subprocess.run(["make", "-C", str(HERE), "-j8", "all", "pymodule"], capture_output=quiet, text=True)
    return r.returncode == 0 and available()


class RefLib:
    def __init__(self):
        self.l = ctypes.CDLL(str(LIB))
        c = ctypes
        vp, cp, i, ll = c.c_void_p, c.c_char_p, c.c_int, c.c_longlong
        sig = {
            "lynx_ref_last_error": (cp, []),
            "lynx_ref_free": (None, [vp]),
            "lynx_ref_serialize_profile": (vp, [cp, i]),
            "lynx_ref_stage_plan": (vp, [cp, i, vp, i, ll]),
            "lynx_ref_fixed_plan": (vp, [cp, i, vp, i, i]),
            "lynx_ref_solve_heu": (vp, [cp, i, i, i, cp, ll]),
            "lynx_ref_partition": (vp, [cp, ll]),
            "lynx_ref_simulate": (vp, [cp, vp, i, cp, i, ll]),
            "lynx_ref_simulate_timelines": (vp, [cp, vp, i, cp, cp]),
            "lynx_ref_stage_period": (vp, [cp, i, i, cp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(self.l, n)
            f.restype = r
            f.argtypes = a

    def _s(self, ptr) -> str:
        if not ptr:
            raise RuntimeError("oracle: " + self.l.lynx_ref_last_error().decode())
        try:
            return ctypes.cast(ptr, ctypes.c_char_p).value.decode()
        finally:
            self.l.lynx_ref_free(ptr)

    @staticmethod
    def _layers(layers):
        if not layers:
            return None, 0
        a = (ctypes.c_int * len(layers))(*layers)
        return ctypes.cast(a, ctypes.c_void_p), len(layers)

    def stage_plan(self, profile: str, stage: int, layers=None, time_limit_ms: int = 10000) -> dict:
        lp, n = self._layers(layers)
        return json.loads(self._s(self.l.lynx_ref_stage_plan(profile.encode(), stage, lp, n, time_limit_ms)))

    def fixed_plan(self, profile: str, stage: int, layers=None, retain_all: bool = False) -> dict:
        lp, n = self._layers(layers)
        return json.loads(self._s(self.l.lynx_ref_fixed_plan(profile.encode(), stage, lp, n, int(retain_all))))

    def solve_heu(self, profile: str, stage: int, stage_layers: int, policy: int = 0, delta: str = "0",
                  time_limit_ms: int = 10000) -> dict:
        return json.loads(self._s(self.l.lynx_ref_solve_heu(profile.encode(), stage, stage_layers, policy,
                                                            delta.encode(), time_limit_ms)))

    def partition(self, profile: str, time_limit_ms: int = 10000) -> str:
        return self._s(self.l.lynx_ref_partition(profile.encode(), time_limit_ms))

    def simulate(self, profile: str, layers=None, p2p_us: str = "0", fmt: int = 0, time_limit_ms: int = 10000) -> str:
        lp, n = self._layers(layers)
        return self._s(self.l.lynx_ref_simulate(profile.encode(), lp, n, p2p_us.encode(), fmt, time_limit_ms))

    def simulate_timelines(self, profile: str, layers, timelines: list, p2p_us: str = "0") -> dict:
        lp, n = self._layers(layers)
        return json.loads(self._s(self.l.lynx_ref_simulate_timelines(profile.encode(), lp, n,
                                                                     json.dumps(timelines).encode(),
                                                                     p2p_us.encode())))

    def stage_period(self, profile: str, stage: int, stage_layers: int, timeline: dict) -> str:
        return self._s(self.l.lynx_ref_stage_period(profile.encode(), stage, stage_layers,
                                                    json.dumps(timeline).encode()))


def ref_module():
    """The reference's own pybind `_lynx` module, built in oracle/_ref."""
    cands = sorted(REF_DIR.glob("_lynx*.so"))
    if not cands:
        raise ImportError("oracle/_ref/_lynx*.so not built")
    spec = importlib.util.spec_from_file_location("_lynx", cands[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def run_cli(*args: str) -> tuple[int, str]:
    r = subprocess.run([str(CLI), *args], capture_output=True, text=True)
    return r.returncode, r.stdout
