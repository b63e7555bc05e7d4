"""SM clock and throttle-reason sampling through NVML during a timed region (bench.py, the stage
emulation, tools). In-process: an nvidia-smi subprocess per sample perturbs the step."""
from __future__ import annotations

import statistics
import threading


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 200 ms during the timed region
    (in-process; an nvidia-smi subprocess per sample perturbs the step)."""

    def __init__(self, gpu: int = 0):
        self.gpu = gpu
        self.rows: list[tuple] = []
        self._stop = threading.Event()
        self._t = None
        self._nv = self._hnd = self._mx = None
        self._err = None
        # NVML is initialised here, before the warm-up steps: nvmlInit running concurrently with the
        # first timed step stalled it by up to 1.3 s (driver-level contention).
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv, self._hnd = nv, nv.nvmlDeviceGetHandleByIndex(gpu)
            self._mx = nv.nvmlDeviceGetMaxClockInfo(self._hnd, nv.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self._err = str(e)

    def _run(self):
        if self._err is not None:  # pragma: no cover
            self.rows.append(("error", self._err))
            return
        nv, hnd, mx = self._nv, self._hnd, self._mx
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(hnd, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(hnd)
                self.rows.append((sm, mx, rs))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self) -> dict:
        rows = [r for r in self.rows if r and r[0] != "error"]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        bits = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
        reasons = sorted({name for r in rows for bit, name in bits.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "source": "NVML"}
