"""Measurement helpers for bench.py: roofline arithmetic, peaks, clock sampling.

Roofline definitions:

* algorithmic bytes / element = Table-4 global accesses x sizeof(real)
  (36/66/52/80 reals, ``counts.py:61-76``);
* algorithmic flops / element = Table-4 QSS op total (290/2700/986/4806,
  ``counts.py:40-53``) for every variant;
* binding roof = the slower of bytes / HBM peak and flops / FP64 peak;
  ``frac`` = roof time / measured time.

HBM peak: ``MEASURED_PEAKS.json`` ``hbm_gbs`` (driver-measured copy bandwidth
on this pool's B200s), else the profiling guide's 6650 GB/s fallback.  FP64 /
FP32 peaks: measured on the box by ``tools/probe_peaks.py`` (independent
DFMA/FFMA chains on all SMs; ``profiles/peaks_r01.json``), else the nominal
148 SMs x 64 DFMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s (x2 for fp32).
"""

from __future__ import annotations

import json
import os
import statistics
import threading
import time

from .kernels.counts import algorithmic_bytes, algorithmic_flops
from .problems import ProblemClass
from .refelem import ElementType

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FALLBACK_HBM_GBS = 6650.0
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def hbm_peak() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def flop_peak(real_bytes: int = 8) -> tuple[float, str]:
    """Measured FMA-pipe peak (tools/probe_peaks.py -> profiles/peaks_r01.json), else nominal."""
    key = "fp64_tflops_best" if real_bytes == 8 else "fp32_tflops_best"
    path = os.path.join(ROOT, "profiles", "peaks_r01.json")
    try:
        with open(path) as fh:
            val = float(json.load(fh)[key])
        return val, f"measured (profiles/peaks_r01.json {key}, DFMA/FFMA chains on 148 SMs)"
    except Exception:
        nominal = NOMINAL_FP64_TFLOPS * (1 if real_bytes == 8 else 2)
        return nominal, "nominal (148 SM x 64 DFMA/clk x 2 x 1.965 GHz; x2 for fp32)"


def case_roofline(element: ElementType, problem: ProblemClass, n: int, seconds: float, real_bytes: int = 8) -> dict:
    """Roofline record for n elements integrated in ``seconds`` (one launch)."""
    hbm, hbm_src = hbm_peak()
    peak_f, fp64_source = flop_peak(real_bytes)
    by = algorithmic_bytes(element, problem, real_bytes) * n
    fl = algorithmic_flops(element, problem) * n
    t_mem = by / (hbm * 1e9)
    t_flop = fl / (peak_f * 1e12)
    both = {"hbm_frac": t_mem / seconds, "flop_frac": t_flop / seconds}
    if t_flop / seconds > 1.0:
        # the QSS prism kernels contract in the reference frame and
        # execute fewer FP64 operations than Table 4 counts
        both["note"] = ("flops are the Table-4 model count; the kernel executes fewer, so the model-flop "
                        "fraction exceeds 1 and hbm_frac is the bound left to approach")
    if t_mem >= t_flop:
        return {"bound": "hbm", "achieved": by / seconds / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": t_mem / seconds, "peak_source": hbm_src,
                "bytes_per_launch": by, "flops_per_launch": fl, **both}
    return {"bound": "fp64" if real_bytes == 8 else "fp32", "achieved": fl / seconds / 1e12, "peak": peak_f,
            "unit": "TFLOP/s", "frac": t_flop / seconds, "peak_source": fp64_source,
            "bytes_per_launch": by, "flops_per_launch": fl, **both}


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, sampled in a thread)
# ---------------------------------------------------------------------------

_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """Samples SM clock and clock-event reasons every ``period`` seconds."""

    def __init__(self, device_index: int, period: float = 0.002):
        self.period = period
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # pragma: no cover - depends on the box
            self.error = f"nvml unavailable: {exc}"
            self._nvml = None

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((mhz, reasons))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nvml is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join()

    def summary(self) -> dict:
        if self._nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": getattr(self, "error", "nvml unavailable")}
        busy = [m for m, r in self.samples if not (r & 0x1)] or [m for m, _ in self.samples]
        mask = 0
        for _, r in self.samples:
            mask |= r
        reasons = sorted(name for bit, name in _REASONS.items() if mask & bit and bit != 0x1)
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def clocks_rejected(clocks: dict) -> str | None:
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(clocks.get("reasons", []))
    if bad:
        return "throttled: " + ",".join(sorted(bad))
    mhz, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    if mhz and mx and mhz < 0.6 * mx and "sw_power_cap" not in clocks.get("reasons", []):
        return f"sm clock {mhz} MHz far below max {mx} MHz with no reason"
    return None
