"""NVML sampler for the profiling tools: median SM clock (MHz) and power (W) while a block of work runs."""
import statistics
import threading
import time


class Clock:
    def __init__(self, index=0, period_s=0.005):
        self.index, self.period = index, period_s
        self.sm, self.pw = [], []
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nv = pynvml
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _run(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.pw.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)
        return False

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "power_w": None}
        return {"sm_mhz": statistics.median(self.sm), "power_w": statistics.median(self.pw), "samples": len(self.sm)}
