"""Host-side telemetry around a timed region (NVML): SM clocks + throttle
reasons, and the bytes that actually crossed this GPU's NVLink ports.

Neither touches the data path; bench.py and the tools use them to make a
measurement self-evidencing (SURVEY.md §5 "Tracing/profiling")."""
from __future__ import annotations

import statistics
import threading
import time
from typing import Optional


def _nvml():
    import pynvml

    pynvml.nvmlInit()
    return pynvml


def _handle(nv, device: int):
    """The NVML handle of CUDA device `device`, matched by PCI address: NVML
    enumerates every GPU of the host in bus order while CUDA numbers only the
    visible ones (CUDA_VISIBLE_DEVICES), so the indices need not agree."""
    try:
        import torch

        pr = torch.cuda.get_device_properties(device)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        return nv.nvmlDeviceGetHandleByPciBusId(bus)
    except Exception:
        return nv.nvmlDeviceGetHandleByIndex(device)


class ClockSampler:
    """NVML sampling of the SM clock and the clock-event (throttle) reasons
    every 5 ms while the context is open."""

    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            nv = _nvml()
            self._nv = nv
            self._h = _handle(nv, device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.BITS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def merge_clocks(summaries) -> dict:
    """Combine per-rank ClockSampler summaries: the slowest rank's median clock,
    the union of throttle reasons."""
    got = [s for s in summaries if s and s.get("sm_mhz") is not None]
    if not got:
        return summaries[0] if summaries else {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
    worst = min(got, key=lambda s: s["sm_mhz"])
    return {"sm_mhz": worst["sm_mhz"], "sm_max_mhz": worst["sm_max_mhz"],
            "reasons": sorted({r for s in got for r in s["reasons"]}),
            "samples": sum(s["samples"] for s in got), "ranks": len(summaries),
            "sm_mhz_per_rank": [s.get("sm_mhz") for s in summaries]}


class NvlinkMeter:
    """Bytes this GPU transmitted / received over NVLink between start() and
    stop(), read from NVML.  Sources, first that works on the box:

    1. per-link byte counters (NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES /
       _RCV_BYTES, scope = link id) summed over active links;
    2. aggregate data throughput counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX
       / _RX, KiB);
    3. GPM (NVML_GPM_METRIC_NVLINK_TOTAL_TX/RX_PER_SEC) between two samples,
       times the host interval between them.

    Virtualised boxes often report NVML_ERROR_NOT_SUPPORTED for all three;
    then `result()` carries `tx_bytes: None` and the reason."""

    MAX_LINKS = 18

    def __init__(self, device: int):
        self.device = device
        self.source: Optional[str] = None
        self.error: Optional[str] = None
        self._t0 = self._t1 = None
        self._a = self._b = None
        try:
            nv = _nvml()
            self._nv = nv
            self._h = _handle(nv, device)
        except Exception as e:
            self._nv, self.error = None, f"NVML unavailable: {e!r}"[:200]
            return
        self.links = []
        for l in range(self.MAX_LINKS):
            try:
                if int(nv.nvmlDeviceGetNvLinkState(self._h, l)) == 1:
                    self.links.append(l)
            except Exception:
                pass
        for name, probe in (("nvml_link_byte_counters", self._read_links),
                            ("nvml_throughput_data_kib", self._read_throughput),
                            ("nvml_gpm_total_per_sec", self._gpm_probe)):
            try:
                if probe() is not None:
                    self.source = name
                    break
            except Exception as e:
                self.error = f"{name}: {e!r}"[:200]
        if self.source is None and self.error is None:
            self.error = "no NVLink byte counter supported by NVML on this box (NVML_ERROR_NOT_SUPPORTED)"

    # -- sources ------------------------------------------------------------
    def _fields(self, ids):
        vals = self._nv.nvmlDeviceGetFieldValues(self._h, ids)
        out = []
        for v in vals:
            if int(v.nvmlReturn) != 0:
                return None
            out.append(int(v.value.ullVal))
        return out

    def _read_links(self):
        if not self.links:
            return None
        nv = self._nv
        ids = [(nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, l) for l in self.links] + \
              [(nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, l) for l in self.links]
        v = self._fields(ids)
        if v is None:
            return None
        k = len(self.links)
        return sum(v[:k]), sum(v[k:])

    def _read_throughput(self):
        nv = self._nv
        v = self._fields([(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF),
                          (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)])
        return None if v is None else (v[0] * 1024, v[1] * 1024)

    def _gpm_sample(self):
        s = self._nv.nvmlGpmSampleAlloc()
        self._nv.nvmlGpmSampleGet(self._h, s)
        return s

    def _gpm_probe(self):
        nv = self._nv
        if not int(nv.nvmlGpmQueryDeviceSupport(self._h).isSupportedDevice):
            return None
        a = self._gpm_sample()
        time.sleep(0.01)
        b = self._gpm_sample()
        r = self._gpm_rates(a, b)
        nv.nvmlGpmSampleFree(a)
        nv.nvmlGpmSampleFree(b)
        return r

    def _gpm_rates(self, a, b):
        nv = self._nv
        mg = nv.c_nvmlGpmMetricsGet_t()
        mg.version = nv.NVML_GPM_METRICS_GET_VERSION
        mg.sample1, mg.sample2 = a, b
        mg.numMetrics = 2
        mg.metrics[0].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        mg.metrics[1].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        nv.nvmlGpmMetricsGet(mg)
        if int(mg.metrics[0].nvmlReturn) != 0 or int(mg.metrics[1].nvmlReturn) != 0:
            return None
        # GPM reports MiB/s for the NVLink totals
        return mg.metrics[0].value * 2 ** 20, mg.metrics[1].value * 2 ** 20

    # -- region ---------------------------------------------------------------
    def _read(self):
        if self.source == "nvml_link_byte_counters":
            return self._read_links()
        if self.source == "nvml_throughput_data_kib":
            return self._read_throughput()
        if self.source == "nvml_gpm_total_per_sec":
            return self._gpm_sample()
        return None

    def start(self) -> None:
        self._t0 = time.perf_counter()
        self._a = self._read() if self.source else None

    def stop(self) -> None:
        self._b = self._read() if self.source else None
        self._t1 = time.perf_counter()

    def result(self) -> dict:
        out = {"source": self.source, "device": self.device, "tx_bytes": None, "rx_bytes": None}
        if self.source is None or self._a is None or self._b is None:
            out["error"] = self.error or "not sampled"
            return out
        if self.source == "nvml_gpm_total_per_sec":
            r = self._gpm_rates(self._a, self._b)
            self._nv.nvmlGpmSampleFree(self._a)
            self._nv.nvmlGpmSampleFree(self._b)
            if r is None:
                out["error"] = "GPM metrics unavailable"
                return out
            dt = self._t1 - self._t0
            out["tx_bytes"], out["rx_bytes"] = int(r[0] * dt), int(r[1] * dt)
            out["interval_s"] = round(dt, 6)
        else:
            out["tx_bytes"], out["rx_bytes"] = self._b[0] - self._a[0], self._b[1] - self._a[1]
        return out


class EnergyMeter:
    """Board energy between start() and stop() from NVML's cumulative energy
    counter (mJ since driver load), with the enforced power limit.  Used to
    state a power roofline: a kernel whose mean board power sits at the limit
    cannot run faster than (joules per launch) / limit at that energy per
    launch, so its speed is set by energy per FLOP or byte, not by the pipe."""

    def __init__(self, device: int):
        self.device = device
        self.error: Optional[str] = None
        self.limit_w: Optional[float] = None
        self._e0 = self._e1 = None
        self._t0 = self._t1 = None
        try:
            nv = _nvml()
            self._nv = nv
            self._h = _handle(nv, device)
            self.limit_w = nv.nvmlDeviceGetEnforcedPowerLimit(self._h) / 1e3
            nv.nvmlDeviceGetTotalEnergyConsumption(self._h)
        except Exception as e:
            self._nv, self.error = None, f"NVML energy counter unavailable: {e!r}"[:200]

    def start(self) -> None:
        self._t0 = time.perf_counter()
        if self._nv is not None:
            self._e0 = self._nv.nvmlDeviceGetTotalEnergyConsumption(self._h)

    def stop(self) -> None:
        if self._nv is not None:
            self._e1 = self._nv.nvmlDeviceGetTotalEnergyConsumption(self._h)
        self._t1 = time.perf_counter()

    def joules(self) -> Optional[float]:
        if self._e0 is None or self._e1 is None:
            return None
        return (self._e1 - self._e0) / 1e3

    def measure(self, fn, calls: int, sync) -> dict:
        """Energy of `calls` back-to-back calls of fn (asynchronous launches;
        `sync` waits for them).  Returns joules per call, mean board watts over
        the region, the limit, and whether the region ran at the cap."""
        sync()
        self.start()
        for _ in range(calls):
            fn()
        sync()
        self.stop()
        j, dt = self.joules(), self._t1 - self._t0
        if j is None:
            return {"error": self.error or "no energy reading"}
        w = j / dt
        return {"calls": calls, "seconds": round(dt, 3), "joules_per_call": round(j / calls, 4),
                "board_w": round(w, 1), "limit_w": self.limit_w,
                "at_cap": bool(self.limit_w and w >= 0.95 * self.limit_w)}
