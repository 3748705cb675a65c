"""NVLink traffic from the GPU's own counters (NVML), read around a pass of the kernel.

ncu cannot profile the multi-GPU kernel (its replay would re-run a kernel whose CTAs wait on
flags that other ranks write; B200_PROFILING.md: never wrap a multi-rank command in ncu), so the
NVLink half of the roofline evidence (north star: "NVLink GB/s against 900 GB/s per direction")
comes from counters NVML exposes, whichever the driver answers:

* GPM (``nvmlGpmSampleGet`` twice + ``nvmlGpmMetricsGet``): ``NVLINK_TOTAL_TX/RX_PER_SEC``
  (MiB/s over all links between the two samples; bytes = rate × the host time between them);
* field values ``NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES`` (202 / 204, bytes) and
  ``NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX`` (138 / 139, KiB), per link (scope id = link)
  and aggregated (scope id 0xFFFFFFFF).

``NvlCounters.begin()`` / ``end()`` bracket a region and return ``{name: bytes}`` for every
source that answered; ``summarize`` turns that into per-direction bytes per step.
``python tools/nvlcounters.py`` copies 8 GiB GPU0 -> GPU1 and reports what answered.

Result on this pool's B200 boxes (profiles/round1/nvlink/nvml_counters_probe.json): every
field returns NVML_ERROR_NOT_SUPPORTED (3), GPM sampling fails, and ``nvidia-smi nvlink -gt d``
prints N/A for every link — the link counters are not exposed to tenants here, so bench.py
does not use them and the NVLink roofline stays algorithmic bytes / kernel time.
"""
import json
import sys
import time

FIELDS = {"xmit_bytes": (202, 1), "rcv_bytes": (204, 1), "data_tx_kib": (138, 1024), "data_rx_kib": (139, 1024)}
MAX_LINKS = 18
ALL_LINKS = 0xFFFFFFFF
GPM_RX, GPM_TX = 60, 61   # NVML_GPM_METRIC_NVLINK_TOTAL_{RX,TX}_PER_SEC (MiB/s)


class NvlCounters:
    def __init__(self, index):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.keys = [(name, link) for name in FIELDS for link in list(range(MAX_LINKS)) + [ALL_LINKS]]
        self.errors = {}
        self.gpm = None
        try:
            if pynvml.nvmlGpmQueryDeviceSupport(self.h).isSupportedDevice:
                self.gpm = (pynvml.nvmlGpmSampleAlloc(), pynvml.nvmlGpmSampleAlloc())
        except Exception as e:
            self.errors["gpm"] = str(e)[:80]

    def _fields(self):
        out = {}
        try:
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, [(FIELDS[n][0], l) for n, l in self.keys])
        except Exception as e:
            self.errors["fields"] = str(e)[:80]
            return out
        for key, v in zip(self.keys, vals):
            if v.nvmlReturn == 0:
                out[key] = int(v.value.ullVal)
            else:
                self.errors.setdefault(f"field {key[0]}", int(v.nvmlReturn))
        return out

    def begin(self):
        self.f0 = self._fields()
        if self.gpm:
            try:
                self.nv.nvmlGpmSampleGet(self.h, self.gpm[0])
            except Exception as e:
                self.errors["gpm"] = str(e)[:80]
                self.gpm = None
        self.t0 = time.perf_counter()

    def end(self):
        t1 = time.perf_counter()
        tot = {}
        if self.gpm:
            try:
                self.nv.nvmlGpmSampleGet(self.h, self.gpm[1])
                mg = self.nv.c_nvmlGpmMetricsGet_t()
                mg.version = self.nv.NVML_GPM_METRICS_GET_VERSION
                mg.numMetrics = 2
                mg.sample1, mg.sample2 = self.gpm
                mg.metrics[0].metricId, mg.metrics[1].metricId = GPM_TX, GPM_RX
                self.nv.nvmlGpmMetricsGet(mg)
                dt = time.perf_counter() - self.t0
                for i, name in ((0, "gpm_tx"), (1, "gpm_rx")):
                    if mg.metrics[i].nvmlReturn == 0:
                        tot[name] = int(mg.metrics[i].value * (1 << 20) * dt)
                    else:
                        self.errors[name] = int(mg.metrics[i].nvmlReturn)
                tot["gpm_window_s"] = dt
            except Exception as e:
                self.errors["gpm"] = str(e)[:80]
        f1 = self._fields()
        for key, v1 in f1.items():
            if key in self.f0:
                name = key[0] + ("_all" if key[1] == ALL_LINKS else "")
                tot[name] = tot.get(name, 0) + (v1 - self.f0[key]) * FIELDS[key[0]][1]
        tot["host_window_s"] = t1 - self.t0
        return tot


PAIRS = (("xmit_bytes", "rcv_bytes"), ("data_tx_kib", "data_rx_kib"), ("xmit_bytes_all", "rcv_bytes_all"),
         ("data_tx_kib_all", "data_rx_kib_all"), ("gpm_tx", "gpm_rx"))


def summarize(delta, steps, algorithmic_per_step):
    """Per-direction NVLink bytes per step from ``end()``'s totals: the first counter pair that
    moved, exact byte counters before the GPM rate × window estimate."""
    for tx, rx in PAIRS:
        if tx in delta and rx in delta and (delta[tx] or delta[rx]):
            t, r = delta[tx] // max(steps, 1), delta[rx] // max(steps, 1)
            return {"counters": f"nvml {tx}/{rx}", "tx_bytes_per_step": t, "rx_bytes_per_step": r,
                    "per_direction_vs_algorithmic": round(max(t, r) / algorithmic_per_step, 4),
                    "steps_counted": steps, "all": delta}
    return {"counters": "none answered", "all": delta}


def main():
    import torch
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    nbytes, reps = 1 << 30, 8
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    c0, c1 = NvlCounters(0), NvlCounters(1)
    c0.begin()
    c1.begin()
    t0 = time.perf_counter()
    for _ in range(reps):
        b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    secs = time.perf_counter() - t0
    d0, d1 = c0.end(), c1.end()
    print(json.dumps({"probe": "nvlcounters", "copied_bytes": nbytes * reps, "seconds": secs,
                      "copy_gbs": round(nbytes * reps / secs / 1e9, 1), "gpu0": d0, "gpu1": d1,
                      "gpu0_summary": summarize(d0, reps, nbytes), "errors": c0.errors}), flush=True)
    sys.exit(0)


if __name__ == "__main__":
    main()
