"""Which NVML NVLink byte counters does this box expose?  Prints, per visible
GPU, the active links and the raw values of the throughput / byte-count
fields (aggregate and per link), so bench.py's NVLink traffic reader can use
the ones that work here."""
import json

import pynvml as nv

FIELDS = {
    "THROUGHPUT_DATA_TX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
    "THROUGHPUT_DATA_RX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
    "THROUGHPUT_RAW_TX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX,
    "THROUGHPUT_RAW_RX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX,
    "COUNT_XMIT_BYTES": nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
    "COUNT_RCV_BYTES": nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES,
}


def main():
    nv.nvmlInit()
    out = []
    for i in range(nv.nvmlDeviceGetCount()):
        h = nv.nvmlDeviceGetHandleByIndex(i)
        d = {"gpu": i, "name": nv.nvmlDeviceGetName(h)}
        links = []
        for l in range(18):
            try:
                links.append((l, int(nv.nvmlDeviceGetNvLinkState(h, l))))
            except nv.NVMLError as e:
                links.append((l, str(e)))
        d["links"] = links
        vals = {}
        for name, fid in FIELDS.items():
            for scope in (0xFFFFFFFF, 0, 1):
                try:
                    v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                    vals[f"{name}@{scope:#x}"] = (int(v.nvmlReturn), int(v.valueType), int(v.value.ullVal))
                except Exception as e:
                    vals[f"{name}@{scope:#x}"] = str(e)
        d["fields"] = vals
        out.append(d)
    print(json.dumps(out, indent=1))


def gpm():
    """GPM (GPU performance monitoring) NVLink totals between two samples."""
    import time

    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    res = {}
    try:
        res["supported"] = int(nv.nvmlGpmQueryDeviceSupport(h).isSupportedDevice)
        s1, s2 = nv.nvmlGpmSampleAlloc(), nv.nvmlGpmSampleAlloc()
        nv.nvmlGpmSampleGet(h, s1)
        time.sleep(0.2)
        nv.nvmlGpmSampleGet(h, s2)
        mg = nv.c_nvmlGpmMetricsGet_t()
        mg.version = nv.NVML_GPM_METRICS_GET_VERSION
        mg.sample1, mg.sample2 = s1, s2
        ids = [nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC, nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC,
               nv.NVML_GPM_METRIC_NVLINK_L0_TX, nv.NVML_GPM_METRIC_NVLINK_L0_TX_PER_SEC]
        mg.numMetrics = len(ids)
        for i, m in enumerate(ids):
            mg.metrics[i].metricId = m
        nv.nvmlGpmMetricsGet(mg)
        res["metrics"] = [(int(mg.metrics[i].metricId), int(mg.metrics[i].nvmlReturn), mg.metrics[i].value)
                          for i in range(len(ids))]
    except Exception as e:
        res["error"] = repr(e)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
    gpm()
