"""NVLink byte counters of one GPU through NVML (nvidia-ml-py), summed over
its links: data / raw throughput counters (KiB) and the NVLink-5 transmit /
receive byte counters.  Used around a timed region to report the wire bytes
an exchange moved per call beside its algorithmic bytes.  Returns None for
counters this driver does not expose."""
import pynvml

FIELDS = {
    "data_tx": pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,  # KiB
    "data_rx": pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
    "raw_tx": pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX,
    "raw_rx": pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX,
    "xmit_bytes": pynvml.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,  # bytes
    "rcv_bytes": pynvml.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES,
}
_KIB = {"data_tx", "data_rx", "raw_tx", "raw_rx"}
_init = False


def _handle(index):
    global _init
    if not _init:
        pynvml.nvmlInit()
        _init = True
    return pynvml.nvmlDeviceGetHandleByIndex(index)


def read(index, links=18):
    """{counter: bytes summed over links} for GPU `index` (None if unsupported)."""
    h = _handle(index)
    out = {}
    for name, fid in FIELDS.items():
        total, ok = 0, False
        for link in range(links):
            try:
                v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
            except Exception:
                break
            if v.nvmlReturn != 0:
                continue
            ok = True
            raw = v.value.ullVal if hasattr(v.value, "ullVal") else int(v.value)
            total += raw * (1024 if name in _KIB else 1)
        out[name] = total if ok else None
    return out


def delta(before, after):
    return {k: (after[k] - before[k]) if before.get(k) is not None and after.get(k) is not None else None
            for k in before}
