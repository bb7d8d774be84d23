"""Which NVML NVLink byte counters does this driver expose?  Prints, per field
and for scope ids 0 (and link 0..2), the NVML return code and value, plus the
output of `nvidia-smi nvlink -h` (development aid)."""
import subprocess

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name in sorted(n for n in dir(pynvml) if n.startswith("NVML_FI_DEV_NVLINK_") and ("BYTES" in n or "THROUGHPUT" in n
                                                                                     or "PACKETS" in n)):
    fid = getattr(pynvml, name)
    for scope in (0, 1, 2, 0xFFFFFFFF):
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            val = v.value.ullVal if v.nvmlReturn == 0 else None
            print(f"{name} scope {scope:#x}: ret {v.nvmlReturn} value {val}")
        except Exception as e:  # noqa: BLE001
            print(f"{name} scope {scope:#x}: {type(e).__name__} {e}")
for cmd in (["nvidia-smi", "nvlink", "-h"], ["nvidia-smi", "nvlink", "-s", "-i", "0"],
            ["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"]):
    r = subprocess.run(cmd, capture_output=True, text=True)
    print("$", " ".join(cmd), "rc", r.returncode)
    print(r.stdout[-3000:], r.stderr[-500:])
