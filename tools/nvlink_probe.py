"""Print what NVML reports for the NVLink data counters on GPU 0 (probe)."""
import pynvml as N
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
for name in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX",
             "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_LINK_COUNT"):
    fid = getattr(N, name, None)
    if fid is None:
        continue
    for scope in (0, 1, 17, 0xFFFFFFFF):
        try:
            v = N.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, scope, v.nvmlReturn, v.valueType, v.value.ullVal)
        except Exception as e:
            print(name, scope, "exc", e)
try:
    for link in range(18):
        st = N.nvmlDeviceGetNvLinkState(h, link)
        print("link", link, "state", st)
except Exception as e:
    print("link state exc", e)
