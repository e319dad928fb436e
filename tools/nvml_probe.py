"""Which NVML NVLink byte counters does this driver expose? (for bench.py's nvlink key)"""
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
print("driver", nv.nvmlSystemGetDriverVersion())
for l in range(18):
    try:
        print("link", l, "state", nv.nvmlDeviceGetNvLinkState(h, l))
    except Exception as e:
        print("link", l, "state err", e)
        break
for name in ["NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX",
             "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES"]:
    fid = getattr(nv, name)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, scope, "ret", v.nvmlReturn, "val", v.value.ullVal, "type", v.valueType)
        except Exception as e:
            print(name, scope, "exc", e)
    try:
        v = nv.nvmlDeviceGetFieldValues(h, [fid])[0]
        print(name, "noscope ret", v.nvmlReturn, "val", v.value.ullVal)
    except Exception as e:
        print(name, "noscope exc", e)
