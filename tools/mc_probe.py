"""Does this box support NVLink SHARP multicast (NVLS: multimem.* through the NVSwitch)? Device attribute plus an
actual cuMulticastCreate over all visible GPUs (single process)."""
from cuda.bindings import driver as d


def ok(r):
    return r[0] if isinstance(r, tuple) else r


d.cuInit(0)
n = d.cuDeviceGetCount()[1]
for i in range(n):
    dev = d.cuDeviceGet(i)[1]
    print("dev", i, "multicast_supported", d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
prop = d.CUmulticastObjectProp()
prop.numDevices = n
prop.size = 1 << 21
prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
print("granularity", d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
r = d.cuMulticastCreate(prop)
print("cuMulticastCreate", r)
