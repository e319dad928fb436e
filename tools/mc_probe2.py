"""NVLS multicast plumbing probe: which shareable handle types work for multicast objects and physical memory
(FABRIC: a 64-byte blob any process can import; POSIX_FD: needs fd passing), and does pidfd_getfd work here."""
import ctypes
import os
from cuda.bindings import driver as d

d.cuInit(0)
dev = d.cuDeviceGet(0)[1]
ctx = d.cuDevicePrimaryCtxRetain(dev)[1]
d.cuCtxSetCurrent(ctx)
n = d.cuDeviceGetCount()[1]
for attr in ["CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED"]:
    a = getattr(d.CUdevice_attribute, attr, None)
    print(attr, d.cuDeviceGetAttribute(a, dev) if a is not None else "n/a")
for ht in ["CU_MEM_HANDLE_TYPE_FABRIC", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR"]:
    prop = d.CUmulticastObjectProp()
    prop.numDevices = n
    prop.size = 1 << 21
    prop.handleTypes = getattr(d.CUmemAllocationHandleType, ht)
    r = d.cuMulticastCreate(prop)
    print("mc create", ht, r[0])
    if r[0] == d.CUresult.CUDA_SUCCESS:
        e = d.cuMemExportToShareableHandle(r[1], getattr(d.CUmemAllocationHandleType, ht), 0)
        print("  export", e[0], type(e[1]) if len(e) > 1 else None)
    ap = d.CUmemAllocationProp()
    ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    ap.location.id = 0
    ap.requestedHandleTypes = getattr(d.CUmemAllocationHandleType, ht)
    m = d.cuMemCreate(1 << 21, ap, 0)
    print("mem create", ht, m[0])
# pidfd_getfd of our own fd 0 through our own pid
libc = ctypes.CDLL(None, use_errno=True)
SYS_pidfd_open, SYS_pidfd_getfd = 434, 438
pfd = libc.syscall(SYS_pidfd_open, os.getpid(), 0)
print("pidfd_open", pfd, ctypes.get_errno())
if pfd >= 0:
    r = libc.syscall(SYS_pidfd_getfd, pfd, 1, 0)
    print("pidfd_getfd", r, ctypes.get_errno())
print("ptrace_scope", open("/proc/sys/kernel/yama/ptrace_scope").read().strip() if os.path.exists("/proc/sys/kernel/yama/ptrace_scope") else "n/a")
print("CapEff", [l for l in open("/proc/self/status") if l.startswith("CapEff")])
