// NVLink SHARP (NVLS) multicast for the average fan-out of the push exchange (LSGD_B200_NVLS=1).
//
// The owner of slot j of group g pushes the slot's average to the k members' gfull. Unicast that is k-1 NVLink
// stores per element (egress (k-1)*S per owner); through an NVSwitch multicast object bound to the k members'
// gfull buffers it is ONE multimem.st per element: the switch replicates it to every member (egress S). A pure
// copy, so the bits are those of the unicast push (no in-switch arithmetic — the reference's summation order is
// kept by the owner's ordered sums).
//
// Object lifecycle (driver API, cuMulticast* / cuMem*): the group leader creates the multicast object; every member
// adds its device, and only when all k have (a barrier) allocates its gfull as physical memory (cuMemCreate), binds
// it to the object and maps both its local view and the multicast view. Processes share the object as a POSIX file
// descriptor the members duplicate from the leader (pidfd_getfd); threads of one process share the handle.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdint>
#include <string>

#include "common.hpp"
#include "nvls.hpp"

namespace lsgd_b200 {

namespace {

// Driver entry points resolved at run time (cudaGetDriverEntryPoint), never linked: the library must load where
// there is no driver (the CPU build / test container) and fail only when NVLS is actually used.
template <typename F>
F drv(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  LSGD_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
  check<Error>(p != nullptr && q == cudaDriverEntryPointSuccess, "CUDA driver entry point ", name, " unavailable");
  return reinterpret_cast<F>(p);
}
#define LSGD_DRV(fn) (drv<decltype(&fn)>(#fn))

std::string cu_error(CUresult r) {
  const char* s = nullptr;
  static auto get = LSGD_DRV(cuGetErrorString);
  get(r, &s);
  return s ? s : "?";
}

}  // namespace

#define LSGD_CU(fn, ...)                                                                                        \
  do {                                                                                                          \
    static auto fp_ = LSGD_DRV(fn);                                                                             \
    CUresult r_ = fp_(__VA_ARGS__);                                                                             \
    if (r_ != CUDA_SUCCESS)                                                                                     \
      throw ::lsgd_b200::Error(::lsgd_b200::cat("CUDA driver error ", cu_error(r_), " (", static_cast<int>(r_), \
                                                ") at ", __FILE__, ":", __LINE__, " (", #fn, ")"));             \
  } while (0)

namespace {
CUmulticastObjectProp mc_prop(size_t size, int n_devices) {
  CUmulticastObjectProp p{};
  p.numDevices = static_cast<unsigned int>(n_devices);
  p.size = size;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  p.flags = 0;
  return p;
}
size_t round_up_sz(size_t a, size_t b) { return (a + b - 1) / b * b; }
}  // namespace

size_t nvls_size(size_t bytes, int n_devices) {
  LSGD_CU(cuInit, 0);
  CUmulticastObjectProp p = mc_prop(bytes, n_devices);
  size_t g = 0;
  LSGD_CU(cuMulticastGetGranularity, &g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  return round_up_sz(bytes, g ? g : (2u << 20));
}

uint64_t nvls_create(size_t size, int n_devices, int* fd_out) {
  LSGD_CU(cuInit, 0);
  CUmulticastObjectProp p = mc_prop(size, n_devices);
  CUmemGenericAllocationHandle mc = 0;
  LSGD_CU(cuMulticastCreate, &mc, &p);
  if (fd_out) {
    int fd = -1;
    LSGD_CU(cuMemExportToShareableHandle, &fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    *fd_out = fd;
  }
  return static_cast<uint64_t>(mc);
}

uint64_t nvls_import(int pid, int fd) {
  LSGD_CU(cuInit, 0);
  const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, pid, 0));
  check<Error>(pidfd >= 0, "NVLS: pidfd_open(", pid, ") failed");
  const int local = static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, fd, 0));
  close(pidfd);
  check<Error>(local >= 0, "NVLS: pidfd_getfd of the leader's multicast handle failed");
  CUmemGenericAllocationHandle mc = 0;
  static auto imp = LSGD_DRV(cuMemImportFromShareableHandle);
  CUresult r = imp(&mc, reinterpret_cast<void*>(static_cast<uintptr_t>(local)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(local);
  check<Error>(r == CUDA_SUCCESS, "NVLS: importing the multicast handle failed: ", cu_error(r));
  return static_cast<uint64_t>(mc);
}

void nvls_add_device(uint64_t mc, int dev) {
  CUdevice d;
  LSGD_CU(cuDeviceGet, &d, dev);
  LSGD_CU(cuMulticastAddDevice, static_cast<CUmemGenericAllocationHandle>(mc), d);
}

void nvls_bind_map(NvlsBuffer& b, uint64_t mc, size_t size, int dev) {
  LSGD_CUDA(cudaSetDevice(dev));
  LSGD_CUDA(cudaFree(nullptr));  // the primary context is current
  b.size = size;
  b.dev = dev;
  b.mc = mc;
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // as NCCL's NVLS buffers
  size_t gran = 0;
  LSGD_CU(cuMemGetAllocationGranularity, &gran, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  check<Error>(gran > 0 && size % gran == 0, "NVLS: buffer size ", size, " not a multiple of ", gran);
  size_t mgran = 0;  // the multicast object's granularity aligns the mappings
  {
    CUmulticastObjectProp p = mc_prop(size, 1);
    LSGD_CU(cuMulticastGetGranularity, &mgran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (mgran < gran) mgran = gran;
  }
  CUmemGenericAllocationHandle mem = 0;
  LSGD_CU(cuMemCreate, &mem, size, &ap, 0);
  b.mem = static_cast<uint64_t>(mem);
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr va = 0;
  LSGD_CU(cuMemAddressReserve, &va, size, mgran, 0, 0);
  LSGD_CU(cuMemMap, va, size, 0, mem, 0);
  LSGD_CU(cuMemSetAccess, va, size, &acc, 1);
  b.va = static_cast<uint64_t>(va);
  LSGD_CU(cuMulticastBindMem, static_cast<CUmemGenericAllocationHandle>(mc), 0, mem, 0, size, 0);
  CUdeviceptr mva = 0;
  LSGD_CU(cuMemAddressReserve, &mva, size, mgran, 0, 0);
  LSGD_CU(cuMemMap, mva, size, 0, static_cast<CUmemGenericAllocationHandle>(mc), 0);
  LSGD_CU(cuMemSetAccess, mva, size, &acc, 1);
  b.mc_va = static_cast<uint64_t>(mva);
  LSGD_CUDA(cudaMemset(reinterpret_cast<void*>(b.va), 0, size));
  LSGD_CUDA(cudaDeviceSynchronize());
}

void nvls_free(NvlsBuffer& b) {
  if (!b.size) return;
  cudaSetDevice(b.dev);
  cudaDeviceSynchronize();
  static auto dev_get = LSGD_DRV(cuDeviceGet);
  static auto unbind = LSGD_DRV(cuMulticastUnbind);
  static auto unmap = LSGD_DRV(cuMemUnmap);
  static auto addr_free = LSGD_DRV(cuMemAddressFree);
  static auto release = LSGD_DRV(cuMemRelease);
  CUdevice d;
  if (dev_get(&d, b.dev) == CUDA_SUCCESS && b.mc)
    unbind(static_cast<CUmemGenericAllocationHandle>(b.mc), d, 0, b.size);
  if (b.mc_va) {
    unmap(static_cast<CUdeviceptr>(b.mc_va), b.size);
    addr_free(static_cast<CUdeviceptr>(b.mc_va), b.size);
  }
  if (b.va) {
    unmap(static_cast<CUdeviceptr>(b.va), b.size);
    addr_free(static_cast<CUdeviceptr>(b.va), b.size);
  }
  if (b.mem) release(static_cast<CUmemGenericAllocationHandle>(b.mem));
  if (b.mc && b.own_mc) release(static_cast<CUmemGenericAllocationHandle>(b.mc));
  b = NvlsBuffer{};
}

void nvls_release(uint64_t mc) {
  static auto release = LSGD_DRV(cuMemRelease);
  if (mc) release(static_cast<CUmemGenericAllocationHandle>(mc));
}

}  // namespace lsgd_b200
