// NVLS multicast helpers (nvls.cu): the average fan-out of the push exchange through the NVSwitch.
#pragma once

#include <cstddef>
#include <cstdint>

namespace lsgd_b200 {

struct NvlsBuffer {
  uint64_t mc = 0;     // multicast object handle (CUmemGenericAllocationHandle)
  uint64_t mem = 0;    // this device's physical backing
  uint64_t va = 0;     // local view (the member's gfull)
  uint64_t mc_va = 0;  // multicast view: one multimem.st reaches every member
  size_t size = 0;
  int dev = -1;
  bool own_mc = true;  // release the multicast handle on free (false: shared by the threads of one process)
};

size_t nvls_size(size_t bytes, int n_devices);             // rounded to the multicast granularity
uint64_t nvls_create(size_t size, int n_devices, int* fd);  // leader; fd (may be null): POSIX fd to share
uint64_t nvls_import(int pid, int fd);                      // member of another process: dup the leader's fd
void nvls_add_device(uint64_t mc, int dev);                 // every member, before anyone binds
void nvls_bind_map(NvlsBuffer& b, uint64_t mc, size_t size, int dev);
void nvls_free(NvlsBuffer& b);
void nvls_release(uint64_t mc);  // drop a handle reference held outside any NvlsBuffer

}  // namespace lsgd_b200
