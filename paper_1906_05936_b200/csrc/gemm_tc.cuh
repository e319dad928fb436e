// Tensor-core (tcgen05, kind::tf32, split-TF32 x3) path for the dense-layer GEMMs of the fp32 step.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host.hpp"
#include "kernels.cuh"

namespace lsgd_b200 {

struct TcWorkspace {
  bool ready = false;
  std::vector<void*> bufs;  // owned device allocations
};

bool tc_shapes_supported(const std::vector<int32_t>& layers, int batch);
void tc_alloc(TcWorkspace& ws, const Layout& L, int batch, int n_features);
void tc_free(TcWorkspace& ws);
void tc_split_weights(TcWorkspace& ws, const Layout& L, const float* w, cudaStream_t st, LaunchCounter& lc);
void tc_forward_backward(TcWorkspace& ws, const Layout& L, int batch, const float* x, const int32_t* y, float* payload,
                         float* sample_loss, cudaStream_t st, LaunchCounter& lc);

}  // namespace lsgd_b200
