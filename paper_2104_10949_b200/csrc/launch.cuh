// Host-side launch helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>

#include "common.cuh"

namespace mpc3 {

void set_last_error(const char* msg);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    set_last_error(buf);
    return MPC3_ERR_CUDA;
  }
  return MPC3_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// MPC3_PDL=0 disables programmatic dependent launch (common.cuh).
bool pdl_enabled();

// Launch with the programmatic-stream-serialization attribute: the kernel may
// begin while its predecessor in the stream drains (it waits in-kernel with
// griddepcontrol.wait before touching the predecessor's data).
template <typename... Exp, typename... Act>
inline cudaError_t launch_pdl(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Exp>(args)...);
}

// Grid for a grid-stride loop over `work` items with `threads` per CTA:
// a multiple of the SM count once the work is large enough.
inline unsigned grid_for(uint64_t work, int threads, int ctas_per_sm = 8) {
  const uint64_t sms = 148;
  uint64_t need = (work + threads - 1) / threads;
  uint64_t cap = sms * ctas_per_sm;
  if (need > cap) need = cap;
  if (need == 0) need = 1;
  return (unsigned)need;
}

}  // namespace mpc3
