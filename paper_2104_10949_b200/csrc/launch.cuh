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
