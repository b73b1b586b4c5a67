// Debug: TMA-load a 4-D box (k 32, limb 4, row 128) with SWIZZLE_128B into
// shared memory and dump it, to check the smem layout TMA produces.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void dump(const __grid_constant__ CUtensorMap tm, uint8_t* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t sd = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(16384));
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(sd),
        "l"(&tm), "r"(sb), "r"(0), "r"(0), "r"(0), "r"(0) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(sb));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int kp = 64, rows = 128;
  std::vector<uint8_t> h(8 * rows * kp);
  // byte value encodes (limb, row, k-chunk16): limb*32 + (row % 8) * 4 + chunk
  for (int l = 0; l < 8; ++l)
    for (int r = 0; r < rows; ++r)
      for (int k = 0; k < kp; ++k) h[(l * rows + r) * kp + k] = (uint8_t)(l * 32 + (r % 8) * 4 + (k / 16));
  uint8_t *d, *o;
  cudaMalloc(&d, h.size());
  cudaMalloc(&o, 16384);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[4] = {(cuuint64_t)kp, 8, (cuuint64_t)rows, 1};
  cuuint64_t strides[3] = {(cuuint64_t)(rows * kp), (cuuint64_t)kp, (cuuint64_t)(8 * rows * kp)};
  cuuint32_t box[4] = {32, 4, 128, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(dump, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  dump<<<1, 128, 17408>>>(tm, o);
  printf("launch %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<uint8_t> g(16384);
  cudaMemcpy(g.data(), o, 16384, cudaMemcpyDeviceToHost);
  // print each 16-byte smem chunk's source tag for the first 16 x 128-byte rows
  for (int row = 0; row < 16; ++row) {
    printf("smem row %2d:", row);
    for (int c = 0; c < 8; ++c) {
      int v = g[row * 128 + c * 16];
      printf(" (l%d r%d c%d)", v / 32, (v % 32) / 4, v % 4);
    }
    printf("\n");
  }
  return 0;
}
