// sf_probe.cu -- which TMEM lanes / columns does tcgen05.mma kind::mxf4nvf4
// (scale_vec::4X, M=128, N=256, cta_group::1) read its scale factors from?
//
// A (128x64) and B (256x64) are all E2M1 1.0; every scale is UE4M3 1.0 (0x38)
// where a variant places it and 0 elsewhere, written with tcgen05.st.  The MMA
// then gives D[m][n] = 64 exactly when row m's SFA and row n's SFB were found.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sf_probe tools/sf_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2512_02010_b200/csrc/f46_ptx.cuh"

using namespace f46::ptx;

__device__ __forceinline__ void tc_st_32x32b_x4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c,
                                                uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a),
               "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// variant: 0 = replicated in all 4 quadrants (CUTLASS layout), 1 = quadrant 0 only,
// 2 = "diagonal" (quadrant r holds only column r), 3 = quadrant r holds rows 32r..: col 0
__global__ void probe(int variant, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: 128 rows x 32 B, B: 256 rows x 32 B, K-major SW128 (rows 128 B apart): code 2 (1.0) everywhere
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  // scale-factor region: SFA at columns 256..259, SFB at 272..279
  {
    const int q = warp & 3;
    const uint32_t one = 0x38383838u;  // four UE4M3 1.0
    uint32_t va[4] = {0, 0, 0, 0}, vb0[4] = {0, 0, 0, 0}, vb1[4] = {0, 0, 0, 0};
    for (int c = 0; c < 4; ++c) {
      bool on = variant == 0 || (variant == 1 && q == 0) || (variant == 2 && c == q) ||
                (variant == 3 && c == 0);
      va[c] = vb0[c] = vb1[c] = on ? one : 0u;
    }
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
    tc_st_32x32b_x4(lane_base + 256, va[0], va[1], va[2], va[3]);
    tc_st_32x32b_x4(lane_base + 272, vb0[0], vb0[1], vb0[2], vb0[3]);
    tc_st_32x32b_x4(lane_base + 276, vb1[0], vb1[1], vb1[2], vb1[3]);
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint64_t ad = smem_desc(smem_u32(smem), 16, 1024, 2);
    const uint64_t bd = smem_desc(smem_u32(smem + 128 * 128), 16, 1024, 2);
    constexpr uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
    mma_nvf4(tmem, ad, bd, idesc, 0, tmem + 256, tmem + 272);
    tc_commit(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  {
    const int q = warp & 3;
    for (int c = 0; c < 256; c += 32) {
      uint32_t r[32];
      tc_ld_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + c, r);
      tc_wait_ld();
      for (int j = 0; j < 32; ++j) out[(32 * q + lane) * 256 + c + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 256 * 4);
  static float h[128 * 256];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char* names[] = {"replicated x4", "quadrant 0 only", "diagonal (quadrant r, col r)",
                         "col 0 in every quadrant"};
  for (int v = 0; v < 4; ++v) {
    cudaMemset(d, 0, 128 * 256 * 4);
    probe<<<1, 128, 64 * 1024>>>(v, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // summarise: which (row block of 32, col block of 32) came out 64
    printf("%-30s %s\n  rows\\cols(32-blocks): ", names[v], cudaGetErrorString(e));
    for (int rb = 0; rb < 4; ++rb) {
      printf("\n  r%d: ", rb);
      for (int cb = 0; cb < 8; ++cb) {
        int good = 0;
        for (int i = 0; i < 32; ++i)
          for (int j = 0; j < 32; ++j) good += h[(32 * rb + i) * 256 + 32 * cb + j] == 64.0f;
        printf("%5d", good);
      }
    }
    printf("\n");
  }
  return 0;
}
