// mma_rate.cu -- tcgen05 MMA issue-rate microbenchmark (no data movement).
// One CTA per SM; one thread issues ITERS MMAs on fixed shared-memory
// descriptors (zeroed operands / scales), then commits and waits.  Reports the
// chip-wide dense TFLOP/s each MMA form sustains at the running clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2512_02010_b200/csrc/f46_ptx.cuh"

using namespace f46::ptx;

constexpr int ITERS = 8192;

template <int VARIANT>
__global__ void __launch_bounds__(128, 1) mma_loop(long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&holder, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if ((VARIANT == 8 || VARIANT == 9) && warp != 1) {
    // concurrent tcgen05.st traffic from the other warps (their own lane quadrants)
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = 0x38383838u;
    const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 256;
    const long long s0 = clock64();
    for (int i = 0; i < ITERS / 4; ++i) {
      tc_st_32x32b_x32(base + (i & 3) * 48, v);
      tc_wait_st();
    }
    const long long s1 = clock64();
    if (blockIdx.x == 0 && warp == 0 && (threadIdx.x & 31) == 0) cycles[1] = s1 - s0;
  }
  if (threadIdx.x == 32) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint64_t ad = smem_desc(a, 16, 1024, 2), bd = smem_desc(b, 16, 1024, 2);
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
      if (VARIANT == 0) {
        // NVFP4: kind::mxf4nvf4 scale_vec::4X (UE4M3 per 16), M=128 N=256 K=64
        constexpr uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
        mma_nvf4(tmem, ad, bd, idesc, i != 0, tmem + 256, tmem + 272);
      } else if (VARIANT == 1) {
        // MXFP4: kind::mxf4 scale_vec::2X (UE8M0 per 32), M=128 N=256 K=64
        constexpr uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (1u << 23) | (8u << 24);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], "
            "[%6], p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(i != 0)), "r"(tmem + 256), "r"(tmem + 272)
            : "memory");
      } else if (VARIANT == 2) {
        // BF16: kind::f16, M=128 N=256 K=16, f32 accumulate
        constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(i != 0))
            : "memory");
      } else if (VARIANT == 4) {
        // copies only: 12 x 32x128b.warpx4 per "4 MMAs"
        if ((i & 3) == 0)
          for (int j = 0; j < 12; ++j)
            tc_cp_32x128b_x4(tmem + 256 + ((i >> 2) & 1) * 48 + 4 * j,
                             smem_desc(smem_u32(smem + 49152) + 512 * (j & 3), 0, 128, 0));
      } else if (VARIANT == 5) {
        // copies only: 3 x 128x256b (4 KB each, no replication) per "4 MMAs"
        if ((i & 3) == 0)
          for (int j = 0; j < 3; ++j)
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 256 + ((i >> 2) & 1) * 48 + 8 * j),
                         "l"(smem_desc(smem_u32(smem + 49152), 0, 256, 0)) : "memory");
      } else if (VARIANT == 6) {
        // copies only: 12 x 128x128b (2 KB each, no replication) per "4 MMAs"
        if ((i & 3) == 0)
          for (int j = 0; j < 12; ++j)
            asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + 256 + ((i >> 2) & 1) * 48 + 4 * j),
                         "l"(smem_desc(smem_u32(smem + 49152), 0, 128, 0)) : "memory");
      } else if (VARIANT == 7) {
        // NVFP4 MMA + 3 x 128x256b per 4 MMAs
        if ((i & 3) == 0)
          for (int j = 0; j < 3; ++j)
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 256 + ((i >> 2) & 1) * 48 + 8 * j),
                         "l"(smem_desc(smem_u32(smem + 49152), 0, 256, 0)) : "memory");
        constexpr uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
        mma_nvf4(tmem, ad, bd, idesc, i != 0, tmem + 256 + ((i >> 2) & 1) * 48,
                 tmem + 272 + ((i >> 2) & 1) * 48);
      } else if (VARIANT == 9) {
      } else if (VARIANT == 8) {
        constexpr uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
        mma_nvf4(tmem, ad, bd, idesc, i != 0, tmem + 256, tmem + 272);
      } else {
        // NVFP4 with a scale-factor copy every 4 MMAs (the GEMM's steady state)
        if ((i & 3) == 0) {
          for (int j = 0; j < 12; ++j)
            tc_cp_32x128b_x4(tmem + 256 + ((i >> 2) & 1) * 48 + 4 * j,
                             smem_desc(smem_u32(smem + 49152) + 512 * (j & 3), 0, 128, 0));
        }
        constexpr uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
        mma_nvf4(tmem, ad, bd, idesc, i != 0, tmem + 256 + ((i >> 2) & 1) * 48,
                 tmem + 272 + ((i >> 2) & 1) * 48);
      }
    }
    tc_commit(&done);
    mbar_wait(&done, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int V>
void run(const char* name, double flops_per_mma, int sms) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  cudaFuncSetAttribute(mma_loop<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  mma_loop<V><<<sms, 128, 64 * 1024>>>(d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) mma_loop<V><<<sms, 128, 64 * 1024>>>(d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long cyc = 0, st_cyc[2] = {0, 0};
  cudaMemcpy(st_cyc, d, 16, cudaMemcpyDeviceToHost);
  cyc = st_cyc[0];
  if (st_cyc[1]) printf("   [store loop: %.1f cycles per tcgen05.st.x32 + wait::st]\n", (double)st_cyc[1] / (ITERS / 4));
  const double s = ms * 1e-3 / reps;
  printf("%-44s %8.1f TFLOP/s  %6.1f cycles/MMA  (%s)\n", name,
         flops_per_mma * ITERS * sms / s / 1e12, (double)cyc / ITERS,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("nvf4 mxf4nvf4.scale_vec::4X 128x256x64", 2.0 * 128 * 256 * 64, sms);
  run<1>("mxf4 mxf4.scale_vec::2X 128x256x64", 2.0 * 128 * 256 * 64, sms);
  run<2>("bf16 f16 128x256x16", 2.0 * 128 * 256 * 16, sms);
  run<3>("nvf4 + 12 SF copies per 4 MMAs", 2.0 * 128 * 256 * 64, sms);
  run<4>("only 12 x cp.32x128b.warpx4 per 4 slots", 2.0 * 128 * 256 * 64, sms);
  run<5>("only 3 x cp.128x256b per 4 slots", 2.0 * 128 * 256 * 64, sms);
  run<6>("only 12 x cp.128x128b per 4 slots", 2.0 * 128 * 256 * 64, sms);
  run<7>("nvf4 + 3 x cp.128x256b per 4 MMAs", 2.0 * 128 * 256 * 64, sms);
  run<8>("nvf4 while 3 warps tcgen05.st x32 + wait", 2.0 * 128 * 256 * 64, sms);
  run<9>("3 warps tcgen05.st x32 + wait, no MMA", 2.0 * 128 * 256 * 64, sms);
  return 0;
}
