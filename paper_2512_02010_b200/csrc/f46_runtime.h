// f46_runtime.h -- host-side launch state shared by the translation units.
//
// Everything cached here is per device (indexed by cudaGetDevice()), so one
// process may drive several GPUs: the SM count, and each kernel's
// dynamic-shared-memory opt-in and occupancy, are established on the first
// launch on each device.  Test hooks (alternate kernels, forced chunking) are
// set explicitly through f46_set_test_hook, never read from the environment
// on a launch path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

namespace f46rt {

constexpr int kMaxDevices = 64;

inline int device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}

inline int num_sms() {
  static std::atomic<int> sms[kMaxDevices];
  const int d = device();
  int v = sms[d].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    if (v <= 0) v = 148;
    sms[d].store(v, std::memory_order_relaxed);
  }
  return v;
}

// Opt the kernel into `smem` bytes of dynamic shared memory on the current
// device (once per device and kernel) and return its resident CTAs per SM at
// `threads` threads (>= 1).
inline int configure(const void* kernel, int smem, int threads) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ;
  const int d = device();
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(kernel, d);
  auto it = occ.find(key);
  if (it != occ.end()) return it->second;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  if (n < 1) n = 1;
  occ[key] = n;
  return n;
}

// Test / diagnostic hooks (f46_set_test_hook); all default to 0.
enum Hook {
  HOOK_SEG_CHUNK_BYTES = 0,  // > 0: K2 launches at most this many input bytes at a time
  HOOK_DQ_VEC = 1,           // 1: dequantize takes the coalesced (non-TMA) kernel
  HOOK_Q2_V1 = 2,            // 1: 2-D tiles take the one-tile-per-warp kernel
  HOOK_SR_ONE_THREAD = 3,    // 1: stochastic rounding takes the one-thread-per-block kernel
  HOOK_GEMM_KERNEL = 4,      // 0: CTA-pair tcgen05 GEMM, 1: single-CTA persistent, 2: one tile per CTA
  HOOK_COUNT = 5
};

int64_t hook(int h);

}  // namespace f46rt
