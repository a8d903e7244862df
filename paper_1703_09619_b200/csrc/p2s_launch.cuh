// p2s_launch.cuh -- host-side launch helpers shared by the ahead-of-time
// registries (p2s_reg_*.cu) and the generated per-shape modules (p2s_jit.cu).
//
// Kernel attributes (dynamic shared-memory limit, non-portable cluster size)
// belong to the kernel's module instance on ONE device, and the occupancy they
// imply is a per-device number too.  kernel_prepare() sets them once per
// (device, kernel, shared-memory size) under a mutex, so several contexts on
// several devices (p2s::fill_elements with gpus > 1, one host thread each) can
// launch the same kernel concurrently.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

namespace p2s {

// Tuning knobs (chunk sizes, variant selection) are read from the environment
// only in a tuning build (-DP2S_TUNING); the production library ignores them.
inline const char* tuning_env(const char* name) {
#ifdef P2S_TUNING
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Set the kernel's dynamic shared-memory limit (and optionally allow a
// non-portable cluster size) on the current device, once; report the number of
// resident CTAs per SM at `threads` threads and `smem` bytes when asked.
inline cudaError_t kernel_prepare(const void* fn, size_t smem, int threads, bool nonportable_cluster,
                                  int* blocks_per_sm) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(fn, dev, smem, threads);
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it == done.end()) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (nonportable_cluster) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem);
    if (e != cudaSuccess) return e;
    if (b < 1) return cudaErrorInvalidConfiguration;
    it = done.emplace(key, b).first;
  }
  if (blocks_per_sm) *blocks_per_sm = it->second;
  return cudaSuccess;
}

template <class K>
inline cudaError_t kernel_prepare(K* fn, size_t smem, int threads, bool nonportable_cluster = false,
                                  int* blocks_per_sm = nullptr) {
  return kernel_prepare(reinterpret_cast<const void*>(fn), smem, threads, nonportable_cluster, blocks_per_sm);
}

}  // namespace p2s
