// tools/power_probe.cu -- sustained (5 s) pure streaming-store kernel, to see
// whether HBM write traffic alone reaches the 1000 W power cap.  Run with
// nvidia-smi sampling in the background.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void write16(double2* p, size_t n, double v) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) __stcs(p + i, make_double2(v, v + i));
}
int main() {
  const size_t bytes = size_t(16) << 30;
  double2* a;
  cudaMalloc(&a, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto t0 = std::chrono::steady_clock::now();
  int reps = 0;
  cudaEventRecord(e0);
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 6.0) {
    for (int r = 0; r < 20; ++r) write16<<<148 * 8, 256>>>(a, bytes / 16, 1.0);
    cudaDeviceSynchronize();
    reps += 20;
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"sustained_write_GB_s\": %.1f, \"seconds\": %.2f}\n", reps * (double)bytes / (ms * 1e-3) / 1e9, ms / 1e3);
  return 0;
}
