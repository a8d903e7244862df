// tools/memset_probe.cu -- one cudaMemsetAsync of 8 GB, for ncu inspection of the
// driver's fill kernel (which streams writes faster than st.global from user kernels)
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t bytes = size_t(8) << 30;
  char* a;
  cudaMalloc(&a, bytes);
  for (int r = 0; r < 3; ++r) cudaMemsetAsync(a, 0x5a, bytes);
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
