// tools/peaks.cu -- roofline denominators not in MEASURED_PEAKS.json:
//   write-only HBM bandwidth (8-B and 16-B streaming stores, like the fill's),
//   read+write copy bandwidth, and FP64 FMA throughput (DFMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void write8(double* p, size_t n, double v) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) __stcs(p + i, v + i);
}
__global__ void write16(double2* p, size_t n, double v) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) __stcs(p + i, make_double2(v, v + i));
}
__global__ void write16_const(double2* p, size_t n, double v) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) __stcs(p + i, make_double2(v, v));
}
__global__ void write16_wb(double2* p, size_t n, double v) {  // default (write-back) policy
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) p[i] = make_double2(v, v + i);
}
// TMA-engine bulk stores shared -> global (cp.async.bulk.global.shared::cta.bulk_group),
// one elected thread per CTA, CHUNK bytes per instruction, varying data
template <int CHUNK>
__global__ void bulk_store(char* g, size_t bytes) {
  extern __shared__ __align__(128) double sbuf[];
  for (int i = threadIdx.x; i < CHUNK / 8; i += blockDim.x) sbuf[i] = 1.0 + i * 1e-3 + blockIdx.x;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(sbuf));
  const size_t nchunk = bytes / CHUNK;
  int inflight = 0;
  for (size_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(g + c * CHUNK), "r"(s), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++inflight == 8) {
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      inflight = 4;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__global__ void copy16(const double2* a, double2* b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = __ldcs(a + i);
}
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999999;
  double c[8][2];
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t(8) << 30;
  double *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms, best;
  const size_t n8 = bytes / 8, n16 = bytes / 16;
  auto bw = [&](const char* name, auto launch, double moved) {
    best = 1e30f;
    for (int r = 0; r < 8; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2 && ms < best) best = ms;
    }
    printf("{\"test\": \"%s\", \"GB_s\": %.1f}\n", name, moved / (best * 1e-3) / 1e9);
  };
  bw("write_8B_stcs", [&] { write8<<<sms * 8, 256>>>(a, n8, 1.0); }, (double)bytes);
  bw("write_16B_stcs", [&] { write16<<<sms * 8, 256>>>((double2*)a, n16, 1.0); }, (double)bytes);
  bw("write_16B_stcs_const", [&] { write16_const<<<sms * 8, 256>>>((double2*)a, n16, 1.0); }, (double)bytes);
  bw("write_16B_wb", [&] { write16_wb<<<sms * 8, 256>>>((double2*)a, n16, 1.0); }, (double)bytes);
  cudaFuncSetAttribute(bulk_store<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(bulk_store<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  bw("bulk_store_16K", [&] { bulk_store<16384><<<sms * 4, 128, 16384>>>((char*)a, bytes); }, (double)bytes);
  bw("bulk_store_64K", [&] { bulk_store<65536><<<sms * 2, 128, 65536>>>((char*)a, bytes); }, (double)bytes);
  bw("memset", [&] { cudaMemsetAsync(a, 0, bytes); }, (double)bytes);
  bw("memset_0x5a", [&] { cudaMemsetAsync(a, 0x5a, bytes); }, (double)bytes);
  bw("copy_16B", [&] { copy16<<<sms * 8, 256>>>((double2*)a, (double2*)b, n16); }, 2.0 * bytes);
  // FP64 FMA throughput
  const int iters = 1 << 14;
  best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<sms * 4, 512>>>(b, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 1 && ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * iters * (double)sms * 4 * 512;
  printf("{\"test\": \"dfma\", \"TFLOP_s\": %.2f}\n", flops / (best * 1e-3) / 1e12);
  best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dmma_loop<<<sms * 4, 512>>>(b, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 1 && ms < best) best = ms;
  }
  // per warp-instruction 8*8*4 FMA
  const double mflops = 2.0 * 256 * 8 * iters * (double)sms * 4 * 512 / 32;
  printf("{\"test\": \"dmma_m8n8k4\", \"TFLOP_s\": %.2f}\n", mflops / (best * 1e-3) / 1e12);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"max_clock_mhz\": %d}\n", sms, clk / 1000);
  return 0;
}
