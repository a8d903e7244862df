// p2s_scatter.cu -- global scatter-add of element matrices on the GPU: the
// reference's assemble_global (assembly.cpp:594-652), the step after the fill:
//
//   G[gi][gj] += s_i s_j E_e[i][j]   for local DOFs i, j with free indices gi, gj >= 0
//
// (orientation signs s = +-1; PEC-constrained DOFs carry free index -1 and are
// dropped, assembly.cpp:631-640).  One CTA per element: its free indices and
// signs are staged in shared memory, threads walk the n_local^2 entries row by
// row (coalesced reads of the element matrix) and accumulate with native FP64
// atomics -- entries shared between elements (edge / vertex DOFs) add up in
// unspecified order, so results agree with the reference's serial sum to
// rounding, not bitwise.  The ordered variant below (a per-mesh plan) reproduces
// the reference's summation order and arithmetic, bit for bit.  Two layouts: a generic row-major element matrix (the
// 3-D p2s_fill output) and the 2-D mode's eight blocks, read in place.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/p2s_b200.h"

p2s_status p2s_internal_fail(p2s_status st, const std::string& msg);
// 2-D mode block geometry of a context (p2s_cheb2d.cu)
bool p2s_cheb2d_block_layout(const p2s_cheb2d_ctx* c, int64_t off[8], int rows[8], int cols[8],
                             int* n_eu, int* n_ev);

namespace {

constexpr int kMaxLocal = 4096;  // shared staging: 12 B per local DOF

struct Blocks8 {
  int64_t off[8];
  int cols[8];
  int n_eu;
};

template <class Entry>
__device__ __forceinline__ void scatter_element(int n_local, const int32_t* __restrict__ gfree,
                                                const double* __restrict__ gsign, double* G,
                                                int64_t ldG, Entry&& entry) {
  __shared__ int32_t fr[kMaxLocal];
  __shared__ double sg[kMaxLocal];
  for (int i = threadIdx.x; i < n_local; i += blockDim.x) {
    fr[i] = gfree[i];
    sg[i] = gsign[i];
  }
  __syncthreads();
  for (int i = 0; i < n_local; ++i) {
    const int gi = fr[i];
    if (gi < 0) continue;  // uniform across the CTA
    const double si = sg[i];
    double* Grow = G + static_cast<int64_t>(gi) * ldG;
    for (int j = threadIdx.x; j < n_local; j += blockDim.x) {
      const int gj = fr[j];
      if (gj >= 0) atomicAdd(Grow + gj, si * sg[j] * entry(i, j));
    }
  }
}

__global__ void scatter_generic_kernel(const double* __restrict__ E, int64_t estride, int64_t ldE,
                                       int n_local, const int32_t* __restrict__ dof_free,
                                       const double* __restrict__ dof_sign, double* G, int64_t ldG) {
  const int64_t e = blockIdx.x;
  const double* Ee = E + e * estride;
  scatter_element(n_local, dof_free + e * n_local, dof_sign + e * n_local, G, ldG,
                  [&](int i, int j) { return __ldg(Ee + static_cast<int64_t>(i) * ldE + j); });
}

// blockIdx.y: 0 stiffness (blocks 0-3 -> S), 1 mass (blocks 4-7 -> M)
__global__ void scatter_cheb2d_kernel(const __grid_constant__ Blocks8 b, const double* __restrict__ blocks,
                                      int64_t per_elem, int n_local, const int32_t* __restrict__ dof_free,
                                      const double* __restrict__ dof_sign, double* S, double* M,
                                      int64_t ldG) {
  const int64_t e = blockIdx.x;
  const int base = blockIdx.y * 4;
  const double* Be = blocks + e * per_elem;
  scatter_element(n_local, dof_free + e * n_local, dof_sign + e * n_local, blockIdx.y ? M : S, ldG,
                  [&](int i, int j) {
                    const bool iu = i < b.n_eu, ju = j < b.n_eu;  // assembly.cpp:609-624
                    const int q = base + (iu ? (ju ? 0 : 1) : (ju ? 2 : 3));
                    const int bi = iu ? i : i - b.n_eu, bj = ju ? j : j - b.n_eu;
                    return __ldg(Be + b.off[q] + static_cast<int64_t>(bi) * b.cols[q] + bj);
                  });
}

// ---------------------------------------------------------------- ordered scatter
// Deterministic variant: the summation order of the reference's assemble_global
// (elements ascending, then local row i, assembly.cpp:626-641), bit for bit.
// The plan lists, per global row g, the (element, local row i) contributions in
// that order (CSR built once from the host DOF map); one CTA per global row
// walks its list, each entry's local columns j in parallel (distinct global
// columns within one element), a barrier between entries, and the reference's
// arithmetic G += (s_i s_j) E without FMA contraction.

__device__ __forceinline__ void ordered_entry(double* Grow, int n_local, const int32_t* __restrict__ fr,
                                              const double* __restrict__ sg, double si, const double* Erow_ptr,
                                              int64_t estride_unused) {
  (void)estride_unused;
  for (int j = threadIdx.x; j < n_local; j += blockDim.x) {
    const int gj = __ldg(fr + j);
    if (gj < 0) continue;
    const double w = __dmul_rn(si, __ldg(sg + j));
    Grow[gj] = __dadd_rn(Grow[gj], __dmul_rn(w, __ldg(Erow_ptr + j)));
  }
}

__global__ void scatter_ordered_kernel(const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ row_ent,
                                       const double* __restrict__ E, int64_t estride, int64_t ldE, int n_local,
                                       const int32_t* __restrict__ dof_free, const double* __restrict__ dof_sign,
                                       double* G, int64_t ldG) {
  const int64_t g = blockIdx.x;
  double* Grow = G + g * ldG;
  for (int64_t k = row_ptr[g]; k < row_ptr[g + 1]; ++k) {
    const int64_t ent = row_ent[k];
    const int64_t e = ent / n_local;
    const int i = static_cast<int>(ent - e * n_local);
    ordered_entry(Grow, n_local, dof_free + e * n_local, dof_sign + e * n_local,
                  __ldg(dof_sign + e * n_local + i), E + e * estride + static_cast<int64_t>(i) * ldE, 0);
    __syncthreads();  // the next entry may hit the same global columns
  }
}

__global__ void scatter_ordered_cheb2d_kernel(const int64_t* __restrict__ row_ptr,
                                              const int64_t* __restrict__ row_ent, const __grid_constant__ Blocks8 b,
                                              const double* __restrict__ blocks, int64_t per_elem, int n_local,
                                              const int32_t* __restrict__ dof_free,
                                              const double* __restrict__ dof_sign, double* S, double* M,
                                              int64_t ldG) {
  const int64_t g = blockIdx.x;
  const int base = blockIdx.y * 4;
  double* Grow = (blockIdx.y ? M : S) + g * ldG;
  for (int64_t k = row_ptr[g]; k < row_ptr[g + 1]; ++k) {
    const int64_t ent = row_ent[k];
    const int64_t e = ent / n_local;
    const int i = static_cast<int>(ent - e * n_local);
    const int32_t* fr = dof_free + e * n_local;
    const double* sg = dof_sign + e * n_local;
    const double si = __ldg(sg + i);
    const double* Be = blocks + e * per_elem;
    const bool iu = i < b.n_eu;
    const int bi = iu ? i : i - b.n_eu;
    for (int j = threadIdx.x; j < n_local; j += blockDim.x) {
      const int gj = __ldg(fr + j);
      if (gj < 0) continue;
      const bool ju = j < b.n_eu;  // assembly.cpp:609-624
      const int q = base + (iu ? (ju ? 0 : 1) : (ju ? 2 : 3));
      const int bj = ju ? j : j - b.n_eu;
      const double w = __dmul_rn(si, __ldg(sg + j));
      Grow[gj] = __dadd_rn(Grow[gj], __dmul_rn(w, __ldg(Be + b.off[q] + static_cast<int64_t>(bi) * b.cols[q] + bj)));
    }
    __syncthreads();
  }
}

}  // namespace

struct p2s_scatter_plan {
  int device = 0;
  int64_t n_elem = 0;
  int32_t n_local = 0, n_free = 0;
  int64_t* d_row_ptr = nullptr;
  int64_t* d_row_ent = nullptr;
};

extern "C" {

p2s_status p2s_scatter_plan_create(const int32_t* h_dof_free, int64_t n_elem, int32_t n_local, int32_t n_free,
                                   int device, p2s_scatter_plan** out) {
  if (!out) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_plan_create: null out");
  *out = nullptr;
  if (n_elem < 0 || n_local < 0 || n_free < 0 || (n_elem * n_local > 0 && !h_dof_free))
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_plan_create: bad sizes");
  // counting sort by global row, stable in (element, local row) order
  std::vector<int64_t> ptr(static_cast<size_t>(n_free) + 1, 0);
  for (int64_t k = 0; k < n_elem * n_local; ++k) {
    const int32_t g = h_dof_free[k];
    if (g >= n_free) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_plan_create: free index >= n_free");
    if (g >= 0) ++ptr[static_cast<size_t>(g) + 1];
  }
  for (int32_t g = 0; g < n_free; ++g) ptr[static_cast<size_t>(g) + 1] += ptr[static_cast<size_t>(g)];
  std::vector<int64_t> ent(static_cast<size_t>(ptr.back()));
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t k = 0; k < n_elem * n_local; ++k) {
    const int32_t g = h_dof_free[k];
    if (g >= 0) ent[static_cast<size_t>(fill[static_cast<size_t>(g)]++)] = k;  // k = e * n_local + i
  }
  auto* p = new p2s_scatter_plan;
  p->device = device;
  p->n_elem = n_elem;
  p->n_local = n_local;
  p->n_free = n_free;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_row_ptr, sizeof(int64_t) * ptr.size());
  if (e == cudaSuccess) e = cudaMalloc(&p->d_row_ent, sizeof(int64_t) * std::max<size_t>(1, ent.size()));
  if (e == cudaSuccess)
    e = cudaMemcpy(p->d_row_ptr, ptr.data(), sizeof(int64_t) * ptr.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !ent.empty())
    e = cudaMemcpy(p->d_row_ent, ent.data(), sizeof(int64_t) * ent.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    p2s_scatter_plan_destroy(p);
    return p2s_internal_fail(P2S_CUDA_ERROR, std::string("p2s_scatter_plan_create: ") + cudaGetErrorString(e));
  }
  *out = p;
  return P2S_OK;
}

void p2s_scatter_plan_destroy(p2s_scatter_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->d_row_ptr) cudaFree(p->d_row_ptr);
  if (p->d_row_ent) cudaFree(p->d_row_ent);
  delete p;
}

p2s_status p2s_scatter_add_ordered(const p2s_scatter_plan* plan, const double* d_elem, int64_t elem_stride,
                                   int64_t ld_elem, const int32_t* d_dof_free, const double* d_dof_sign,
                                   double* d_G, int64_t ld_G, void* stream) {
  if (!plan) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_add_ordered: null plan");
  const int n_local = plan->n_local;
  if (ld_elem < n_local || ld_G < plan->n_free || elem_stride < static_cast<int64_t>(n_local) * ld_elem)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_add_ordered: bad sizes");
  if (plan->n_free == 0 || plan->n_elem == 0 || n_local == 0) return P2S_OK;
  if (!d_elem || !d_dof_free || !d_dof_sign || !d_G)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_add_ordered: null buffer");
  scatter_ordered_kernel<<<static_cast<unsigned>(plan->n_free), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      plan->d_row_ptr, plan->d_row_ent, d_elem, elem_stride, ld_elem, n_local, d_dof_free, d_dof_sign, d_G, ld_G);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return p2s_internal_fail(P2S_CUDA_ERROR, std::string("scatter_ordered_kernel: ") + cudaGetErrorString(e));
  return P2S_OK;
}

p2s_status p2s_cheb2d_scatter_ordered(const p2s_cheb2d_ctx* ctx, const p2s_scatter_plan* plan,
                                      const double* d_blocks, const int32_t* d_dof_free, const double* d_dof_sign,
                                      double* d_S, double* d_M, int64_t ld_G, void* stream) {
  Blocks8 b{};
  int rows[8], n_ev = 0;
  if (!ctx || !plan || !p2s_cheb2d_block_layout(ctx, b.off, rows, b.cols, &b.n_eu, &n_ev))
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_scatter_ordered: null context or plan");
  const int n_local = b.n_eu + n_ev;
  if (n_local != plan->n_local || ld_G < plan->n_free)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_scatter_ordered: plan / context mismatch");
  if (plan->n_free == 0 || plan->n_elem == 0) return P2S_OK;
  if (!d_blocks || !d_dof_free || !d_dof_sign || !d_S || !d_M)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_scatter_ordered: null buffer");
  int64_t per_elem = 0;
  for (int q = 0; q < 8; ++q) per_elem += static_cast<int64_t>(rows[q]) * b.cols[q];
  scatter_ordered_cheb2d_kernel<<<dim3(static_cast<unsigned>(plan->n_free), 2), 256, 0,
                                  static_cast<cudaStream_t>(stream)>>>(plan->d_row_ptr, plan->d_row_ent, b, d_blocks,
                                                                      per_elem, n_local, d_dof_free, d_dof_sign,
                                                                      d_S, d_M, ld_G);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return p2s_internal_fail(P2S_CUDA_ERROR, std::string("scatter_ordered_cheb2d_kernel: ") + cudaGetErrorString(e));
  return P2S_OK;
}


p2s_status p2s_scatter_add(const double* d_elem, int64_t elem_stride, int64_t ld_elem, int32_t n_local,
                           const int32_t* d_dof_free, const double* d_dof_sign, int64_t n_elem,
                           double* d_G, int64_t ld_G, void* stream) {
  if (n_elem < 0 || n_local < 0 || n_local > kMaxLocal || ld_elem < n_local || ld_G < 1 ||
      elem_stride < static_cast<int64_t>(n_local) * ld_elem)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_add: bad sizes (n_local <= 4096)");
  if (n_elem == 0 || n_local == 0) return P2S_OK;
  if (!d_elem || !d_dof_free || !d_dof_sign || !d_G)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_scatter_add: null buffer");
  scatter_generic_kernel<<<static_cast<unsigned>(n_elem), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_elem, elem_stride, ld_elem, n_local, d_dof_free, d_dof_sign, d_G, ld_G);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return p2s_internal_fail(P2S_CUDA_ERROR, std::string("scatter_generic_kernel: ") + cudaGetErrorString(e));
  return P2S_OK;
}

p2s_status p2s_cheb2d_scatter(const p2s_cheb2d_ctx* ctx, const double* d_blocks, const int32_t* d_dof_free,
                              const double* d_dof_sign, int64_t n_elem, double* d_S, double* d_M,
                              int64_t ld_G, void* stream) {
  Blocks8 b{};
  int rows[8], n_ev = 0;
  if (!ctx || !p2s_cheb2d_block_layout(ctx, b.off, rows, b.cols, &b.n_eu, &n_ev))
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_scatter: null context");
  const int n_local = b.n_eu + n_ev;
  if (n_elem < 0 || ld_G < 1 || n_local > kMaxLocal)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_scatter: bad sizes");
  if (n_elem == 0) return P2S_OK;
  if (!d_blocks || !d_dof_free || !d_dof_sign || !d_S || !d_M)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_scatter: null buffer");
  int64_t per_elem = 0;
  for (int q = 0; q < 8; ++q) per_elem += static_cast<int64_t>(rows[q]) * b.cols[q];
  scatter_cheb2d_kernel<<<dim3(static_cast<unsigned>(n_elem), 2), 256, 0,
                          static_cast<cudaStream_t>(stream)>>>(b, d_blocks, per_elem, n_local, d_dof_free,
                                                              d_dof_sign, d_S, d_M, ld_G);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return p2s_internal_fail(P2S_CUDA_ERROR, std::string("scatter_cheb2d_kernel: ") + cudaGetErrorString(e));
  return P2S_OK;
}

}  // extern "C"
