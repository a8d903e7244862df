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
// rounding, not bitwise.  Two layouts: a generic row-major element matrix (the
// 3-D p2s_fill output) and the 2-D mode's eight blocks, read in place.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

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

}  // namespace

extern "C" {

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
