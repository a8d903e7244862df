// p2s_direct.cu -- the direct-quadrature fill on the GPU: the paper's baseline
// that product-to-sum replaces (the reference's assemble_direct_element,
// assembly.hpp:50 / assembly.cpp:134-274, and fill_elements(.., Backend::direct,
// ..), assembly.hpp:12-15, 82-83), in 3-D:
//
//   M[gi,i][gj,j] = sum_s sum_q  phi^test_{s,i}(q) * w_q alpha_s^{gi gj}(q) * phi^trial_{s,j}(q)
//
// over the full tensor Gauss-Legendre rule (nq_u nq_v nq_w points), i.e. per
// (element, pair, term) one dense GEMM  B_test^T . diag(w alpha) . B_trial  with
// B[q][t] = f_m(u_q) g_n(v_q) h_p(w_q) (P or P' per side and direction).  Dense
// GEMM-shaped FP64 work: it runs on the FP64 tensor cores through cuBLAS DGEMM
// (strided-batched over the elements of a chunk); a small kernel forms
// W = diag(w alpha) B_trial.  It exists as the ablation baseline (bench.py
// "ablation") and as an independent GPU check of the p2s path.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/p2s_b200.h"
#include "p2s_tables.hpp"

p2s_status p2s_internal_fail(p2s_status st, const std::string& msg);

struct p2s_direct_ctx {
  p2s_problem pb{};
  int device = 0;
  int Nt = 0, n_tot = 0, P = 0, S = 0;
  int64_t Q = 0, alpha_per_elem = 0;
  double* d_test[P2S_MAX_TERMS]{};   // [Q][Nt]
  double* d_trial[P2S_MAX_TERMS]{};  // [Q][Nt], weights folded
  double* d_W = nullptr;             // [chunk][Q][Nt]
  int64_t chunk = 1;
  cublasHandle_t blas = nullptr;
};

namespace {

// B[q][t] = f[m][qu] * g[n][qv] * h[p][qw]; q = (qw*nqv + qv)*nqu + qu,
// t = (m*Nv + n)*Nw + p.  f/g/h are [N][nq] 1-D tables.
__global__ void direct_basis_kernel(double* __restrict__ B, const double* __restrict__ f,
                                    const double* __restrict__ g, const double* __restrict__ h,
                                    int Nu, int Nv, int Nw, int nqu, int nqv, int nqw) {
  const int64_t Nt = static_cast<int64_t>(Nu) * Nv * Nw;
  const int64_t total = Nt * nqu * nqv * nqw;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = i / Nt;
    const int t = static_cast<int>(i - q * Nt);
    const int qu = static_cast<int>(q % nqu), qv = static_cast<int>((q / nqu) % nqv),
              qw = static_cast<int>(q / (static_cast<int64_t>(nqu) * nqv));
    const int p = t % Nw, n = (t / Nw) % Nv, m = t / (Nw * Nv);
    B[i] = f[m * nqu + qu] * g[n * nqv + qv] * h[p * nqw + qw];
  }
}

// W[b][q][t] = alpha[e0 + b][pair][s][q] * Btrial[q][t]
__global__ void direct_scale_kernel(double* __restrict__ W, const double* __restrict__ alpha,
                                    const double* __restrict__ Bt, int64_t Q, int Nt,
                                    int64_t alpha_per_elem, int64_t alpha_off) {
  const int64_t b = blockIdx.y;
  const double* a = alpha + b * alpha_per_elem + alpha_off;
  double* w = W + b * Q * Nt;
  const int64_t total = Q * Nt;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w[i] = __ldg(a + i / Nt) * Bt[i];
}

p2s_status cuda_fail(cudaError_t e, const char* what) {
  return p2s_internal_fail(P2S_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

#define DCUDA(x)                                       \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x);   \
  } while (0)

}  // namespace

extern "C" {

p2s_status p2s_direct_create(const p2s_problem* spec, int device, p2s_direct_ctx** out) {
  if (!spec || !out) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_create: null argument");
  *out = nullptr;
  if (spec->n_comp < 1 || spec->n_comp > 3 || spec->n_terms < 1 || spec->n_terms > P2S_MAX_TERMS)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_create: n_comp 1..3, n_terms 1..4");
  for (int d = 0; d < 3; ++d)
    if (spec->order[d] < 1 || spec->order[d] > 32 || spec->nq[d] < 1 || spec->nq[d] > 64)
      return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_create: order 1..32, nq 1..64");
  for (int s = 0; s < spec->n_terms; ++s)
    for (int d = 0; d < 3; ++d)
      if (spec->kind[s][d] < 0 || spec->kind[s][d] > 3)
        return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_create: bad kind");
  if (spec->basis != P2S_BASIS_MODAL && spec->basis != P2S_BASIS_CONFORMING)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_create: bad basis");
  if (spec->basis == P2S_BASIS_CONFORMING)
    for (int d = 0; d < 3; ++d)
      if (spec->order[d] < 2)
        return p2s_internal_fail(P2S_INVALID_ARG, "conforming basis needs order >= 2");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return p2s_internal_fail(P2S_CUDA_ERROR, "p2s_direct_create: no CUDA device (no CPU fallback)");
  if (device < 0 || device >= ndev) return p2s_internal_fail(P2S_INVALID_ARG, "bad device");
  DCUDA(cudaSetDevice(device));

  auto* c = new p2s_direct_ctx;
  c->pb = *spec;
  c->device = device;
  c->Nt = spec->order[0] * spec->order[1] * spec->order[2];
  c->n_tot = spec->n_comp * c->Nt;
  c->P = spec->n_comp * spec->n_comp;
  c->S = spec->n_terms;
  c->Q = static_cast<int64_t>(spec->nq[0]) * spec->nq[1] * spec->nq[2];
  c->alpha_per_elem = static_cast<int64_t>(c->P) * c->S * c->Q;
  auto bail = [&](p2s_status st) {
    p2s_direct_destroy(c);
    return st;
  };

  // 1-D tables per direction: value / derivative, unweighted and weighted
  std::vector<double> x[3], w[3];
  for (int d = 0; d < 3; ++d) p2s::gauss_legendre_ld(spec->nq[d], x[d], w[d]);
  const size_t tb = sizeof(double) * static_cast<size_t>(c->Q) * c->Nt;
  double* d_1d = nullptr;
  size_t one_d = 0;
  for (int d = 0; d < 3; ++d) one_d += static_cast<size_t>(spec->order[d]) * spec->nq[d];
  if (cudaMalloc(&d_1d, sizeof(double) * one_d * 2) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "p2s_direct_create: cudaMalloc"));
  for (int s = 0; s < c->S; ++s)
    for (int side = 0; side < 2; ++side) {  // 0 test (row), 1 trial (column, weighted)
      std::vector<double> host(one_d);
      size_t off[3], o = 0;
      for (int d = 0; d < 3; ++d) {
        off[d] = o;
        const int kind = spec->kind[s][d], N = spec->order[d], nq = spec->nq[d];
        const bool deriv = side == 0 ? (kind == p2s::DD || kind == p2s::DP)
                                     : (kind == p2s::DD || kind == p2s::PD);
        const bool conf = spec->basis == P2S_BASIS_CONFORMING;
        std::vector<long double> P(static_cast<size_t>(N) + 2), dP(static_cast<size_t>(N) + 2);
        for (int q = 0; q < nq; ++q) {
          p2s::legendre_ld(N + 1, x[d][q], P.data(), dP.data());
          for (int m = 0; m < N; ++m) {
            long double v = 0.0L;
            if (conf) {  // phi_m = sum_i R P_{sup(m, i)} (reference conforming_matrix)
              for (int i = 0; i < 2; ++i) {
                const int a = p2s::conf_sup(m, i);
                v += p2s::conf_r(m, i) * (deriv ? dP[a] : P[a]);
              }
            } else {
              v = deriv ? dP[m] : P[m];
            }
            if (side == 1) v *= static_cast<long double>(w[d][q]);
            host[o + static_cast<size_t>(m) * nq + q] = static_cast<double>(v);
          }
        }
        o += static_cast<size_t>(N) * nq;
      }
      double* dst = nullptr;
      if (cudaMalloc(&dst, tb) != cudaSuccess) {
        cudaFree(d_1d);
        return bail(cuda_fail(cudaGetLastError(), "p2s_direct_create: basis tables"));
      }
      (side == 0 ? c->d_test : c->d_trial)[s] = dst;
      if (cudaMemcpy(d_1d, host.data(), sizeof(double) * one_d, cudaMemcpyHostToDevice) !=
          cudaSuccess) {
        cudaFree(d_1d);
        return bail(cuda_fail(cudaGetLastError(), "p2s_direct_create: upload"));
      }
      direct_basis_kernel<<<1184, 256>>>(dst, d_1d + off[0], d_1d + off[1], d_1d + off[2],
                                         spec->order[0], spec->order[1], spec->order[2],
                                         spec->nq[0], spec->nq[1], spec->nq[2]);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(d_1d);
        return bail(cuda_fail(cudaGetLastError(), "direct_basis_kernel"));
      }
    }
  cudaFree(d_1d);
  // W scratch: as many elements as fit in ~1 GiB (at least one)
  c->chunk = std::max<int64_t>(1, (int64_t(1) << 30) / static_cast<int64_t>(tb));
  if (cudaMalloc(&c->d_W, tb * static_cast<size_t>(c->chunk)) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "p2s_direct_create: W scratch"));
  if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS)
    return bail(p2s_internal_fail(P2S_CUDA_ERROR, "p2s_direct_create: cublasCreate"));
  *out = c;
  return P2S_OK;
}

void p2s_direct_destroy(p2s_direct_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (int s = 0; s < P2S_MAX_TERMS; ++s) {
    if (c->d_test[s]) cudaFree(c->d_test[s]);
    if (c->d_trial[s]) cudaFree(c->d_trial[s]);
  }
  if (c->d_W) cudaFree(c->d_W);
  if (c->blas) cublasDestroy(c->blas);
  delete c;
}

p2s_status p2s_direct_fill(p2s_direct_ctx* c, const double* d_alpha, double* d_M, int64_t ld_M,
                           int64_t n_elem, void* stream) {
  if (!c) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_fill: null context");
  if (n_elem < 0 || ld_M < c->n_tot)
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_fill: n_elem >= 0, ld_M >= n_tot");
  if (n_elem == 0) return P2S_OK;
  if (!d_alpha || !d_M) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_direct_fill: null buffer");
  DCUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cublasSetStream(c->blas, st) != CUBLAS_STATUS_SUCCESS)
    return p2s_internal_fail(P2S_CUDA_ERROR, "cublasSetStream");
  const int Nt = c->Nt, nc = c->pb.n_comp;
  const int64_t mstride = static_cast<int64_t>(c->n_tot) * ld_M;
  const double one = 1.0, zero = 0.0;
  for (int64_t e0 = 0; e0 < n_elem; e0 += c->chunk) {
    const int nb = static_cast<int>(std::min(c->chunk, n_elem - e0));
    for (int pair = 0; pair < c->P; ++pair) {
      const int gi = pair / nc, gj = pair % nc;
      double* Mb = d_M + e0 * mstride + static_cast<int64_t>(gi) * Nt * ld_M + gj * Nt;
      for (int s = 0; s < c->S; ++s) {
        const int64_t aoff = (static_cast<int64_t>(pair) * c->S + s) * c->Q;
        direct_scale_kernel<<<dim3(296, static_cast<unsigned>(nb)), 256, 0, st>>>(
            c->d_W, d_alpha + e0 * c->alpha_per_elem, c->d_trial[s], c->Q, Nt, c->alpha_per_elem,
            aoff);
        DCUDA(cudaGetLastError());
        // column-major view: M_block^T (Nt x Nt, ld ld_M) = W^T-view (Nt x Q) * B_test-view^T
        const cublasStatus_t bs = cublasDgemmStridedBatched(
            c->blas, CUBLAS_OP_N, CUBLAS_OP_T, Nt, Nt, static_cast<int>(c->Q), &one, c->d_W, Nt,
            c->Q * Nt, c->d_test[s], Nt, 0, s == 0 ? &zero : &one, Mb, static_cast<int>(ld_M),
            mstride, nb);
        if (bs != CUBLAS_STATUS_SUCCESS)
          return p2s_internal_fail(P2S_CUDA_ERROR,
                                   "p2s_direct_fill: cublasDgemmStridedBatched status " +
                                       std::to_string(static_cast<int>(bs)));
      }
    }
  }
  return P2S_OK;
}

}  // extern "C"
