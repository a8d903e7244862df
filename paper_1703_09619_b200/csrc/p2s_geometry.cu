// p2s_geometry.cu -- coupling factors sampled on the device from element
// geometry (the 3-D analogue of build_element_quad,
// assembly.cpp:51-119): alpha_s^{gi gj}(q) = alpha_mat detJ (J^T J)^-1 (even s)
// and alpha_mat (J^T J) / detJ (odd s) of a hexahedron's trilinear map, at the
// Gauss-Legendre points, from a 28-double record per element (8 corners, the
// material's (a, b, c, phi); layout in include/p2s_b200.h).
//
// Grid (element, slab of 256 points): each CTA turns the record into the map's
// polynomial form x(u,v,w) = A0 + A1 u + A2 v + A3 w + A4 uv + A5 uw + A6 vw +
// A7 uvw per component (shared memory), so a point's Jacobian is 27 FMAs; one
// reciprocal of detJ per point replaces the nine divisions; a thread owns one
// point (u fastest) and writes its P*S coupling values with coalesced stores.
// Compiled with FMA contraction (unlike the seeded generator p2s_alpha.cu,
// which rounds like the host): values agree with it to ~1e-15 relative.
#include <cuda_runtime.h>

#include "p2s_launch.cuh"

#include <algorithm>
#include <cstdlib>

#include <cstdint>

namespace p2s {

namespace {

// NC components, S terms compile-time: the pair/term loops unroll and the 3x3
// matrices stay in registers
template <int NC, int S>
__global__ void __launch_bounds__(256) alpha_geometry_fast_kernel(
    double* __restrict__ alpha, const double* __restrict__ geom, const double* __restrict__ x0,
    const double* __restrict__ x1, const double* __restrict__ x2, int nq0, int nq1, int nq2,
    int64_t per_elem, int* __restrict__ bad) {
  __shared__ double A[8][3];  // polynomial coefficients of the map, per component
  __shared__ double mat[4];
  __shared__ double xs[3][64];
  const int64_t e = blockIdx.x;
  const double* g = geom + e * 28;
  if (threadIdx.x < 24) {
    // corner c at (s0, s1, s2), s_d = +-1 (bit d of c): N_c = prod (1 + s_d r_d) / 8
    // -> coefficient of monomial m (bit d set = factor r_d) is sum_c X_c prod_{d in m} s_d / 8
    const int m = threadIdx.x / 3, comp = threadIdx.x % 3;
    double acc = 0.0;
    for (int c = 0; c < 8; ++c) {
      double sgn = 1.0;
      for (int d = 0; d < 3; ++d)
        if ((m >> d) & 1) sgn *= ((c >> d) & 1) ? 1.0 : -1.0;
      acc += sgn * __ldg(g + c * 3 + comp);
    }
    A[m][comp] = 0.125 * acc;
  } else if (threadIdx.x < 28) {
    mat[threadIdx.x - 24] = __ldg(g + threadIdx.x);
  }
  for (int i = threadIdx.x; i < nq0 + nq1 + nq2; i += blockDim.x) {
    if (i < nq0)
      xs[0][i] = x0[i];
    else if (i < nq0 + nq1)
      xs[1][i - nq0] = x1[i - nq0];
    else
      xs[2][i - nq0 - nq1] = x2[i - nq0 - nq1];
  }
  __syncthreads();
  const int npts = nq0 * nq1 * nq2;
  double* ae = alpha + e * per_elem;
  for (int q = blockIdx.y * blockDim.x + threadIdx.x; q < npts; q += gridDim.y * blockDim.x) {
    const int i = q % nq0, j = (q / nq0) % nq1, k = q / (nq0 * nq1);
    const double u = xs[0][i], v = xs[1][j], w = xs[2][k];
    // monomials 1:u 2:v 4:w 3:uv 5:uw 6:vw 7:uvw (bit d = r_d)
    double J[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      J[c][0] = A[1][c] + v * A[3][c] + w * A[5][c] + v * w * A[7][c];
      J[c][1] = A[2][c] + u * A[3][c] + w * A[6][c] + u * w * A[7][c];
      J[c][2] = A[4][c] + u * A[5][c] + v * A[6][c] + u * v * A[7][c];
    }
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double G[3][3];
#pragma unroll
    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
      for (int a2 = a1; a2 < 3; ++a2) {
        G[a1][a2] = J[0][a1] * J[0][a2] + J[1][a1] * J[1][a2] + J[2][a1] * J[2][a2];
        G[a2][a1] = G[a1][a2];
      }
    // the reference throws GeometryError on J <= 0 (assembly.cpp:95-99): flag it
    if (!(det > 0.0)) atomicOr(bad, 1);
    const double rdet = 1.0 / det;
    const double am = 1.0 + 0.3 * sin(mat[0] * u + mat[1] * v + mat[2] * w + mat[3]);
    const double ms = am * rdet;  // mass: am detJ (G^-1) = am cof(G) / detJ (det G = detJ^2)
    double Gi[3][3];
    Gi[0][0] = G[1][1] * G[2][2] - G[1][2] * G[2][1];
    Gi[0][1] = G[0][2] * G[2][1] - G[0][1] * G[2][2];
    Gi[0][2] = G[0][1] * G[1][2] - G[0][2] * G[1][1];
    Gi[1][1] = G[0][0] * G[2][2] - G[0][2] * G[2][0];
    Gi[1][2] = G[0][2] * G[1][0] - G[0][0] * G[1][2];
    Gi[2][2] = G[0][0] * G[1][1] - G[0][1] * G[1][0];
    Gi[1][0] = Gi[0][1];
    Gi[2][0] = Gi[0][2];
    Gi[2][1] = Gi[1][2];
#pragma unroll
    for (int gi = 0; gi < NC; ++gi)
#pragma unroll
      for (int gj = 0; gj < NC; ++gj) {
        const double mass = ms * Gi[gi][gj], curl = ms * G[gi][gj];
        double* o = ae + static_cast<int64_t>(gi * NC + gj) * S * npts + q;
#pragma unroll
        for (int s = 0; s < S; ++s) o[static_cast<int64_t>(s) * npts] = (s % 2 == 0) ? mass : curl;
      }
  }
}

}  // namespace

cudaError_t launch_alpha_geometry_fast(double* alpha, const double* geom, const double* const x[3],
                                       const int nq[3], int nc, int S, int64_t n, int64_t per_elem,
                                       int* bad, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (nq[0] > 64 || nq[1] > 64 || nq[2] > 64) return cudaErrorInvalidValue;
  // points per thread (P2S_GEO_PPT, default 4): the per-CTA prologue (record ->
  // polynomial map, nodes) is amortised over several points per thread
  int ppt = 4;
  if (const char* v = tuning_env("P2S_GEO_PPT")) ppt = std::max(1, std::atoi(v));
  const unsigned slabs = static_cast<unsigned>((nq[0] * nq[1] * nq[2] + 256 * ppt - 1) / (256 * ppt));
  const dim3 grid(static_cast<unsigned>(n), slabs);
#define P2S_GEO_CASE(NC_, S_)                                                                         \
  if (nc == NC_ && S == S_) {                                                                       \
    alpha_geometry_fast_kernel<NC_, S_><<<grid, 256, 0, stream>>>(alpha, geom, x[0], x[1], x[2], nq[0], \
                                                                  nq[1], nq[2], per_elem, bad);          \
    return cudaGetLastError();                                                                      \
  }
  P2S_GEO_CASE(1, 1) P2S_GEO_CASE(1, 2) P2S_GEO_CASE(1, 3) P2S_GEO_CASE(1, 4)
  P2S_GEO_CASE(3, 1) P2S_GEO_CASE(3, 2) P2S_GEO_CASE(3, 3) P2S_GEO_CASE(3, 4)
#undef P2S_GEO_CASE
  return cudaErrorInvalidValue;
}

}  // namespace p2s
