// p2s_fused.cuh -- the fill as ONE persistent kernel: per (element, pair)
// unit the CTA computes the moments of every term from alpha straight into
// shared memory (moments_unit, p2s_moments_v2.cuh), then contracts them and
// streams the element matrix out (v2_unit, p2s_contract_v2.cuh).  HBM traffic
// is alpha read + M write only; the FP64-heavy moment phase of one CTA
// overlaps the store-heavy contraction phase of the other CTA(s) on the SM.
#pragma once

#include <cooperative_groups.h>

#include "p2s_contract_v2.cuh"
#include "p2s_contract_wl.cuh"
#include "p2s_moments_v2.cuh"

namespace p2s {

template <class Sh, class Ms>
struct FusedParams {
  V2Params<Sh> c;      // contraction part (c.I unused)
  const double* alpha;
  const double* geom;  // GEO kernels: element geometry records (28 doubles each)
  int* bad;            // GEO kernels: non-positive Jacobian flag
  double xq[Ms::Q(0) + Ms::Q(1) + Ms::Q(2)];  // GL nodes u, v, w (GEO kernels)
  int64_t prefetch_stride;  // resident CTAs on the GPU (non-persistent launch)
  double tab[Ms::TALL];
};

// GEO = 2 (cluster mode): the unit's alpha lives in shared memory over the
// moment scratch's second buffer (T2, written only after pass u consumed alpha)
template <class Sh, class Ms, int GEO = 0>
struct FusedLayout {
  static_assert(Sh::MPP == Ms::MPP, "moment block layouts differ");
  static constexpr int AB = Sh::A_DBL + Sh::B_DBL;
  static constexpr int MS = Ms::scratch_all_dbl();
  static constexpr int AOFF = Ms::t1off(Ms::S);  // alpha offset inside WORK (GEO == 2)
  static constexpr int MSG = GEO == 2 ? (AOFF + Ms::S * Ms::Q(0) * Ms::Q(1) * Ms::Q(2) > MS
                                             ? AOFF + Ms::S * Ms::Q(0) * Ms::Q(1) * Ms::Q(2)
                                             : MS)
                                      : MS;
  static constexpr int WORK = AB > MSG ? AB : MSG;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(Sh::MPP + WORK + mma_smem_dbl<Sh>());
};

// Cluster mode, geometry phase: the P CTAs of an element (one per component
// pair, cluster rank = pair) split the element's quadrature points; each
// computes the point's Jacobian, Gram matrix and cofactors once and stores
// every pair's coupling values into that pair's CTA through distributed shared
// memory (mapa / st.shared::cluster).  NC compile-time (1 or 3).
template <class Ms, int NC, int NTHR>
__device__ __forceinline__ void geo_cluster_phase(const GeoUnit& g, const double* xq, double* as,
                                                  int rank, int P) {
  namespace cg = cooperative_groups;
  constexpr int QU = Ms::Q(0), QV = Ms::Q(1), QW = Ms::Q(2), S = Ms::S;
  constexpr int slab = QU * QV * QW;
  cg::cluster_group cl = cg::this_cluster();
  double* peer[NC * NC];
#pragma unroll
  for (int pp = 0; pp < NC * NC; ++pp) peer[pp] = cl.map_shared_rank(as, pp);
  const int per = (slab + P - 1) / P;
  const int q1 = (rank + 1) * per < slab ? (rank + 1) * per : slab;
  for (int q = rank * per + static_cast<int>(threadIdx.x); q < q1; q += NTHR) {
    const int i = q % QU, j = (q / QU) % QV, k = q / (QU * QV);
    const double u = xq[i], v = xq[QU + j], w = xq[QU + QV + k];
    double J[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      J[c][0] = g.A[1][c] + v * g.A[3][c] + w * g.A[5][c] + v * w * g.A[7][c];
      J[c][1] = g.A[2][c] + u * g.A[3][c] + w * g.A[6][c] + u * w * g.A[7][c];
      J[c][2] = g.A[4][c] + u * g.A[5][c] + v * g.A[6][c] + u * v * g.A[7][c];
    }
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(det > 0.0)) atomicOr(g.bad, 1);
    double G[3][3];
#pragma unroll
    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
      for (int a2 = a1; a2 < 3; ++a2) {
        G[a1][a2] = J[0][a1] * J[0][a2] + J[1][a1] * J[1][a2] + J[2][a1] * J[2][a2];
        G[a2][a1] = G[a1][a2];
      }
    double C[3][3];  // cofactors (adjugate of the symmetric Gram matrix)
    C[0][0] = G[1][1] * G[2][2] - G[1][2] * G[2][1];
    C[0][1] = G[0][2] * G[2][1] - G[0][1] * G[2][2];
    C[0][2] = G[0][1] * G[1][2] - G[0][2] * G[1][1];
    C[1][1] = G[0][0] * G[2][2] - G[0][2] * G[2][0];
    C[1][2] = G[0][2] * G[1][0] - G[0][0] * G[1][2];
    C[2][2] = G[0][0] * G[1][1] - G[0][1] * G[1][0];
    C[1][0] = C[0][1];
    C[2][0] = C[0][2];
    C[2][1] = C[1][2];
    const double ms = (1.0 + 0.3 * sin(g.mat[0] * u + g.mat[1] * v + g.mat[2] * w + g.mat[3])) / det;
#pragma unroll
    for (int gi = 0; gi < NC; ++gi)
#pragma unroll
      for (int gj = 0; gj < NC; ++gj) {
        const double mass = ms * C[gi][gj], curl = ms * G[gi][gj];
        double* dst = peer[gi * NC + gj] + q;
#pragma unroll
        for (int s = 0; s < S; ++s) dst[s * slab] = (s % 2 == 0) ? mass : curl;
      }
  }
}

// The w-first moment pass reads alpha with loads that do not allocate in L1
// (ld.global.nc.L1::no_allocate; C4: 1.150 M vs 1.127 M elem/s, L2 read misses
// 29.7 M -> 19.4 M sectors per 2048 elements, profiles/r2_c4_alpha_noalloc.txt).
// Shape FLAGS bit 10 (AL1) restores the allocating loads for A/B runs.
template <class Sh>
constexpr bool alpha_no_allocate() {
  if constexpr (Sh::WLAST)
    return true;
  else
    return Sh::AL1 == 0;
}

// GEO: 0 alpha from HBM; 1 the moment phase computes the coupling factors
// from the element's geometry record per unit; 2 cluster mode (one cluster of
// P CTAs per element shares the per-point geometry through DSMEM).
template <class Sh, class Ms, int GEO = 0>
__global__ void __launch_bounds__(Sh::THREADS, Sh::MINB)
    fill_fused_kernel(const __grid_constant__ FusedParams<Sh, Ms> p) {
  extern __shared__ __align__(16) double sm[];
  double* Ibuf = sm;
  double* Abuf = Ibuf + Sh::MPP;
  double* Bbuf = Abuf + Sh::A_DBL;
  const MmaSmem mm = mma_carve<Sh>(Abuf + FusedLayout<Sh, Ms, GEO>::WORK);
  if constexpr (Sh::MMA)  // visible to stage C after the moment phase's barriers
    mma_setup<Sh>(p.c.amma, const_cast<double*>(mm.A), const_cast<int2*>(mm.ctab));
  constexpr int slab = Ms::Q(0) * Ms::Q(1) * Ms::Q(2);
  auto do_unit = [&](int64_t unit, int64_t stride) {
    const int64_t e = unit / p.c.P;
    const int pair = static_cast<int>(unit - e * p.c.P);
    const int gci = pair / p.c.nc, gcj = pair - gci * p.c.nc;
    const double* a = p.alpha + unit * (static_cast<int64_t>(Ms::S) * slab);
    if constexpr (GEO == 1) {
      __shared__ GeoUnit geo;
      geo_unit_setup(p.geom + e * 28, gci, gcj, &geo, p.bad);
      __syncthreads();
      static_assert(!Ms::WFIRST, "geometry mode uses the u-first pass order");
      moments_all_terms<Ms, Sh::THREADS, 1>(nullptr, p.tab, Abuf, Ibuf, &geo, p.xq);
    } else if constexpr (GEO == 2) {
      static_assert(!Ms::WFIRST, "geometry mode uses the u-first pass order");
      __shared__ GeoUnit geo;
      double* as = Abuf + FusedLayout<Sh, Ms, GEO>::AOFF;
      geo_unit_setup(p.geom + e * 28, gci, gcj, &geo, p.bad);
      cooperative_groups::this_cluster().sync();  // every CTA of the element resident, geo set
      if (p.c.nc == 3)
        geo_cluster_phase<Ms, 3, Sh::THREADS>(geo, p.xq, as, pair, p.c.P);
      else
        geo_cluster_phase<Ms, 1, Sh::THREADS>(geo, p.xq, as, pair, p.c.P);
      cooperative_groups::this_cluster().sync();  // the unit's alpha complete in shared memory
      moments_all_terms<Ms, Sh::THREADS, 2>(as, p.tab, Abuf, Ibuf);
    } else {
    // warm L2 with alpha `stride` units ahead while this unit is processed
    if constexpr ((Ms::S * slab) % 2 == 0)  // 16-B granularity of the bulk prefetch
      if (threadIdx.x == 0 && unit + stride < p.c.n_units)
        prefetch_l2(a + stride * Ms::S * slab, static_cast<uint32_t>(Ms::S * slab * 8));
    if constexpr (Ms::WFIRST)
      moments_all_terms_wfirst<Ms, Sh::THREADS, alpha_no_allocate<Sh>()>(a, p.tab, Abuf, Ibuf);
    else
      moments_all_terms<Ms, Sh::THREADS>(a, p.tab, Abuf, Ibuf);
    }
    double* Mbase =
        p.c.M + e * p.c.mat_stride + static_cast<int64_t>(gci * p.c.Nt) * p.c.ldM + gcj * p.c.Nt;
    if constexpr (Sh::WLAST)
      wl_unit<Sh>(p.c, Ibuf, Abuf, Bbuf, Mbase);
    else
      v2_unit<Sh>(p.c, Ibuf, Abuf, Bbuf, Mbase, []() {}, mm);
  };
  if constexpr (Sh::PERSIST) {
    for (int64_t unit = blockIdx.x; unit < p.c.n_units; unit += gridDim.x) do_unit(unit, gridDim.x);
  } else {
    // one unit per CTA; prefetch for the CTA that runs on this SM slot next
    if (blockIdx.x < p.c.n_units) do_unit(blockIdx.x, p.prefetch_stride);
  }
}

}  // namespace p2s
