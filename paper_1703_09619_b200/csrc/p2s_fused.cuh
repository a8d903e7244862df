// p2s_fused.cuh -- the fill as ONE persistent kernel: per (element, pair)
// unit the CTA computes the moments of every term from alpha straight into
// shared memory (moments_unit, p2s_moments_v2.cuh), then contracts them and
// streams the element matrix out (v2_unit, p2s_contract_v2.cuh).  HBM traffic
// is alpha read + M write only; the FP64-heavy moment phase of one CTA
// overlaps the store-heavy contraction phase of the other CTA(s) on the SM.
#pragma once

#include "p2s_contract_v2.cuh"
#include "p2s_moments_v2.cuh"

namespace p2s {

template <class Sh, class Ms>
struct FusedParams {
  V2Params<Sh> c;      // contraction part (c.I unused)
  const double* alpha;
  const double* geom;  // GEO kernels: element geometry records (28 doubles each)
  double xq[Ms::Q(0) + Ms::Q(1) + Ms::Q(2)];  // GL nodes u, v, w (GEO kernels)
  int64_t prefetch_stride;  // resident CTAs on the GPU (non-persistent launch)
  double tab[Ms::TALL];
};

template <class Sh, class Ms>
struct FusedLayout {
  static_assert(Sh::MPP == Ms::MPP, "moment block layouts differ");
  static constexpr int AB = Sh::A_DBL + Sh::B_DBL;
  static constexpr int MS = Ms::scratch_all_dbl();
  static constexpr int WORK = AB > MS ? AB : MS;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(Sh::MPP + WORK + mma_smem_dbl<Sh>());
};

// GEO: the moment phase computes the coupling factors from the element's
// geometry record (p2s_fill_geometry) instead of reading alpha from HBM.
template <class Sh, class Ms, bool GEO = false>
__global__ void __launch_bounds__(Sh::THREADS, Sh::MINB)
    fill_fused_kernel(const __grid_constant__ FusedParams<Sh, Ms> p) {
  extern __shared__ __align__(16) double sm[];
  double* Ibuf = sm;
  double* Abuf = Ibuf + Sh::MPP;
  double* Bbuf = Abuf + Sh::A_DBL;
  const MmaSmem mm = mma_carve<Sh>(Abuf + FusedLayout<Sh, Ms>::WORK);
  if constexpr (Sh::MMA)  // visible to stage C after the moment phase's barriers
    mma_setup<Sh>(p.c.amma, const_cast<double*>(mm.A), const_cast<int2*>(mm.ctab));
  constexpr int slab = Ms::Q(0) * Ms::Q(1) * Ms::Q(2);
  auto do_unit = [&](int64_t unit, int64_t stride) {
    const int64_t e = unit / p.c.P;
    const int pair = static_cast<int>(unit - e * p.c.P);
    const int gci = pair / p.c.nc, gcj = pair - gci * p.c.nc;
    const double* a = p.alpha + unit * (static_cast<int64_t>(Ms::S) * slab);
    if constexpr (GEO) {
      __shared__ GeoUnit geo;
      geo_unit_setup(p.geom + e * 28, gci, gcj, &geo);
      __syncthreads();
      static_assert(!Ms::WFIRST, "geometry mode uses the u-first pass order");
      moments_all_terms<Ms, Sh::THREADS, true>(nullptr, p.tab, Abuf, Ibuf, &geo, p.xq);
    } else {
    // warm L2 with alpha `stride` units ahead while this unit is processed
    if constexpr ((Ms::S * slab) % 2 == 0)  // 16-B granularity of the bulk prefetch
      if (threadIdx.x == 0 && unit + stride < p.c.n_units)
        prefetch_l2(a + stride * Ms::S * slab, static_cast<uint32_t>(Ms::S * slab * 8));
    if constexpr (Ms::WFIRST)
      moments_all_terms_wfirst<Ms, Sh::THREADS>(a, p.tab, Abuf, Ibuf);
    else
      moments_all_terms<Ms, Sh::THREADS>(a, p.tab, Abuf, Ibuf);
    }
    double* Mbase =
        p.c.M + e * p.c.mat_stride + static_cast<int64_t>(gci * p.c.Nt) * p.c.ldM + gcj * p.c.Nt;
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
