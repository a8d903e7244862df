// p2s_reg_fused.cuh -- launcher and registry-entry factory of the fused fill
// kernel (fill_fused_kernel, p2s_fused.cuh), shared by the ahead-of-time
// registry (p2s_reg_fused.cu) and generated per-shape modules (p2s_jit.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "p2s_fused.cuh"
#include "p2s_launch.cuh"
#include "p2s_reg_common.cuh"

namespace p2s {
namespace reg {

// GEO > 0: `alpha` is the geometry records and the kernel computes the coupling
// factors itself (xq = the GL nodes u, v, w appended to mpack); GEO == 2 launches
// one thread-block cluster of P CTAs per element (non-portable size for P = 9)
template <class Sh, class Ms, int GEO = 0, bool PF = true>
cudaError_t launch_fused(const double* alpha, double* M, int64_t ldM, int64_t n_tot, int64_t n_elem,
                         int nc, int P, int Nt, const std::vector<double>& cpack,
                         const std::vector<double>& mpack, const double* amma, cudaStream_t st,
                         int num_sms, int* bad) {
  FusedParams<Sh, Ms> p;
  p.geom = GEO ? alpha : nullptr;
  p.bad = bad;
  if constexpr (GEO != 0)
    std::memcpy(p.xq, mpack.data() + Ms::TALL, sizeof(double) * (Ms::Q(0) + Ms::Q(1) + Ms::Q(2)));
  p.c.I = nullptr;
  p.c.M = M;
  p.c.ldM = ldM;
  p.c.mat_stride = n_tot * ldM;
  p.c.n_units = n_elem * P;
  p.c.nc = nc;
  p.c.P = P;
  p.c.Nt = Nt;
  p.c.mom_per_elem = 0;
  p.c.amma = amma;
  p.c.vec2 = vec2_ok(M, ldM);
  p.c.prefetch_stride = 0;  // (contract_v2 only)
  std::memcpy(p.c.cu, cpack.data(), sizeof(double) * Sh::ctot(0));
  std::memcpy(p.c.cv, cpack.data() + Sh::ctot(0), sizeof(double) * Sh::ctot(1));
  std::memcpy(p.c.cw, cpack.data() + Sh::ctot(0) + Sh::ctot(1), sizeof(double) * Sh::ctot(2));
  p.alpha = alpha;
  p.prefetch_stride = 0;
  std::memcpy(p.tab, mpack.data(), sizeof(double) * Ms::TALL);
  if (p.c.n_units == 0) return cudaSuccess;
  constexpr size_t smem = FusedLayout<Sh, Ms, GEO>::SMEM;
  int blocks_per_sm = 0;
  cudaError_t e = kernel_prepare(fill_fused_kernel<Sh, Ms, GEO>, smem, Sh::THREADS, GEO == 2, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  const int64_t resident = static_cast<int64_t>(blocks_per_sm) * num_sms;
  const int64_t grid = Sh::PERSIST ? std::min<int64_t>(p.c.n_units, resident) : p.c.n_units;
  // L2 prefetch of the alpha of the unit that takes this SM slot next (PF, per
  // shape; P2S_PREFETCH_AHEAD=k overrides): C2 +0.6 %, C4 -1.5 % (L2 pressure)
  p.prefetch_stride = PF ? resident : 0;
  if (const char* v = tuning_env("P2S_PREFETCH_AHEAD")) p.prefetch_stride = resident * std::max(0, std::atoi(v));
  if constexpr (GEO == 2) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(p.c.n_units));
    cfg.blockDim = dim3(Sh::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(P);  // one element per cluster
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fill_fused_kernel<Sh, Ms, GEO>, p);
  }
  fill_fused_kernel<Sh, Ms, GEO><<<static_cast<unsigned>(grid), Sh::THREADS, smem, st>>>(p);
  return cudaGetLastError();
}


template <class Sh, class Ms, bool WITH_GEO = false, bool PREFER_TWO_STAGE = false, bool PF = true>
FusedEntry make_fused() {
  FusedEntry r{};
  for (int d = 0; d < 3; ++d) {
    r.order[d] = Sh::N(d);
    r.nq[d] = Ms::Q(d);
  }
  r.S = Sh::S;
  for (int s = 0; s < Sh::S; ++s)
    for (int d = 0; d < 3; ++d) r.kinds[s][d] = Sh::kind(s, d);
  r.launch = &launch_fused<Sh, Ms, 0, PF>;
  r.launch_geo = r.launch_geo_cluster = nullptr;
  if constexpr (WITH_GEO) {
    r.launch_geo = &launch_fused<Sh, Ms, 1>;
    r.launch_geo_cluster = &launch_fused<Sh, Ms, 2>;
  }
  r.cpack = &pack_v2<Sh>;
  r.mpack = &pack_mv2<Ms>;
  r.mma_pack = &pack_mma<Sh>;
  r.desc = stage_c_desc<Sh>();
  r.prefer_two_stage = PREFER_TWO_STAGE;
  return r;
}

}  // namespace reg
}  // namespace p2s
