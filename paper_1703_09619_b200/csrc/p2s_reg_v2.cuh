// p2s_reg_v2.cuh -- launchers and registry-entry factories of the shape-
// specialised two-stage kernels (contract_v2_kernel, moments_v2_kernel),
// shared by the ahead-of-time registry (p2s_reg_v2.cu) and generated modules.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "p2s_launch.cuh"
#include "p2s_reg_common.cuh"

namespace p2s {
namespace reg {

template <class Sh>
cudaError_t launch_v2(const V2Args& a, const std::vector<double>& packed, cudaStream_t st,
                      int num_sms) {
  V2Params<Sh> p;
  p.I = a.I;
  p.M = a.M;
  p.ldM = a.ldM;
  p.mat_stride = a.n_tot * a.ldM;
  p.n_units = a.n_elem * a.P;
  p.nc = a.nc;
  p.P = a.P;
  p.Nt = a.Nt;
  p.mom_per_elem = a.mom_per_elem;
  p.amma = a.amma;
  p.vec2 = vec2_ok(a.M, a.ldM);
  std::memcpy(p.cu, packed.data(), sizeof(double) * Sh::ctot(0));
  std::memcpy(p.cv, packed.data() + Sh::ctot(0), sizeof(double) * Sh::ctot(1));
  std::memcpy(p.cw, packed.data() + Sh::ctot(0) + Sh::ctot(1), sizeof(double) * Sh::ctot(2));
  if (p.n_units == 0) return cudaSuccess;
  int blocks_per_sm = 0;
  cudaError_t e = kernel_prepare(contract_v2_kernel<Sh>, v2_smem<Sh>(), Sh::THREADS, false, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  const int64_t grid = Sh::PERSIST
                           ? std::min<int64_t>(p.n_units, static_cast<int64_t>(blocks_per_sm) * num_sms)
                           : p.n_units;
  p.prefetch_stride = static_cast<int64_t>(blocks_per_sm) * num_sms;
  if (const char* v = tuning_env("P2S_V2_NOPREFETCH"))
    if (v[0] == '1') p.prefetch_stride = 0;
  contract_v2_kernel<Sh><<<static_cast<unsigned>(grid), Sh::THREADS, v2_smem<Sh>(), st>>>(p);
  return cudaGetLastError();
}


template <class Sh>
V2Entry make_v2() {
  V2Entry r{};
  for (int d = 0; d < 3; ++d) r.order[d] = Sh::N(d);
  r.S = Sh::S;
  for (int s = 0; s < Sh::S; ++s)
    for (int d = 0; d < 3; ++d) r.kinds[s][d] = Sh::kind(s, d);
  r.launch = &launch_v2<Sh>;
  r.pack = &pack_v2<Sh>;
  r.mma_pack = &pack_mma<Sh>;
  r.smem = v2_smem<Sh>();
  r.desc = stage_c_desc<Sh>();
  return r;
}


template <class Ms>
cudaError_t launch_mv2(const double* alpha, double* I, int64_t n_elem, int P, int64_t mom_per_elem,
                       const std::vector<double>& packed, cudaStream_t st) {
  MV2Params<Ms> p;
  p.alpha = alpha;
  p.I = I;
  p.P = P;
  p.n_units = n_elem * P * Ms::S;
  p.mom_per_elem = mom_per_elem;
  std::memcpy(p.tab, packed.data(), sizeof(double) * Ms::TALL);
  if (p.n_units == 0) return cudaSuccess;
  cudaError_t e = kernel_prepare(moments_v2_kernel<Ms>, Ms::SMEM, Ms::THREADS);
  if (e != cudaSuccess) return e;
  moments_v2_kernel<Ms><<<static_cast<unsigned>(p.n_units), Ms::THREADS, Ms::SMEM, st>>>(p);
  return cudaGetLastError();
}


template <class Ms>
MV2Entry make_mv2() {
  MV2Entry r{};
  for (int d = 0; d < 3; ++d) {
    r.order[d] = Ms::N(d);
    r.nq[d] = Ms::Q(d);
  }
  r.S = Ms::S;
  for (int s = 0; s < Ms::S; ++s)
    for (int d = 0; d < 3; ++d) r.kinds[s][d] = Ms::kind(s, d);
  r.launch = &launch_mv2<Ms>;
  r.pack = &pack_mv2<Ms>;
  return r;
}

}  // namespace reg
}  // namespace p2s
