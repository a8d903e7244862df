// p2s_reg_generic.cu -- runtime-shaped kernels: contract_kernel<UCfg> registry (compile-time u direction) and moments_kernel<KMAX>.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "p2s_kernels.cuh"
#include "p2s_launch.cuh"
#include "p2s_registry.hpp"

namespace p2s {
namespace reg {

// ------------------------------------------------------------ contraction registry


template <class Cfg>
cudaError_t launch_contract(const ContractArgs& a, const Plan& pl, cudaStream_t st) {
  ContractParams<Cfg> p;
  std::memset(&p, 0, sizeof(p));
  p.I = a.I;
  p.M = a.M;
  p.ldM = a.ldM;
  p.mat_stride = a.n_tot * a.ldM;
  p.nc = a.nc;
  p.P = a.P;
  p.Nv = a.Nv;
  p.Nw = a.Nw;
  p.Nt = a.Nt;
  p.G = pl.G;
  p.NG = pl.NG;
  p.mom_per_elem = a.mom_per_elem;
  p.mom_per_pair = a.mom_per_pair;
  p.i_doubles = static_cast<int>(a.mom_per_pair);
  int ao = 0, co = 0;
  for (int s = 0; s < Cfg::S; ++s) {
    p.Kv[s] = a.Kv[s];
    p.Kw[s] = a.Kw[s];
    p.kind_v[s] = a.kind_v[s];
    p.kind_w[s] = a.kind_w[s];
    p.mom_off[s] = static_cast<int>(a.mom_off[s]);
    p.a_off[s] = ao;
    ao += pl.G * Cfg::K(s) * a.Nv * a.Kw[s];
    p.cv_off[s] = co;
    co += a.Nv * a.Nv * a.Kv[s];
    p.cw_off[s] = co;
    co += a.Nw * a.Nw * a.Kw[s];
    p.Cv[s] = a.Cv[s];
    p.Cw[s] = a.Cw[s];
  }
  p.a_doubles = (ao + 1) & ~1;
  p.c_doubles = (co + 1) & ~1;
  std::memcpy(p.cu, a.cu_packed, sizeof(double) * Cfg::CTOT);
  const int64_t n_cta = a.n_elem * a.P * pl.NG;
  p.n_cta = n_cta;
  if (n_cta == 0) return cudaSuccess;
  cudaError_t e = kernel_prepare(contract_kernel<Cfg>, 227 * 1024, 256);
  if (e != cudaSuccess) return e;
  contract_kernel<Cfg><<<static_cast<unsigned>(n_cta), pl.threads, pl.smem, st>>>(p);
  return cudaGetLastError();
}

template <class Cfg>
std::vector<double> pack_cu(const std::vector<const std::vector<double>*>& dense) {
  // dense[s] = [NU][NU][K_s]
  std::vector<double> out(static_cast<size_t>(Cfg::CTOT), 0.0);
  for (int s = 0; s < Cfg::S; ++s) {
    const int K = Cfg::K(s), kd = Cfg::kind(s);
    for (int a = 0; a < Cfg::NU; ++a)
      for (int b = 0; b < Cfg::NU; ++b) {
        const int lo = band_lo(kd, a, b), cnt = band_count(kd, a, b);
        for (int j = 0; j < cnt; ++j)
          out[static_cast<size_t>(Cfg::coff(s, a, b) + j)] =
              (*dense[static_cast<size_t>(s)])[(static_cast<size_t>(a) * Cfg::NU + b) * K + lo +
                                               band_step(kd, a, b) * j];
      }
  }
  return out;
}


template <int NU, int... KINDS>
RegEntry make_entry() {
  using Cfg = UCfg<NU, KINDS...>;
  RegEntry r{};
  r.NU = NU;
  r.S = Cfg::S;
  const int ks[] = {KINDS...};
  for (int s = 0; s < Cfg::S; ++s) r.kinds[s] = ks[s];
  r.launch = &launch_contract<Cfg>;
  r.pack = &pack_cu<Cfg>;
  r.ktot = Cfg::KTOT;
  return r;
}

// Compiled shapes: (N_u, u-kind of each term).  The v / w orders, kinds,
// component count and quadrature sizes are runtime parameters.
const std::vector<RegEntry>& registry() {
  static const std::vector<RegEntry> reg = {
      make_entry<1, PP>(),          make_entry<2, PP>(),      make_entry<3, PP>(),
      make_entry<4, PP>(),          make_entry<5, PP>(),      make_entry<6, PP>(),
      make_entry<8, PP>(),          make_entry<10, PP>(),
      make_entry<2, PP, DD>(),      make_entry<3, PP, DD>(),  make_entry<4, PP, DD>(),
      make_entry<5, PP, DD>(),      make_entry<6, PP, DD>(),  make_entry<8, PP, DD>(),
      make_entry<10, PP, DD>(),
      make_entry<3, DD>(),          make_entry<3, DP>(),      make_entry<3, PD>(),
      make_entry<4, DP, PD>(),      make_entry<3, PP, DP>(),  make_entry<4, PP, DD, DP, PD>(),
      // conforming basis (kind | kConforming)
      make_entry<3, PP | kConforming, DD | kConforming>(), make_entry<4, PP | kConforming>(),
      make_entry<6, PP | kConforming, DD | kConforming>(),
      make_entry<4, DP | kConforming, PD | kConforming>(),
  };
  return reg;
}


// ------------------------------------------------------------ moment launch

template <int KMAX>
cudaError_t launch_moments_k(const MomentParams& p, size_t smem, cudaStream_t st) {
  cudaError_t e = kernel_prepare(moments_kernel<KMAX>, 227 * 1024, 256);
  if (e != cudaSuccess) return e;
  moments_kernel<KMAX><<<static_cast<unsigned>(p.n_units), 256, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_moments(int kmax, const MomentParams& p, size_t smem, cudaStream_t st) {
  if (p.n_units == 0) return cudaSuccess;
  switch (kmax) {
    case 8: return launch_moments_k<8>(p, smem, st);
    case 12: return launch_moments_k<12>(p, smem, st);
    case 16: return launch_moments_k<16>(p, smem, st);
    case 20: return launch_moments_k<20>(p, smem, st);
    case 24: return launch_moments_k<24>(p, smem, st);
    default: return launch_moments_k<32>(p, smem, st);
  }
}

}  // namespace reg
}  // namespace p2s
