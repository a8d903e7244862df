// p2s_reg_large.cuh -- table packing, launchers and registry-entry factory of
// the large-order path (p2s_large.cuh), shared by the ahead-of-time registry
// (p2s_reg_large.cu) and generated per-shape modules (p2s_jit.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "p2s_large.cuh"
#include "p2s_launch.cuh"
#include "p2s_reg_common.cuh"

namespace p2s {
namespace reg {

template <class Ls>
bool pack_large(const LargeArgs& a, LargePack& out) {
  out.tab.assign(static_cast<size_t>(Ls::TALL), 0.0);
  for (int d = 0; d < 3; ++d) {
    // shared rows: the term with the most kernel polynomials in this direction
    int sb = 0;
    for (int s = 0; s < Ls::S; ++s)
      if (Ls::K(s, d) > Ls::K(sb, d)) sb = s;
    const int Q = Ls::Q(d), H = Ls::H(d);
    for (int k = 0; k < Ls::KMAX(d); ++k)
      for (int h = 0; h < H; ++h)
        out.tab[static_cast<size_t>(Ls::ttoff(d) + k * H + h)] =
            a.phi[sb][d][static_cast<size_t>(k) * Q + h];
  }
  auto band_pack = [&](int d, std::vector<double>& v, size_t base) {
    for (int s = 0; s < Ls::S; ++s) {
      const int K = Ls::K(s, d), kd = Ls::kind(s, d), N = Ls::N(d);
      const std::vector<double>& C = *a.dense[s][d];
      for (int x = 0; x < N; ++x)
        for (int y = 0; y < N; ++y) {
          const int lo = band_lo(kd, x, y), cnt = band_count(kd, x, y);
          for (int j = 0; j < cnt; ++j)
            v[base + static_cast<size_t>(Ls::coff(d, s, x, y) + j)] =
                C[(static_cast<size_t>(x) * N + y) * K + lo + band_step(kd, x, y) * j];
        }
    }
  };
  out.cu.assign(static_cast<size_t>(Ls::ctot(0)), 0.0);
  band_pack(0, out.cu, 0);
  if (cudaMalloc(&out.d_cu, sizeof(double) * out.cu.size()) != cudaSuccess) return false;
  if (cudaMemcpy(out.d_cu, out.cu.data(), sizeof(double) * out.cu.size(), cudaMemcpyHostToDevice) !=
      cudaSuccess)
    return false;
  out.cvw.assign(static_cast<size_t>(Ls::ctot(1) + Ls::ctot(2)), 0.0);
  band_pack(1, out.cvw, 0);
  band_pack(2, out.cvw, static_cast<size_t>(Ls::ctot(1)));
  if (cudaMalloc(&out.d_cvw, sizeof(double) * out.cvw.size()) != cudaSuccess) return false;
  if (cudaMemcpy(out.d_cvw, out.cvw.data(), sizeof(double) * out.cvw.size(), cudaMemcpyHostToDevice) !=
      cudaSuccess)
    return false;
  return true;
}

template <class Ls>
cudaError_t launch_large_moments(const double* alpha, double* I, int64_t n_units, const LargePack& pk,
                                 cudaStream_t st) {
  LMomParams<Ls> p;
  p.alpha = alpha;
  p.I = I;
  p.n_units = n_units;
  std::memcpy(p.tab, pk.tab.data(), sizeof(double) * Ls::TALL);
  if (n_units == 0) return cudaSuccess;
  cudaError_t e = kernel_prepare(large_moments_kernel<Ls>, Ls::MOM_SMEM, P2S_LARGE_MOM_THREADS);
  if (e != cudaSuccess) return e;
  const unsigned grid = static_cast<unsigned>(n_units * Ls::S * Ls::NCH);
  if (pk.mom_split && pk.d_T1) {
    // split moments: u pass (all k1 per alpha row) into the L2-resident T1
    // scratch, then v/w passes per k1 chunk, over sub-batches of (unit, term)s
    if ((e = kernel_prepare(large_mom_vw_kernel<Ls>, Ls::MOM_SMEM, P2S_LARGE_MOM_THREADS)) != cudaSuccess) return e;
    constexpr int RB = (Ls::Q(1) * Ls::Q(2) + LMomSplit<Ls>::ROWS - 1) / LMomSplit<Ls>::ROWS;
    const int64_t total = n_units * Ls::S;
    for (int64_t u0 = 0; u0 < total; u0 += pk.t1_units) {
      const int64_t cnt = std::min(pk.t1_units, total - u0);
      large_mom_u_kernel<Ls><<<static_cast<unsigned>(cnt * RB), LMomSplit<Ls>::ROWS, 0, st>>>(p, pk.d_T1, u0);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      large_mom_vw_kernel<Ls><<<static_cast<unsigned>(cnt * Ls::NCH), P2S_LARGE_MOM_THREADS, Ls::MOM_SMEM, st>>>(
          p, pk.d_T1, u0);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
#ifndef P2S_LEAN
  if constexpr (Ls::Q(0) % 2 == 0 && Ls::NCH <= 8)
  if (pk.mom_cluster) {
    if ((e = kernel_prepare(large_moments_kernel<Ls, true>, Ls::MOM_SMEM, P2S_LARGE_MOM_THREADS)) != cudaSuccess)
      return e;
    // one cluster of NCH chunk CTAs per (unit, term)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(P2S_LARGE_MOM_THREADS);
    cfg.dynamicSmemBytes = Ls::MOM_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(Ls::NCH);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, large_moments_kernel<Ls, true>, p);
  }
#endif
  if constexpr (LMomW<Ls>::FITS)
    if (pk.mom_wfirst) {
      if ((e = kernel_prepare(large_moments_w_kernel<Ls>, LMomW<Ls>::SMEM, LMomW<Ls>::NT)) != cudaSuccess) return e;
      large_moments_w_kernel<Ls><<<static_cast<unsigned>(n_units * Ls::S * LMomW<Ls>::NCH), LMomW<Ls>::NT,
                                   LMomW<Ls>::SMEM, st>>>(p);
      return cudaGetLastError();
    }
#ifndef P2S_LEAN  // measurement variants (u-first tiles, grouped v / w items): ahead-of-time builds only
  if constexpr (LMomT<Ls>::FITS)
    if (pk.mom_tiled) {
      if ((e = kernel_prepare(large_moments_t_kernel<Ls>, LMomT<Ls>::SMEM, LMomT<Ls>::NT)) != cudaSuccess) return e;
      large_moments_t_kernel<Ls><<<grid, LMomT<Ls>::NT, LMomT<Ls>::SMEM, st>>>(p);
      return cudaGetLastError();
    }
  if constexpr (LMomG<Ls>::FITS)
    if (pk.mom_grouped) {
      if ((e = kernel_prepare(large_moments_g_kernel<Ls>, LMomG<Ls>::SMEM, LMomG<Ls>::NT)) != cudaSuccess) return e;
      large_moments_g_kernel<Ls><<<grid, LMomG<Ls>::NT, LMomG<Ls>::SMEM, st>>>(p);
      return cudaGetLastError();
    }
#endif
  large_moments_kernel<Ls><<<grid, P2S_LARGE_MOM_THREADS, Ls::MOM_SMEM, st>>>(p);
  return cudaGetLastError();
}

// contraction of n_units units from I (device) via the X scratch (chunks of xchunk units)
template <class Ls>
cudaError_t launch_large_contract(const double* I, double* X, double* M, int64_t n_units,
                                  int64_t xchunk, int64_t ldM, int nc, int P, int Nt,
                                  const LargePack& pk, cudaStream_t st) {
  cudaError_t e0 = cudaSuccess;
  LUParams<Ls> up;
  up.M = M;
  up.ldM = ldM;
  up.mat_stride = static_cast<int64_t>(nc) * Nt * ldM;
  up.nc = nc;
  up.P = P;
  up.Nt = Nt;
  std::memcpy(up.cu, pk.cu.data(), sizeof(double) * Ls::cpar(0));
  up.cu_g = pk.d_cu;
  up.xs = pk.u_xs ? 1 : 0;
  up.roll = pk.u_roll == 0 ? 0 : 1;  // unrolled rows measured slower (c12 0.535 vs 0.583)
  up.pair = pk.u_pair && (reinterpret_cast<uintptr_t>(M) % 16 == 0) && (ldM % 2 == 0) ? 1 : 0;
  // bulk stores need 16-B aligned rows: M base, ld_M and N_v N_w even
  up.bulk = pk.u_bulk && (reinterpret_cast<uintptr_t>(M) % 16 == 0) && (ldM % 2 == 0) &&
                    ((Ls::NV * Ls::NW) % 2 == 0)
                ? 1
                : 0;
  LWParams<Ls> wp;
  wp.Z = pk.d_Z;
  wp.cg = pk.d_cvw + Ls::ctot(1);
  std::memcpy(wp.cw, pk.cvw.data() + Ls::ctot(1), sizeof(double) * Ls::cpar(2));
  LVParams<Ls> vp;
  vp.Z = pk.d_Z;
  vp.cg = pk.d_cvw;
  std::memcpy(vp.cv, pk.cvw.data(), sizeof(double) * Ls::cpar(1));
  // over-size v / w tables are staged in shared memory per CTA (Ls::GS)
  if (Ls::cs_bytes(2) > 0 &&
      (e0 = kernel_prepare(large_w_kernel<Ls>, Ls::cs_bytes(2), 32 * kLargeWWarps)) != cudaSuccess)
    return e0;
  if (Ls::cs_bytes(1) > 0 &&
      (e0 = kernel_prepare(large_v_kernel<Ls>, Ls::cs_bytes(1), LVRows<Ls>::VR * Ls::NW * Ls::NW)) != cudaSuccess)
    return e0;
  // X holds two chunk buffers; chunk i uses buffer i % 2
  const bool ov = pk.overlap && pk.aux != nullptr;
  const bool two = ov && pk.two_u && pk.aux_u != nullptr && n_units > xchunk;
  cudaError_t e;
  if (ov) {
    if ((e = cudaEventRecord(pk.ev_start, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(pk.aux, pk.ev_start, 0)) != cudaSuccess) return e;  // I ready
    if (two && (e = cudaStreamWaitEvent(pk.aux_u, pk.ev_start, 0)) != cudaSuccess) return e;
  }
  int64_t i = 0;
  for (int64_t u0 = 0; u0 < n_units; u0 += xchunk, ++i) {
    const int64_t cnt = std::min(xchunk, n_units - u0);
    const int b = static_cast<int>(i % 2);
    double* Xb = X + (ov ? b : 0) * xchunk * Ls::XPU;
    wp.I = I + u0 * Ls::MPP;
    wp.n_units = vp.n_units = cnt;
    vp.X = Xb;
    cudaStream_t vs = ov ? pk.aux : st;
    if (ov && i >= 2 && (e = cudaStreamWaitEvent(pk.aux, pk.ev_u[b], 0)) != cudaSuccess) return e;
    // w step then v step (Z single-buffered: both on the same stream)
    const int64_t wblocks = (cnt * Ls::KGTOT() + kLargeWWarps - 1) / kLargeWWarps * Ls::NGRP;
    large_w_kernel<Ls><<<static_cast<unsigned>(wblocks), 32 * kLargeWWarps, Ls::cs_bytes(2), vs>>>(wp);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    {
      constexpr int VR = LVRows<Ls>::VR;
      const int64_t items = (cnt * Ls::KUTOT() + VR - 1) / VR;
      // few items per chunk (C5: 300 CTAs, one latency-bound wave): deal the n1 rows of
      // an item to several CTAs
      int64_t ns = 1;
      if (pk.v_split > 0)
        ns = std::max<int64_t>(1, std::min<int64_t>(Ls::NV, (int64_t(pk.v_split) * 2 * pk.num_sms + items - 1) / items));
      vp.ns = static_cast<int>(ns);
      large_v_kernel<Ls><<<static_cast<unsigned>(items * ns), VR * Ls::NW * Ls::NW, Ls::cs_bytes(1), vs>>>(vp);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    cudaStream_t us = (two && b == 1) ? pk.aux_u : st;
    if (ov) {
      if ((e = cudaEventRecord(pk.ev_vw[b], pk.aux)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(us, pk.ev_vw[b], 0)) != cudaSuccess) return e;
    }
    // u stage: absolute units u0 .. u0+cnt-1; Xb holds the chunk
    up.X = Xb;
    up.n_units = cnt;
    if ((e = large_u_dispatch<Ls>(up, u0, cnt, pk.ps, pk.ufib, pk.u_ctas, pk.u_smemc, pk.num_sms, us)) != cudaSuccess)
      return e;
    if (ov && (e = cudaEventRecord(pk.ev_u[b], us)) != cudaSuccess) return e;
  }
  if (two) {  // join: the caller's stream sees every u stage
    if ((e = cudaEventRecord(pk.ev_join, pk.aux_u)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, pk.ev_join, 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}


template <class Ls>
LargeEntry make_large() {
  LargeEntry r{};
  for (int d = 0; d < 3; ++d) {
    r.order[d] = Ls::N(d);
    r.nq[d] = Ls::Q(d);
  }
  r.S = Ls::S;
  for (int s = 0; s < Ls::S; ++s)
    for (int d = 0; d < 3; ++d) r.kinds[s][d] = Ls::kind(s, d);
  r.pack = &pack_large<Ls>;
  r.moments = &launch_large_moments<Ls>;
  r.contract = &launch_large_contract<Ls>;
  r.mpp = Ls::MPP;
  r.t1u = LMomSplit<Ls>::T1U;
  r.xpu = Ls::XPU;
  r.zpu = Ls::ZPU;
  return r;
}

}  // namespace reg
}  // namespace p2s
