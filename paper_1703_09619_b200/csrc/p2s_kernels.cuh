// p2s_kernels.cuh -- the two sm_100a kernels of the fill.
//
//   moments_kernel   I_s[k1][k2][k3] = sum_q alpha_s(q) phi_k1(u) phi_k2(v) phi_k3(w)
//                    (phi = w_q P_k(x_q)); three 1-D passes in shared memory.
//                    Replaces compute_kernel_tables (assembly.cpp:276-314).
//   contract_kernel  M[m1 n1 p1][m2 n2 p2] = sum_s sum_k Cu Cv Cw I_s; staged
//                    v -> w -> u with the last (u) stage unrolled at compile
//                    time on a register-resident fiber; every entry of M is
//                    written exactly once.  Replaces assemble_p2s_element
//                    (assembly.cpp:375-474).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "p2s_device.cuh"
#include "p2s_tables.hpp"

namespace p2s {

constexpr int kMaxTerms = 4;

// ============================================================ moment stage

struct MomentParams {
  const double* alpha;
  double* I;
  int64_t n_units;                 // E * P * S CTAs
  int P, S;
  int nq[3];
  int K[kMaxTerms][3];
  int Kpad[kMaxTerms][3];          // even row length of the transposed tables
  const double* phiT[kMaxTerms][3];  // [nq][Kpad], k contiguous
  int64_t mom_per_elem, mom_per_pair;
  int64_t mom_off[kMaxTerms];
  int S2, S3;                      // odd smem row strides (bank-conflict free)
};

// One CTA per (element, pair, term).  Stage 1 contracts u (thread = row
// (q_w, q_v), alpha row read with 16-B loads), stage 2 contracts v (thread =
// (k1, q_w)), stage 3 contracts w (thread = (k1, k2)); every inner loop reads
// its table entry as a warp-uniform broadcast.
template <int KMAX>
__global__ void __launch_bounds__(256) moments_kernel(const __grid_constant__ MomentParams p) {
  extern __shared__ __align__(16) double sm[];
  const int64_t unit = blockIdx.x;
  const int ps = static_cast<int>(unit % (p.P * p.S));
  const int64_t e = unit / (p.P * p.S);
  const int pair = ps / p.S, s = ps % p.S;
  const int nqu = p.nq[0], nqv = p.nq[1], nqw = p.nq[2];
  const int Ku = p.K[s][0], Kv = p.K[s][1], Kw = p.K[s][2];
  const int KpU = p.Kpad[s][0], KpV = p.Kpad[s][1], KpW = p.Kpad[s][2];
  const int S2 = p.S2, S3 = p.S3;

  double* Lu = sm;
  double* Lv = Lu + nqu * KpU;
  double* Lw = Lv + nqv * KpV;
  double* T1 = Lw + nqw * KpW;                 // [Ku][nqw][S2]
  double* T2 = T1 + Ku * nqw * S2;             // [Ku*Kv][S3]
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < nqu * KpU; i += nt) Lu[i] = p.phiT[s][0][i];
  for (int i = tid; i < nqv * KpV; i += nt) Lv[i] = p.phiT[s][1][i];
  for (int i = tid; i < nqw * KpW; i += nt) Lw[i] = p.phiT[s][2][i];
  __syncthreads();

  const double* a = p.alpha + unit * static_cast<int64_t>(nqu * nqv * nqw);

  // ---- stage 1: u
  for (int r = tid; r < nqw * nqv; r += nt) {
    const int q3 = r / nqv, q2 = r - q3 * nqv;
    const double* row = a + static_cast<int64_t>(r) * nqu;
    double acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = 0.0;
    auto step = [&](double x, int q1) {
      const double* L = Lu + q1 * KpU;
#pragma unroll
      for (int k = 0; k < KMAX; k += 2) {
        if (k < Ku) {
          const double2 l = *reinterpret_cast<const double2*>(L + k);
          acc[k] = fma(x, l.x, acc[k]);
          acc[k + 1] = fma(x, l.y, acc[k + 1]);
        }
      }
    };
    if ((nqu & 1) == 0) {
      const double2* row2 = reinterpret_cast<const double2*>(row);
      for (int q = 0; q < nqu / 2; ++q) {
        const double2 x = __ldg(row2 + q);
        step(x.x, 2 * q);
        step(x.y, 2 * q + 1);
      }
    } else {
      for (int q1 = 0; q1 < nqu; ++q1) step(__ldg(row + q1), q1);
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < Ku) T1[(k * nqw + q3) * S2 + q2] = acc[k];
  }
  __syncthreads();

  // ---- stage 2: v
  for (int r = tid; r < Ku * nqw; r += nt) {
    const int k1 = r / nqw, q3 = r - k1 * nqw;
    const double* src = T1 + (k1 * nqw + q3) * S2;
    double acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = 0.0;
    for (int q2 = 0; q2 < nqv; ++q2) {
      const double x = src[q2];
      const double* L = Lv + q2 * KpV;
#pragma unroll
      for (int k = 0; k < KMAX; k += 2) {
        if (k < Kv) {
          const double2 l = *reinterpret_cast<const double2*>(L + k);
          acc[k] = fma(x, l.x, acc[k]);
          acc[k + 1] = fma(x, l.y, acc[k + 1]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < Kv) T2[(k1 * Kv + k) * S3 + q3] = acc[k];
  }
  __syncthreads();

  // ---- stage 3: w
  double* out = p.I + e * p.mom_per_elem + pair * p.mom_per_pair + p.mom_off[s];
  for (int r = tid; r < Ku * Kv; r += nt) {
    const double* src = T2 + r * S3;
    double acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = 0.0;
    for (int q3 = 0; q3 < nqw; ++q3) {
      const double x = src[q3];
      const double* L = Lw + q3 * KpW;
#pragma unroll
      for (int k = 0; k < KMAX; k += 2) {
        if (k < Kw) {
          const double2 l = *reinterpret_cast<const double2*>(L + k);
          acc[k] = fma(x, l.x, acc[k]);
          acc[k + 1] = fma(x, l.y, acc[k + 1]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < Kw) out[r * Kw + k] = acc[k];
  }
}

// ============================================================ contraction

// Compile-time description of the u direction: order NU and the u-kind of
// every term.  Bands of the u expansion are compile-time, so the final stage
// indexes its register fiber with constants.
template <int NU_, int... KINDS>
struct UCfg {
  static constexpr int NU = NU_;
  static constexpr int S = sizeof...(KINDS);
  static constexpr int kind(int s) {
    const int k[] = {KINDS...};
    return k[s];
  }
  static constexpr int K(int s) { return kernel_count(kind(s), NU); }
  static constexpr int koff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i);
    return o;
  }
  static constexpr int KTOT = koff(S);
  // offset of the packed band coefficients of (s, a, b)
  static constexpr int coff(int s, int a, int b) {
    int o = 0;
    for (int t = 0; t < s; ++t)
      for (int x = 0; x < NU; ++x)
        for (int y = 0; y < NU; ++y) o += band_count(kind(t), x, y);
    for (int x = 0; x < NU; ++x)
      for (int y = 0; y < NU; ++y) {
        if (x == a && y == b) return o;
        o += band_count(kind(s), x, y);
      }
    return o;
  }
  static constexpr int CTOT = coff(S, 0, 0) > 0 ? coff(S, 0, 0) : 1;
};

template <class Cfg>
struct ContractParams {
  const double* I;
  double* M;
  int64_t ldM, mat_stride;         // mat_stride = n_tot * ldM
  int64_t n_cta;
  int nc, P, Nv, Nw, Nt, G, NG;
  int Kv[Cfg::S], Kw[Cfg::S], kind_v[Cfg::S], kind_w[Cfg::S];
  int64_t mom_per_elem, mom_per_pair;
  int mom_off[Cfg::S];
  int i_doubles;                    // one pair's moment block (multiple of 2)
  int a_off[Cfg::S];                // per-term offsets inside the A buffer
  int cv_off[Cfg::S], cw_off[Cfg::S];
  int a_doubles, c_doubles;
  const double* Cv[Cfg::S];         // dense [Nv][Nv][Kv]
  const double* Cw[Cfg::S];         // dense [Nw][Nw][Kw]
  double cu[Cfg::CTOT];             // packed u bands (constant bank)
};

__device__ __forceinline__ int dband_lo(int kind, int a, int b) { return band_lo(kind, a, b); }
__device__ __forceinline__ int dband_hi(int kind, int a, int b) { return band_hi(kind, a, b); }
__device__ __forceinline__ int dband_step(int kind, int a, int b) { return band_step(kind, a, b); }

// One CTA per (element, pair, group of G n1-values).
//   load:     the pair's moments I (all terms) -> smem with one bulk copy
//             (TMA engine) on an mbarrier; v/w coefficient tables -> smem
//   stage A:  A_s[n1][k1][n2][k3] = sum_k2 Cv[n1][n2][k2] I_s[k1][k2][k3]
//   stage B:  per fiber (n1, p1, n2, p2), in registers:
//             b_s[k1] = sum_k3 Cw[p1][p2][k3] A_s[n1][k1][n2][k3]
//   stage C:  M[m1 n1 p1][m2 n2 p2] = sum_s sum_k1 Cu_s[m1][m2][k1] b_s[k1]
//             fully unrolled, Cu from the constant bank, one store per entry.
template <class Cfg>
__global__ void __launch_bounds__(256) contract_kernel(const __grid_constant__ ContractParams<Cfg> p) {
  extern __shared__ __align__(16) double sm[];
  constexpr int S = Cfg::S;
  constexpr int NU = Cfg::NU;
  const int64_t cta = blockIdx.x;
  const int g = static_cast<int>(cta % p.NG);
  const int64_t ep = cta / p.NG;
  const int pair = static_cast<int>(ep % p.P);
  const int64_t e = ep / p.P;
  const int gci = pair / p.nc, gcj = pair - gci * p.nc;
  const int Nv = p.Nv, Nw = p.Nw, G = p.G;
  const int tid = threadIdx.x, nt = blockDim.x;

  double* Ibuf = sm;
  double* Abuf = Ibuf + p.i_doubles;
  double* Ctab = Abuf + p.a_doubles;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Ctab + p.c_doubles);

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t bytes = static_cast<uint32_t>(p.i_doubles) * 8u;
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(Ibuf, p.I + e * p.mom_per_elem + pair * p.mom_per_pair, bytes, bar);
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int nv = Nv * Nv * p.Kv[s], nw = Nw * Nw * p.Kw[s];
    for (int i = tid; i < nv; i += nt) Ctab[p.cv_off[s] + i] = __ldg(p.Cv[s] + i);
    for (int i = tid; i < nw; i += nt) Ctab[p.cw_off[s] + i] = __ldg(p.Cw[s] + i);
  }
  __syncthreads();
  mbar_wait_parity(bar, 0);

  // ---- stage A: v contraction for the CTA's n1 group
  static_for<0, S>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    constexpr int Ku = Cfg::K(s);
    const int Kv = p.Kv[s], Kw = p.Kw[s], kv = p.kind_v[s];
    const double* Is = Ibuf + p.mom_off[s];
    const double* Cv = Ctab + p.cv_off[s];
    double* As = Abuf + p.a_off[s];
    const int total = G * Ku * Nv * Kw;
    for (int idx = tid; idx < total; idx += nt) {
      const int k3 = idx % Kw;
      int t = idx / Kw;
      const int n2 = t % Nv;
      t /= Nv;
      const int k1 = t % Ku;
      const int gi = t / Ku;
      const int n1 = g * G + gi;
      double acc = 0.0;
      if (n1 < Nv) {
        const int lo = dband_lo(kv, n1, n2), hi = dband_hi(kv, n1, n2), st = dband_step(kv, n1, n2);
        const double* c = Cv + (n1 * Nv + n2) * Kv;
        const double* src = Is + k1 * Kv * Kw + k3;
        for (int k2 = lo; k2 <= hi; k2 += st) acc = fma(c[k2], src[k2 * Kw], acc);
      }
      As[idx] = acc;
    }
  });
  __syncthreads();

  // ---- stages B + C per fiber
  const int nfib = G * Nw * Nv * Nw;
  const int64_t rowstep = static_cast<int64_t>(Nv) * Nw * p.ldM;
  const int colstep = Nv * Nw;
  for (int f = tid; f < nfib; f += nt) {
    const int p2 = f % Nw;
    int t = f / Nw;
    const int n2 = t % Nv;
    t /= Nv;
    const int p1 = t % Nw;
    const int gi = t / Nw;
    const int n1 = g * G + gi;
    if (n1 >= Nv) continue;

    double b[Cfg::KTOT];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      constexpr int Ku = Cfg::K(s);
      constexpr int ko = Cfg::koff(s);
      const int Kw = p.Kw[s];
      const int astride = Nv * Kw;
      const double* As = Abuf + p.a_off[s] + (gi * Ku * Nv + n2) * Kw;
      const double* cw = Ctab + p.cw_off[s] + (p1 * Nw + p2) * Kw;
      const int lo = dband_lo(p.kind_w[s], p1, p2), hi = dband_hi(p.kind_w[s], p1, p2),
                st = dband_step(p.kind_w[s], p1, p2);
#pragma unroll
      for (int k1 = 0; k1 < Ku; ++k1) b[ko + k1] = 0.0;
      for (int k3 = lo; k3 <= hi; k3 += st) {
        const double c = cw[k3];
#pragma unroll
        for (int k1 = 0; k1 < Ku; ++k1) b[ko + k1] = fma(c, As[k1 * astride + k3], b[ko + k1]);
      }
    });

    double* out = p.M + e * p.mat_stride +
                  static_cast<int64_t>(gci * p.Nt + n1 * Nw + p1) * p.ldM + gcj * p.Nt + n2 * Nw + p2;
    static_for<0, NU>([&](auto m1c) {
      constexpr int m1 = decltype(m1c)::value;
      static_for<0, NU>([&](auto m2c) {
        constexpr int m2 = decltype(m2c)::value;
        double v = 0.0;
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          constexpr int kd = Cfg::kind(s);
          constexpr int lo = band_lo(kd, m1, m2);
          constexpr int cnt = band_count(kd, m1, m2);
          constexpr int co = Cfg::coff(s, m1, m2);
          constexpr int ko = Cfg::koff(s);
          static_for<0, cnt>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            v = fma(p.cu[co + j], b[ko + lo + band_step(kd, m1, m2) * j], v);
          });
        });
        st_cs(out + m1 * rowstep + m2 * colstep, v);
      });
    });
  }
}

}  // namespace p2s
