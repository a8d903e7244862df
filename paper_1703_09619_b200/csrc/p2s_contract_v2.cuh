// p2s_contract_v2.cuh -- shape-specialised contraction kernel (all orders,
// kinds and tile sizes compile-time).  Used for the registered benchmark
// shapes; the runtime-shaped contract_kernel (p2s_kernels.cuh) covers the
// rest.
//
// Persistent CTAs walk (element, pair) units.  Per unit:
//   I  -> smem            one bulk copy (TMA engine, cp.async.bulk) on an
//                         mbarrier; the next unit's copy is issued as soon as
//                         the last stage A of this unit has read I
// and per tile of T n1-values:
//   stage A (v):  thread = fiber (k1, k3) of I_s, Kv values in registers;
//                 A_s[i][k1][n2][k3] = sum_k2 Cv[n1][n2][k2] I_s[k1][k2][k3]
//   stage B (w):  thread = fiber (i, k1, n2) of A_s, Kw values in registers;
//                 B_s[i][k1][p1][n2][p2] = sum_k3 Cw[p1][p2][k3] A_s[i][k1][n2][k3]
//   stage C (u):  thread = fiber (i, p1, n2, p2) of B_s over all terms;
//                 M[m1 n1 p1][m2 n2 p2] = sum_s sum_k1 Cu[m1][m2][k1] B_s[..k1..]
// Every output loop is unrolled with compile-time bands, every coefficient is
// a constant-bank operand, every fiber is register resident: one DFMA per
// product-to-sum term and one store per element-matrix entry.
#pragma once

#include "p2s_kernels.cuh"

namespace p2s {

constexpr int enc_kind(int ku, int kv, int kw) { return ku | (kv << 2) | (kw << 4); }

template <int NU_, int NV_, int NW_, int T_, int THREADS_, int MINB_, int... TK>
struct Shape {
  static constexpr int NU = NU_, NV = NV_, NW = NW_, T = T_, THREADS = THREADS_, MINB = MINB_;
  static constexpr int S = sizeof...(TK);
  static constexpr int NT = NV / T;
  static_assert(NV % T == 0, "n1 tile must divide N_v");
  static constexpr int N(int d) { return d == 0 ? NU : d == 1 ? NV : NW; }
  static constexpr int kind(int s, int d) {
    const int k[] = {TK...};
    return (k[s] >> (2 * d)) & 3;
  }
  static constexpr int K(int s, int d) { return kernel_count(kind(s, d), N(d)); }
  static constexpr int KTOT_U() {
    int o = 0;
    for (int s = 0; s < S; ++s) o += K(s, 0);
    return o;
  }
  static constexpr int kuoff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0);
    return o;
  }
  // packed band coefficients of direction d: terms in order, (a, b) row-major
  static constexpr int coff(int d, int s, int a, int b) {
    int o = 0;
    for (int t = 0; t < s; ++t)
      for (int x = 0; x < N(d); ++x)
        for (int y = 0; y < N(d); ++y) o += band_count(kind(t, d), x, y);
    for (int x = 0; x < N(d); ++x)
      for (int y = 0; y < N(d); ++y) {
        if (x == a && y == b) return o;
        o += band_count(kind(s, d), x, y);
      }
    return o;
  }
  static constexpr int ctot(int d) { return coff(d, S, 0, 0) > 0 ? coff(d, S, 0, 0) : 1; }
  // moment block of one pair (doubles), terms back to back, padded to 4
  static constexpr int moff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0) * K(i, 1) * K(i, 2);
    return o;
  }
  static constexpr int MPP = (moff(S) + 3) & ~3;
  // smem (doubles)
  static constexpr int BSTR = (NW * NV * NW) | 1;  // odd k1 stride of B
  static constexpr int aoff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += T * K(i, 0) * NV * K(i, 2);
    return o;
  }
  static constexpr int boff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += T * K(i, 0) * BSTR;
    return o;
  }
  static constexpr int A_DBL = (aoff(S) + 1) & ~1;
  static constexpr int B_DBL = (boff(S) + 1) & ~1;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(MPP + A_DBL + B_DBL) + 16;
};

template <class Sh>
struct V2Params {
  const double* I;
  double* M;
  int64_t ldM, mat_stride;
  int64_t n_units;
  int nc, P, Nt;
  int64_t mom_per_elem;
  double cu[Sh::ctot(0)];
  double cv[Sh::ctot(1)];
  double cw[Sh::ctot(2)];
};

template <class Sh, int N1>
__device__ __forceinline__ void v2_stage_a_n1(const V2Params<Sh>& p, const double* Ibuf,
                                              double* Abuf, int i) {
  // one n1 value (compile-time) of the tile, slot i
  constexpr int NV = Sh::NV;
  static_for<0, Sh::S>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    constexpr int Ku = Sh::K(s, 0), Kv = Sh::K(s, 1), Kw = Sh::K(s, 2);
    constexpr int kv = Sh::kind(s, 1);
    const double* Is = Ibuf + Sh::moff(s);
    double* As = Abuf + Sh::aoff(s) + i * (Ku * NV * Kw);
    for (int f = threadIdx.x; f < Ku * Kw; f += Sh::THREADS) {
      const int k1 = f / Kw, k3 = f - (f / Kw) * Kw;
      double x[Kv];
#pragma unroll
      for (int k2 = 0; k2 < Kv; ++k2) x[k2] = Is[(k1 * Kv + k2) * Kw + k3];
      static_for<0, NV>([&](auto n2c) {
        constexpr int n2 = decltype(n2c)::value;
        constexpr int lo = band_lo(kv, N1, n2), cnt = band_count(kv, N1, n2);
        constexpr int co = Sh::coff(1, s, N1, n2);
        double v = 0.0;
        static_for<0, cnt>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          v = fma(p.cv[co + j], x[lo + 2 * j], v);
        });
        As[(k1 * NV + n2) * Kw + k3] = v;
      });
    }
  });
}

template <class Sh>
__global__ void __launch_bounds__(Sh::THREADS, Sh::MINB)
    contract_v2_kernel(const __grid_constant__ V2Params<Sh> p) {
  extern __shared__ __align__(16) double sm[];
  constexpr int S = Sh::S, NU = Sh::NU, NV = Sh::NV, NW = Sh::NW, T = Sh::T;
  double* Ibuf = sm;
  double* Abuf = Ibuf + Sh::MPP;
  double* Bbuf = Abuf + Sh::A_DBL;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bbuf + Sh::B_DBL);
  const int tid = threadIdx.x;
  constexpr uint32_t kIBytes = Sh::MPP * 8u;

  int64_t unit = blockIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    if (unit < p.n_units) {
      const int64_t e = unit / p.P;
      const int pair = static_cast<int>(unit - e * p.P);
      mbar_arrive_expect_tx(bar, kIBytes);
      bulk_g2s(Ibuf, p.I + e * p.mom_per_elem + pair * Sh::MPP, kIBytes, bar);
    }
  }
  __syncthreads();
  uint32_t phase = 0;
  for (; unit < p.n_units; unit += gridDim.x) {
    const int64_t e = unit / p.P;
    const int pair = static_cast<int>(unit - e * p.P);
    const int gci = pair / p.nc, gcj = pair - gci * p.nc;
    mbar_wait_parity(bar, phase);
    phase ^= 1u;
    double* Mbase = p.M + e * p.mat_stride + static_cast<int64_t>(gci * p.Nt) * p.ldM + gcj * p.Nt;

    for (int t = 0; t < Sh::NT; ++t) {
      // ---- stage A
      static_for<0, Sh::NT>([&](auto tc) {
        constexpr int tt = decltype(tc)::value;
        if (t == tt) {
          static_for<0, T>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            v2_stage_a_n1<Sh, tt * T + i>(p, Ibuf, Abuf, i);
          });
        }
      });
      __syncthreads();
      if (t == Sh::NT - 1 && tid == 0) {
        const int64_t nxt = unit + gridDim.x;
        if (nxt < p.n_units) {
          const int64_t e2 = nxt / p.P;
          const int pair2 = static_cast<int>(nxt - e2 * p.P);
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(bar, kIBytes);
          bulk_g2s(Ibuf, p.I + e2 * p.mom_per_elem + pair2 * Sh::MPP, kIBytes, bar);
        }
      }
      // ---- stage B
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        constexpr int Ku = Sh::K(s, 0), Kw = Sh::K(s, 2);
        constexpr int kw = Sh::kind(s, 2);
        const double* As = Abuf + Sh::aoff(s);
        double* Bs = Bbuf + Sh::boff(s);
        for (int f = tid; f < T * Ku * NV; f += Sh::THREADS) {
          // f = (i*Ku + k1)*NV + n2
          const int n2 = f % NV;
          const int ik = f / NV;
          double y[Kw];
#pragma unroll
          for (int k3 = 0; k3 < Kw; ++k3) y[k3] = As[f * Kw + k3];
          double* dst = Bs + ik * Sh::BSTR + n2 * NW;
          static_for<0, NW>([&](auto p1c) {
            constexpr int p1 = decltype(p1c)::value;
            static_for<0, NW>([&](auto p2c) {
              constexpr int p2 = decltype(p2c)::value;
              constexpr int lo = band_lo(kw, p1, p2), cnt = band_count(kw, p1, p2);
              constexpr int co = Sh::coff(2, s, p1, p2);
              double v = 0.0;
              static_for<0, cnt>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                v = fma(p.cw[co + j], y[lo + 2 * j], v);
              });
              dst[p1 * NV * NW + p2] = v;
            });
          });
        }
      });
      __syncthreads();
      // ---- stage C
      constexpr int NF = T * NW * NV * NW;
      for (int f = tid; f < NF; f += Sh::THREADS) {
        // f = ((i*NW + p1)*NV + n2)*NW + p2
        const int r = f % (NV * NW);  // n2*NW + p2
        const int ip = f / (NV * NW);
        const int p1 = ip % NW, i = ip / NW;
        const int n1 = t * T + i;
        double b[Sh::KTOT_U()];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          constexpr int Ku = Sh::K(s, 0);
          const double* src = Bbuf + Sh::boff(s) + (i * Ku) * Sh::BSTR + p1 * NV * NW + r;
#pragma unroll
          for (int k1 = 0; k1 < Ku; ++k1) b[Sh::kuoff(s) + k1] = src[k1 * Sh::BSTR];
        });
        double* out = Mbase + static_cast<int64_t>(n1 * NW + p1) * p.ldM + r;
        const int64_t rowstep = static_cast<int64_t>(NV * NW) * p.ldM;
        static_for<0, NU>([&](auto m1c) {
          constexpr int m1 = decltype(m1c)::value;
          static_for<0, NU>([&](auto m2c) {
            constexpr int m2 = decltype(m2c)::value;
            double v = 0.0;
            static_for<0, S>([&](auto sc) {
              constexpr int s = decltype(sc)::value;
              constexpr int ku = Sh::kind(s, 0);
              constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
              constexpr int co = Sh::coff(0, s, m1, m2);
              constexpr int ko = Sh::kuoff(s);
              static_for<0, cnt>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                v = fma(p.cu[co + j], b[ko + lo + 2 * j], v);
              });
            });
            st_cs(out + m1 * rowstep + m2 * (NV * NW), v);
          });
        });
      }
      __syncthreads();
    }
  }
}

}  // namespace p2s
