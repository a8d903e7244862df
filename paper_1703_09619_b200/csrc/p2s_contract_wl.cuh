// p2s_contract_wl.cuh -- "w-last" contraction for anisotropic orders (C4:
// N = (10, 6, 4)).  The v2 contraction (p2s_contract_v2.cuh) contracts u last;
// the last stage dominates (N_last^2 outputs per fiber times the band), so for
// N_u >> N_w contracting w last is ~3x fewer FMAs:
//   stage A (u):  A_s[t(m1,m2)][k2][k3] = sum_k1 Cu[m1][m2][k1] I_s[k1][k2][k3]
//   stage B (v):  B_s[t(m1,m2)][t(n1,n2)][k3] = sum_k2 Cv[n1][n2][k2] A_s[..][k2][k3]
//   stage C (w):  M[m1 n1 p1][m2 n2 p2] = sum_s sum_k3 Cw[p1][p2][k3] B_s[..][..][k3]
// Symmetric kinds (P.P, P'.P') in u and v: A and B are kept for the upper
// triangles t(m1 <= m2), t(n1 <= n2) only, and a stage-C fiber (t(m1,m2), n1,
// n2) writes its N_w x N_w block for both (m1, m2) and (m2, m1).  The (m1, m2)
// triangle is processed in tiles of TM entries so A and B stay small (two or
// more CTAs per SM); stage A is compiled once per tile (its u-bands are
// compile-time), stages B and C once (their (m1, m2) is runtime addressing).
// Stage-C stores: each thread writes N_w contiguous doubles per output row
// (16-B stores), consecutive threads consecutive (m2, n2) column blocks.
#pragma once

#include "p2s_contract_v2.cuh"

namespace p2s {

template <int NU_, int NV_, int NW_, int TM_, int THREADS_, int MINB_, int... TK>
struct WShape {
  static constexpr int NU = NU_, NV = NV_, NW = NW_, TM = TM_, THREADS = THREADS_, MINB = MINB_;
  static constexpr int S = sizeof...(TK);
  static constexpr int MMA = 0, PAIR = 0, PSPLIT = 0, QUAD = 0, NSYM = 0, SYM = 1, PERSIST = 0;  // registry interface
  static constexpr int N(int d) { return d == 0 ? NU : d == 1 ? NV : NW; }
  static constexpr int kind(int s, int d) {
    const int k[] = {TK...};
    return (k[s] >> (3 * d)) & 7;
  }
  static constexpr int K(int s, int d) { return kernel_count(kind(s, d), N(d)); }
  static constexpr bool sym_ok() {
    for (int s = 0; s < S; ++s)
      for (int d = 0; d < 2; ++d)
        if (base_kind(kind(s, d)) != PP && base_kind(kind(s, d)) != DD) return false;
    return true;
  }
  static_assert(sym_ok(), "w-last contraction needs symmetric u / v kinds");
  static_assert(NW % 2 == 0, "16-B stage-C stores need an even N_w");
  static constexpr int tri(int a, int b, int n) { return a * n - a * (a - 1) / 2 + (b - a); }
  static constexpr int NQU = NU * (NU + 1) / 2, NQV = NV * (NV + 1) / 2;
  static constexpr int NTILE = (NQU + TM - 1) / TM;
  // band-packed coefficients per direction (same layout as Shape: pack_v2 works)
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
  static constexpr int moff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0) * K(i, 1) * K(i, 2);
    return o;
  }
  static constexpr int MPP = (moff(S) + 3) & ~3;
  // shared buffers (doubles): A tile [TM][Kv*Kw | 1], B tile [TM][NQV*Kw | 1] per term
  static constexpr int ast(int s) { return (K(s, 1) * K(s, 2)) | 1; }
  static constexpr int bst(int s) { return (NQV * K(s, 2)) | 1; }
  static constexpr int aoff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += TM * ast(i);
    return o;
  }
  static constexpr int boff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += TM * bst(i);
    return o;
  }
  static constexpr int A_DBL = (aoff(S) + 1) & ~1;
  static constexpr int B_DBL = (boff(S) + 1) & ~1;
  static constexpr int KWTOT() {
    int o = 0;
    for (int s = 0; s < S; ++s) o += K(s, 2);
    return o;
  }
  static constexpr int kwoff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 2);
    return o;
  }
  // (m1, m2) of triangle index t of order NU (compile time)
  static constexpr int trow(int t) {
    int a = 0;
    while (t >= NU - a) t -= NU - a, ++a;
    return a;
  }
  static constexpr int tcol(int t) { return trow(t) + (t - tri(trow(t), trow(t), NU)); }
  static constexpr bool WLAST = true;
  // (m1, m2) of triangle index t (runtime; rows of the triangle of order n)
  __device__ static __forceinline__ void untri(int t, int n, int& a, int& b) {
    a = 0;
    while (t >= n - a) {
      t -= n - a;
      ++a;
    }
    b = a + t;
  }
};

template <class Ws>
__device__ __forceinline__ void wl_unit(const V2Params<Ws>& p, const double* Ibuf, double* Abuf,
                                        double* Bbuf, double* Mbase) {
  constexpr int S = Ws::S, NU = Ws::NU, NV = Ws::NV, NW = Ws::NW, TM = Ws::TM, NQU = Ws::NQU;
  constexpr int NT = Ws::THREADS;
  const int64_t rowstep_m = static_cast<int64_t>(NV * NW) * p.ldM;  // row of m1
#pragma unroll 1
  for (int tile = 0; tile < Ws::NTILE; ++tile) {
    const int t0 = tile * TM;
    // ---- stage A (u), compile-time bands per tile: thread = fiber (k2, k3) of I_s
    static_for<0, Ws::NTILE>([&](auto tc) {
      constexpr int TT = decltype(tc)::value;
      if (tile == TT) {
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          constexpr int Ku = Ws::K(s, 0), Kv = Ws::K(s, 1), Kw = Ws::K(s, 2);
          constexpr int ku = Ws::kind(s, 0);
          for_items<Kv * Kw, NT>([&](int f) {
            const double* Is = Ibuf + Ws::moff(s) + f;  // f = k2*Kw + k3
            double x[Ku];
#pragma unroll
            for (int k1 = 0; k1 < Ku; ++k1) x[k1] = Is[k1 * Kv * Kw];
            double* As = Abuf + Ws::aoff(s) + f;
            static_for<0, TM>([&](auto lc) {
              constexpr int tl = decltype(lc)::value;
              constexpr int t = TT * TM + tl;
              if constexpr (t < NQU) {
                constexpr int m1 = Ws::trow(t), m2 = Ws::tcol(t);
                constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
                constexpr int st = band_step(ku, m1, m2);
                constexpr int co = Ws::coff(0, s, m1, m2);
                double v = 0.0;
                static_for<0, cnt>([&](auto jc) {
                  constexpr int j = decltype(jc)::value;
                  v = fma(p.cu[co + j], x[lo + st * j], v);
                });
                As[tl * Ws::ast(s)] = v;
              }
            });
          });
        });
      }
    });
    __syncthreads();
    const int tcount = NQU - t0 < TM ? NQU - t0 : TM;
    // ---- stage B (v): thread = fiber (tl, k3); n-pairs compile-time
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      constexpr int Kv = Ws::K(s, 1), Kw = Ws::K(s, 2);
      constexpr int kv = Ws::kind(s, 1);
      for (int f = threadIdx.x; f < tcount * Kw; f += NT) {
        const int tl = f / Kw, k3 = f - (f / Kw) * Kw;
        const double* src = Abuf + Ws::aoff(s) + tl * Ws::ast(s) + k3;
        double y[Kv];
#pragma unroll
        for (int k2 = 0; k2 < Kv; ++k2) y[k2] = src[k2 * Kw];
        double* dst = Bbuf + Ws::boff(s) + tl * Ws::bst(s) + k3;
        static_for<0, NV>([&](auto n1c) {
          constexpr int n1 = decltype(n1c)::value;
          static_for<n1, NV>([&](auto n2c) {
            constexpr int n2 = decltype(n2c)::value;
            constexpr int lo = band_lo(kv, n1, n2), cnt = band_count(kv, n1, n2);
            constexpr int st = band_step(kv, n1, n2);
            constexpr int co = Ws::coff(1, s, n1, n2);
            double v = 0.0;
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              v = fma(p.cv[co + j], y[lo + st * j], v);
            });
            dst[Ws::tri(n1, n2, NV) * Kw] = v;
          });
        });
      }
    });
    __syncthreads();
    // ---- stage C (w): thread = fiber (tl, n1, n2), n2 fastest; N_w x N_w block
    for (int f = threadIdx.x; f < tcount * NV * NV; f += NT) {
      const int tl = f / (NV * NV), nn = f - (f / (NV * NV)) * (NV * NV);
      const int n1 = nn / NV, n2 = nn - (nn / NV) * NV;
      const int tn = n1 <= n2 ? Ws::tri(n1, n2, NV) : Ws::tri(n2, n1, NV);
      double z[Ws::KWTOT()];
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        constexpr int Kw = Ws::K(s, 2);
        const double* src = Bbuf + Ws::boff(s) + tl * Ws::bst(s) + tn * Kw;
#pragma unroll
        for (int k3 = 0; k3 < Kw; ++k3) z[Ws::kwoff(s) + k3] = src[k3];
      });
      int m1, m2;
      Ws::untri(t0 + tl, NU, m1, m2);
      double* o1 = Mbase + m1 * rowstep_m + static_cast<int64_t>(n1 * NW) * p.ldM + (m2 * NV + n2) * NW;
      double* o2 = Mbase + m2 * rowstep_m + static_cast<int64_t>(n1 * NW) * p.ldM + (m1 * NV + n2) * NW;
      const bool twice = m1 != m2;
      static_for<0, NW>([&](auto p1c) {
        constexpr int p1 = decltype(p1c)::value;
        double v[NW];
        static_for<0, NW>([&](auto p2c) {
          constexpr int p2 = decltype(p2c)::value;
          double acc = 0.0;
          static_for<0, S>([&](auto sc) {
            constexpr int s = decltype(sc)::value;
            constexpr int kw = Ws::kind(s, 2);
            constexpr int lo = band_lo(kw, p1, p2), cnt = band_count(kw, p1, p2);
            constexpr int st = band_step(kw, p1, p2);
            constexpr int co = Ws::coff(2, s, p1, p2);
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              acc = fma(p.cw[co + j], z[Ws::kwoff(s) + lo + st * j], acc);
            });
          });
          v[p2] = acc;
        });
        if (p.vec2) {
#pragma unroll
          for (int q = 0; q < NW; q += 2) {
            st_cs2(o1 + p1 * p.ldM + q, v[q], v[q + 1]);
            if (twice) st_cs2(o2 + p1 * p.ldM + q, v[q], v[q + 1]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < NW; ++q) {
            st_cs(o1 + p1 * p.ldM + q, v[q]);
            if (twice) st_cs(o2 + p1 * p.ldM + q, v[q]);
          }
        }
      });
    }
    __syncthreads();
  }
}

}  // namespace p2s
