// p2s_large.cuh -- large-order path (C5: N = 16, K = 31 / 29, 36^3 points),
// where one element's moment block (433 KB) and intermediates do not fit a
// CTA's shared memory.  Three kernels per chunk of elements:
//   large_moments_kernel  I_s[k1][k2][k3], one CTA per (unit, term, k1 chunk)
//                         (three even/odd-folded 1-D passes as in
//                         p2s_moments_v2.cuh, pass u restricted to the chunk)
//   large_vw_kernel       X_s[k1][tri(n1,n2)][tri(p1,p2)] =
//                         sum_k2 Cv[n1 n2 k2] sum_k3 Cw[p1 p2 k3] I_s[k1][k2][k3]
//                         one CTA per (unit, term, k1); symmetric v/w kinds, so
//                         only the (n1<=n2, p1<=p2) triangles are formed; the
//                         chunk's X stays L2-resident (8.9 MB per C5 element)
//   large_u_kernel        M[m1 n1 p1][m2 n2 p2] = sum_s sum_k1 Cu[m1 m2 k1] X_s[..]
//                         one CTA per (unit, n1, p1), thread = fiber (n2, p2):
//                         every warp store is 256 contiguous bytes
#pragma once

#include "p2s_kernels.cuh"
#include "p2s_moments_v2.cuh"  // fold_contract

namespace p2s {

template <int NU_, int NV_, int NW_, int QU_, int QV_, int QW_, int KC_, int... TK>
struct LShape {
  static constexpr int NU = NU_, NV = NV_, NW = NW_, KC = KC_;
  static constexpr int S = sizeof...(TK);
  static constexpr int N(int d) { return d == 0 ? NU : d == 1 ? NV : NW; }
  static constexpr int Q(int d) { return d == 0 ? QU_ : d == 1 ? QV_ : QW_; }
  static constexpr int H(int d) { return (Q(d) + 1) / 2; }
  static constexpr int kind(int s, int d) {
    const int k[] = {TK...};
    return (k[s] >> (3 * d)) & 7;
  }
  static constexpr int K(int s, int d) { return kernel_count(kind(s, d), N(d)); }
  static constexpr int KMAX(int d) {
    int m = 0;
    for (int s = 0; s < S; ++s) m = K(s, d) > m ? K(s, d) : m;
    return m;
  }
  static constexpr int NCH = (KMAX(0) + KC - 1) / KC;   // k1 chunks of the moment kernel
  static constexpr int NQV = NV * (NV + 1) / 2, NQW = NW * (NW + 1) / 2;
  static constexpr int tri(int a, int b, int n) { return a * n - a * (a - 1) / 2 + (b - a); }
  static constexpr int moff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0) * K(i, 1) * K(i, 2);
    return o;
  }
  static constexpr int MPP = (moff(S) + 3) & ~3;
  // X block of one unit: terms back to back, [K_u][NQV][NQW]
  static constexpr int64_t xoff(int s) {
    int64_t o = 0;
    for (int i = 0; i < s; ++i) o += static_cast<int64_t>(K(i, 0)) * NQV * NQW;
    return o;
  }
  static constexpr int64_t XPU = xoff(S);
  static constexpr int KUTOT() {
    int o = 0;
    for (int s = 0; s < S; ++s) o += K(s, 0);
    return o;
  }
  static constexpr int kuoff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0);
    return o;
  }
  // u-kernels of term s in the parity class par of m1+m2 (k1 = uk0 + 2 idx)
  static constexpr int ushift(int s) {
    return (base_kind(kind(s, 0)) == DP || base_kind(kind(s, 0)) == PD) ? 1 : 0;
  }
  static constexpr bool u_conforming() {
    for (int s = 0; s < S; ++s)
      if (conforming(kind(s, 0))) return true;
    return false;
  }
  static constexpr int uk0(int s, int par) { return (par + ushift(s)) % 2; }
  static constexpr int ucnt(int s, int par) { return (K(s, 0) - uk0(s, par) + 1) / 2; }
  static constexpr int kpo(int s, int par) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += ucnt(i, par);
    return o;
  }
  static constexpr int KX(int par) { return par < 0 ? KUTOT() : kpo(S, par); }
  // band-packed coefficients of direction d (as Shape::coff)
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
  // shared half tables [KMAX(d)][H(d)] per direction
  static constexpr int ttoff(int d) {
    int o = 0;
    for (int e = 0; e < d; ++e) o += KMAX(e) * H(e);
    return o;
  }
  static constexpr int TALL = ttoff(3);
  static constexpr int S2 = Q(1) | 1, S3 = Q(2) | 1;
  static constexpr size_t MOM_SMEM =
      sizeof(double) * (size_t)(KC * Q(2) * S2 + KC * KMAX(1) * S3);
  static_assert(KC % 2 == 0, "k1 chunks must be even (parity of k1 = parity of the slot)");
  static constexpr bool sym_ok() {
    for (int s = 0; s < S; ++s)
      for (int d = 1; d < 3; ++d)
        if (base_kind(kind(s, d)) != PP && base_kind(kind(s, d)) != DD) return false;
    return true;
  }
  static_assert(sym_ok(), "large path needs symmetric v/w kinds (PP / DD)");
};

// ------------------------------------------------------------------ moments

template <class Ls>
struct LMomParams {
  const double* alpha;
  double* I;
  int64_t n_units;   // E * P
  double tab[Ls::TALL];
};

template <class Ls, int s>
__device__ __forceinline__ void large_moments_term(const LMomParams<Ls>& p, const double* a, double* Iout,
                                                   int chunk, double* sm) {
  constexpr int QU = Ls::Q(0), QV = Ls::Q(1), QW = Ls::Q(2);
  constexpr int KU = Ls::K(s, 0), KV = Ls::K(s, 1), KW = Ls::K(s, 2), KC = Ls::KC;
  constexpr int S2 = Ls::S2, S3 = Ls::S3;
  constexpr int NT = 256;
  const int k0 = chunk * KC;
  if (k0 >= KU) return;
  double* T1 = sm;                         // [KC][QW][S2]
  double* T2 = sm + KC * QW * S2;          // [KC*KV][S3]
  const double* tu = p.tab + Ls::ttoff(0) + k0 * Ls::H(0);
  // pass u (rows of alpha), outputs k1 = k0 .. k0+KC-1
  for_items<QW * QV, NT>([&](int r) {
    constexpr int Hf = QU / 2, H = (QU + 1) / 2;
    const int q3 = r / QV, q2 = r - (r / QV) * QV;
    double x[QU];
    const double2* row = reinterpret_cast<const double2*>(a + static_cast<int64_t>(r) * QU);
    static_assert(QU % 2 == 0, "large path expects an even rule along u");
#pragma unroll
    for (int q = 0; q < QU / 2; ++q) {
      const double2 v = __ldg(row + q);
      x[2 * q] = v.x;
      x[2 * q + 1] = v.y;
    }
    double ev[Hf], od[Hf];
#pragma unroll
    for (int h = 0; h < Hf; ++h) {
      ev[h] = x[h] + x[QU - 1 - h];
      od[h] = x[h] - x[QU - 1 - h];
    }
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      double v = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) v = fma(tu[j * H + h], (j & 1) ? od[h] : ev[h], v);
      T1[(j * QW + q3) * S2 + q2] = v;
    }
  });
  __syncthreads();
  const double* tv = p.tab + Ls::ttoff(1);
  for_items<KC * QW, NT>([&](int r) {
    const int j = r / QW, q3 = r - (r / QW) * QW;
    double x[QV];
#pragma unroll
    for (int q = 0; q < QV; ++q) x[q] = T1[(j * QW + q3) * S2 + q];
    fold_contract<QV, KV>(x, tv, [&](int k, double v) { T2[(j * KV + k) * S3 + q3] = v; });
  });
  __syncthreads();
  const double* tw = p.tab + Ls::ttoff(2);
  for_items<KC * KV, NT>([&](int r) {
    const int j = r / KV, k2 = r - (r / KV) * KV;
    if (k0 + j >= KU) return;
    double x[QW];
#pragma unroll
    for (int q = 0; q < QW; ++q) x[q] = T2[(j * KV + k2) * S3 + q];
    double* out = Iout + ((k0 + j) * KV + k2) * KW;
    fold_contract<QW, KW>(x, tw, [&](int k, double v) { out[k] = v; });
  });
}

template <class Ls>
__global__ void __launch_bounds__(256) large_moments_kernel(const __grid_constant__ LMomParams<Ls> p) {
  extern __shared__ __align__(16) double sm[];
  const int64_t b = blockIdx.x;
  const int chunk = static_cast<int>(b % Ls::NCH);
  const int64_t us = b / Ls::NCH;               // (unit, term)
  const int s = static_cast<int>(us % Ls::S);
  const int64_t unit = us / Ls::S;
  constexpr int slab = Ls::Q(0) * Ls::Q(1) * Ls::Q(2);
  const double* a = p.alpha + us * slab;        // alpha [E][P][S][slab]
  double* Ib = p.I + unit * Ls::MPP;
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int ss = decltype(sc)::value;
    if (s == ss) large_moments_term<Ls, ss>(p, a, Ib + Ls::moff(ss), chunk, sm);
  });
}

// ------------------------------------------------------------------ v/w stage

template <class Ls>
struct LVWParams {
  const double* I;      // [units][MPP]
  double* X;            // [units][XPU]
  const double* cvw;    // global band-packed Cv then Cw (copied to smem per CTA)
  int64_t n_units;
};

template <class Ls>
constexpr size_t large_vw_smem() {
  return sizeof(double) * (size_t)(Ls::KMAX(1) * Ls::KMAX(2) + Ls::NQV * Ls::KMAX(2) +
                                   Ls::ctot(1) + Ls::ctot(2) + 2);
}

template <class Ls, int s>
__device__ __forceinline__ void large_vw_term(const LVWParams<Ls>& p, int64_t unit, int k1, double* sm) {
  constexpr int NV = Ls::NV, NW = Ls::NW, NQV = Ls::NQV, NQW = Ls::NQW;
  constexpr int KV = Ls::K(s, 1), KW = Ls::K(s, 2);
  constexpr int kv = Ls::kind(s, 1), kw = Ls::kind(s, 2);
  constexpr int NT = 256;
  double* Is = sm;                                   // [KV][KW]
  double* Y = Is + Ls::KMAX(1) * Ls::KMAX(2);        // [NQV][KW]
  const double* cv = Y + NQV * Ls::KMAX(2);          // band-packed Cv (smem copy)
  const double* cw = cv + Ls::ctot(1);
  const double* src = p.I + unit * Ls::MPP + Ls::moff(s) + k1 * KV * KW;
  for (int i = threadIdx.x; i < KV * KW; i += NT) Is[i] = src[i];
  __syncthreads();
  // stage A: Y[tri(n1,n2)][k3], thread = (n1, k3), outputs n2 >= n1 (runtime n1,
  // compile-time n2 via dispatch on n1)
  // runtime loops here (coefficients come from smem, nothing to hoist); unrolled
  // rounds would multiply the 136-output dispatch code and thrash the I-cache
  for (int r = threadIdx.x; r < NV * KW; r += NT) {
    const int n1 = r / KW, k3 = r - (r / KW) * KW;
    double x[KV];
#pragma unroll
    for (int k2 = 0; k2 < KV; ++k2) x[k2] = Is[k2 * KW + k3];
    static_for<0, NV>([&](auto n1c) {
      constexpr int a = decltype(n1c)::value;
      if (n1 == a) {
        static_for<a, NV>([&](auto n2c) {
          constexpr int b = decltype(n2c)::value;
          constexpr int lo = band_lo(kv, a, b), cnt = band_count(kv, a, b);
          constexpr int co = Ls::coff(1, s, a, b) - Ls::coff(1, 0, 0, 0);
          double v = 0.0;
          static_for<0, cnt>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            v = fma(cv[co + j], x[lo + band_step(kv, a, b) * j], v);
          });
          Y[Ls::tri(a, b, NV) * KW + k3] = v;
        });
      }
    });
  }
  __syncthreads();
  // stage B: X[qv][tri(p1,p2)], thread = (qv, p1)
  double* Xo = p.X + unit * Ls::XPU + Ls::xoff(s) + static_cast<int64_t>(k1) * NQV * NQW;
  for (int r = threadIdx.x; r < NQV * NW; r += NT) {
    const int p1 = r / NQV, qv = r - (r / NQV) * NQV;   // p1 warp-uniform (dispatch below)
    double y[KW];
#pragma unroll
    for (int k3 = 0; k3 < KW; ++k3) y[k3] = Y[qv * KW + k3];
    double* o = Xo + static_cast<int64_t>(qv) * NQW;
    static_for<0, NW>([&](auto p1c) {
      constexpr int a = decltype(p1c)::value;
      if (p1 == a) {
        static_for<a, NW>([&](auto p2c) {
          constexpr int b = decltype(p2c)::value;
          constexpr int lo = band_lo(kw, a, b), cnt = band_count(kw, a, b);
          constexpr int co = Ls::coff(2, s, a, b) - Ls::coff(2, 0, 0, 0);
          double v = 0.0;
          static_for<0, cnt>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            v = fma(cw[co + j], y[lo + band_step(kw, a, b) * j], v);
          });
          o[Ls::tri(a, b, NW)] = v;
        });
      }
    });
  }
}

template <class Ls>
__global__ void __launch_bounds__(256) large_vw_kernel(const __grid_constant__ LVWParams<Ls> p) {
  extern __shared__ __align__(16) double sm[];
  const int64_t b = blockIdx.x;
  const int row = static_cast<int>(b % Ls::KUTOT());
  const int64_t unit = b / Ls::KUTOT();
  // coefficient copy to smem (after the I slab and Y)
  double* cvs = sm + Ls::KMAX(1) * Ls::KMAX(2) + Ls::NQV * Ls::KMAX(2);
  for (int i = threadIdx.x; i < Ls::ctot(1) + Ls::ctot(2); i += 256) cvs[i] = __ldg(p.cvw + i);
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    if (row >= Ls::kuoff(s) && row < Ls::kuoff(s) + Ls::K(s, 0))
      large_vw_term<Ls, s>(p, unit, row - Ls::kuoff(s), sm);
  });
}

// ------------------------------------------------------------------ u stage

template <class Ls>
struct LUParams {
  const double* X;
  double* M;
  int64_t ldM, mat_stride, n_units;
  int nc, P, Nt;
  double cu[Ls::ctot(0)];
};

// PS: the (m1, m2) classes of even and odd m1+m2 run one after the other, each
// holding only the x_s[k1] of its parity (half the registers: 2 CTAs per SM)
template <class Ls, bool PS>
__global__ void __launch_bounds__(Ls::NV * Ls::NW, PS ? 2 : 1)
    large_u_kernel(const __grid_constant__ LUParams<Ls> p, int64_t unit0) {
  constexpr int NU = Ls::NU, NV = Ls::NV, NW = Ls::NW, S = Ls::S, NQV = Ls::NQV, NQW = Ls::NQW;
  const int64_t b = blockIdx.x;
  const int np = static_cast<int>(b % (NV * NW));
  const int64_t unit = unit0 + b / (NV * NW);
  const int n1 = np / NW, p1 = np - (np / NW) * NW;
  const int n2 = threadIdx.x / NW, p2 = threadIdx.x - (threadIdx.x / NW) * NW;
  const int64_t e = unit / p.P;
  const int pair = static_cast<int>(unit - e * p.P);
  const int gci = pair / p.nc, gcj = pair - gci * p.nc;
  const int qv = n1 <= n2 ? Ls::tri(n1, n2, NV) : Ls::tri(n2, n1, NV);
  const int qw = p1 <= p2 ? Ls::tri(p1, p2, NW) : Ls::tri(p2, p1, NW);
  const double* Xu = p.X + (unit - unit0) * Ls::XPU + static_cast<int64_t>(qv) * NQW + qw;
  double* out = p.M + e * p.mat_stride + static_cast<int64_t>(gci * p.Nt + n1 * NW + p1) * p.ldM +
                gcj * p.Nt + n2 * NW + p2;
  const int64_t rowstep = static_cast<int64_t>(NV * NW) * p.ldM;
  auto run = [&](auto parc) {
    constexpr int PAR = decltype(parc)::value;  // -1: every (m1, m2)
    double x[Ls::KX(PAR)];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      if constexpr (PAR < 0) {
#pragma unroll
        for (int k1 = 0; k1 < Ls::K(s, 0); ++k1)
          x[Ls::kuoff(s) + k1] = __ldg(Xu + Ls::xoff(s) + static_cast<int64_t>(k1) * NQV * NQW);
      } else {
#pragma unroll
        for (int j = 0; j < Ls::ucnt(s, PAR); ++j)
          x[Ls::kpo(s, PAR) + j] = __ldg(
              Xu + Ls::xoff(s) + static_cast<int64_t>(Ls::uk0(s, PAR) + 2 * j) * NQV * NQW);
      }
    });
    auto row = [&](auto m1c) {
      constexpr int m1 = decltype(m1c)::value;
      static_for<0, NU>([&](auto m2c) {
        constexpr int m2 = decltype(m2c)::value;
        if constexpr (PAR < 0 || (m1 + m2) % 2 == PAR) {
          double v = 0.0;
          static_for<0, S>([&](auto sc) {
            constexpr int s = decltype(sc)::value;
            constexpr int ku = Ls::kind(s, 0);
            constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
            constexpr int co = Ls::coff(0, s, m1, m2);
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              constexpr int xi = PAR < 0 ? Ls::kuoff(s) + lo + band_step(ku, m1, m2) * j
                                         : Ls::kpo(s, PAR) + (lo - Ls::uk0(s, PAR)) / 2 + j;
              v = fma(p.cu[co + j], x[xi], v);
            });
          });
          st_cs(out + m1 * rowstep + m2 * (NV * NW), v);
        }
      });
    };
#pragma unroll 1
    for (int m1 = 0; m1 < NU; ++m1)
      static_for<0, NU>([&](auto m1c) {
        if (m1 == decltype(m1c)::value) row(m1c);
      });
  };
  if constexpr (PS && !Ls::u_conforming()) {
    run(std::integral_constant<int, 0>{});
    run(std::integral_constant<int, 1>{});
  } else {
    run(std::integral_constant<int, -1>{});
  }
}

template <class Ls>
void large_u_dispatch(const LUParams<Ls>& p, int64_t unit0, int64_t cnt, bool ps, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(cnt * Ls::NV * Ls::NW);
  if (ps)
    large_u_kernel<Ls, true><<<grid, Ls::NV * Ls::NW, 0, st>>>(p, unit0);
  else
    large_u_kernel<Ls, false><<<grid, Ls::NV * Ls::NW, 0, st>>>(p, unit0);
}

}  // namespace p2s
