// p2s_large.cuh -- large-order path (C5: N = 16, K = 31 / 29, 36^3 points),
// where one element's moment block (433 KB) and intermediates do not fit a
// CTA's shared memory.  Kernels per chunk of elements:
//   large_moments_w_kernel  I_s[k1][k2][k3], one CTA per (unit, term, k3 chunk):
//                         w-first register-tiled passes (default; section "w-first
//                         tiled moments" below)
//   large_moments_kernel  the round-1 kernel, one CTA per (unit, term, k1 chunk)
//                         (three even/odd-folded 1-D passes as in
//                         p2s_moments_v2.cuh, pass u restricted to the chunk); used
//                         where the w-first kernel's first pass is too narrow
//   large_w_kernel,       X_s[k1][tri(n1,n2)][p1][p2] =
//   large_v_kernel        sum_k2 Cv[n1 n2 k2] sum_k3 Cw[p1 p2 k3] I_s[k1][k2][k3]
//                         (w step into Z, then v step; symmetric v kinds, so
//                         only the n1 <= n2 triangle is formed; full (p1, p2)
//                         rows for coalesced u-stage loads); the chunk's X stays
//                         L2-resident (16.7 MB per C5 element)
//   large_u_kernel        M[m1 n1 p1][m2 n2 p2] = sum_s sum_k1 Cu[m1 m2 k1] X_s[..]
//                         one CTA per (unit, n1, p1), thread = fiber (n2, p2):
//                         every warp store is 256 contiguous bytes
#pragma once

#include <cooperative_groups.h>

#include "p2s_kernels.cuh"
#include "p2s_launch.cuh"
#include "p2s_moments_v2.cuh"  // fold_contract

#ifndef P2S_LARGE_MOM_THREADS
#define P2S_LARGE_MOM_THREADS 256  // threads of large_moments_kernel
#endif
#ifndef P2S_LARGE_MOM_MINB
#define P2S_LARGE_MOM_MINB 2
#endif

#ifndef P2S_LARGE_FIB2_MINB
#define P2S_LARGE_FIB2_MINB 2  // CTAs per SM of the two-fiber u stage (3: 170-register cap, spills)
#endif

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
  // symmetric v kinds (PP / DD, either basis): X holds the n1 <= n2 triangle, else
  // the full N_v x N_v square
  static constexpr bool v_symmetric() {
    for (int s = 0; s < S; ++s)
      if (base_kind(kind(s, 1)) != PP && base_kind(kind(s, 1)) != DD) return false;
    return true;
  }
  static constexpr bool VSYM = v_symmetric();
  static constexpr int NQV = VSYM ? NV * (NV + 1) / 2 : NV * NV, NQW = NW * (NW + 1) / 2;
  static constexpr int tri(int a, int b, int n) { return a * n - a * (a - 1) / 2 + (b - a); }
  // slot of (n1, n2) in X
  static constexpr int vidx(int a, int b) { return VSYM ? (a <= b ? tri(a, b, NV) : tri(b, a, NV)) : a * NV + b; }
  static constexpr int moff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0) * K(i, 1) * K(i, 2);
    return o;
  }
  static constexpr int MPP = (moff(S) + 3) & ~3;
  // X block of one unit: terms back to back, [K_u][NQV][N_w][N_w] (v triangle,
  // full (p1, p2): the u stage's lanes read contiguous p2 runs)
  static constexpr int64_t xoff(int s) {
    int64_t o = 0;
    for (int i = 0; i < s; ++i) o += static_cast<int64_t>(K(i, 0)) * NQV * NW * NW;
    return o;
  }
  static constexpr int64_t XPU = xoff(S);
  // Z block of one unit (w-contracted moments): terms back to back,
  // [K_u][N_w][N_w][K2P], k2 fastest and padded to a power of two >= 4 (32-B fiber
  // loads in the v step; one lane per k2 up to 32, two k2 per lane above).  (A fixed
  // pad of 32 made Z of a (10, 1, 14) shape, K_v = 1, 2.8 MB per unit written 8 bytes
  // per 256: the w step took 0.5 ms per chunk whatever its thread mapping.)
  static constexpr int K2P = KMAX(1) > 32 ? 64 : KMAX(1) > 16 ? 32 : KMAX(1) > 8 ? 16 : KMAX(1) > 4 ? 8 : 4;
  static constexpr int64_t zoff(int s) {
    int64_t o = 0;
    for (int i = 0; i < s; ++i) o += static_cast<int64_t>(K(i, 0)) * NW * NW * K2P;
    return o;
  }
  static constexpr int64_t ZPU = zoff(S);
  static constexpr int NGRP = (NW + 1) / 2;  // w-step p1 groups {g, N_w-1-g}
  // w step: a warp's lanes are k2; with few kernel polynomials along v (small N_v)
  // a warp takes WR = 32 / K2S consecutive k1 rows of a term (lane = (k1 offset, k2))
  // instead of idling 32 - K_v lanes -- (10, 1, 14): K_v = 1, one lane in 32 worked
  static constexpr int K2S = KMAX(1) > 16 ? 32 : KMAX(1) > 8 ? 16 : KMAX(1) > 4 ? 8 : KMAX(1) > 2 ? 4 : KMAX(1) > 1 ? 2 : 1;
  static constexpr int WR = 32 / K2S;
  static constexpr int kgrp(int s) { return (K(s, 0) + WR - 1) / WR; }  // row groups of term s
  static constexpr int kgoff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += kgrp(i);
    return o;
  }
  static constexpr int KGTOT() { return kgoff(S); }
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
  // band-packed coefficients travel as kernel parameters (constant bank, LDCU with
  // immediate offsets) unless a direction's table exceeds what fits the 32 KB
  // parameter space; then kernels read them from global memory (uniform __ldg)
  static constexpr int kParamBytes = 30 * 1024;
  static constexpr bool GC(int d) { return ctot(d) * 8 > kParamBytes; }
  static constexpr int cpar(int d) { return GC(d) ? 1 : ctot(d); }
  // ... staged once per CTA into shared memory (uniform-address LDS instead of one
  // global load per FMA) while the table leaves room for the kernel's own buffers
  static constexpr bool GS(int d) { return GC(d) && ctot(d) * 8 <= 128 * 1024; }
  static constexpr size_t cs_bytes(int d) { return GS(d) ? sizeof(double) * static_cast<size_t>(ctot(d)) : 0; }
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
  static_assert(KMAX(1) <= 64, "w step: at most 64 kernel polynomials along v");
  // symmetric u-kinds: the u stage forms m2 >= m1 and stores (m1, m2) and (m2, m1)
  // (as Shape::USYM); -DP2S_LARGE_NOUSYM turns it off for A/B measurements
  static constexpr bool u_symmetric() {
    for (int s = 0; s < S; ++s)
      if (base_kind(kind(s, 0)) != PP && base_kind(kind(s, 0)) != DD) return false;
    return true;
  }
#ifdef P2S_LARGE_NOUSYM
  static constexpr bool USYM = false;
#else
  static constexpr bool USYM = u_symmetric();
#endif
  // u stage: one thread per fiber (n2, p2); CTAs per SM the launch bounds ask
  // for (register cap 65536 / (UT * UMINB)): 3 CTAs of 144 threads for N = 12
  // (ncu: 2 CTAs left the SM at 15 % occupancy, latency-bound), 2 of 256 for C5
  static constexpr int UT = NV * NW;
  static constexpr int UMINB = UT <= 96 ? 4 : UT <= 170 ? 3 : UT <= 256 ? 2 : 1;
};

// ------------------------------------------------------------------ moments

template <class Ls>
struct LMomParams {
  const double* alpha;
  double* I;
  int64_t n_units;   // E * P
  double tab[Ls::TALL];
};

// CL (cluster mode): the NCH chunk CTAs of one (unit, term) form a thread-block
// cluster; each loads and folds 1/NCH of the alpha rows once, computes every k1
// of them and stores each value into the T1 of the CTA owning that k1 through
// distributed shared memory -- alpha is read and folded once instead of NCH times.
template <class Ls, int s, bool CL>
__device__ __forceinline__ void large_moments_term(const LMomParams<Ls>& p, const double* a, double* Iout,
                                                   int chunk, double* sm) {
  constexpr int QU = Ls::Q(0), QV = Ls::Q(1), QW = Ls::Q(2);
  constexpr int KU = Ls::K(s, 0), KV = Ls::K(s, 1), KW = Ls::K(s, 2), KC = Ls::KC;
  constexpr int S2 = Ls::S2, S3 = Ls::S3;
  constexpr int NT = P2S_LARGE_MOM_THREADS;
  const int k0 = chunk * KC;
  double* T1 = sm;                         // [KC][QW][S2]
  double* T2 = sm + KC * QW * S2;          // [KC*KV][S3]
  if constexpr (CL) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int NCH = Ls::NCH, H = (QU + 1) / 2, Hf = QU / 2;
    constexpr int RPC = (QW * QV + NCH - 1) / NCH;  // alpha rows per CTA
    static_assert(QU % 2 == 0, "cluster moments expect an even rule along u");
    double* peer[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) peer[c] = cl.map_shared_rank(T1, c);
    const double* tu = p.tab + Ls::ttoff(0);
    for_items<RPC, NT>([&](int i) {
      const int r = chunk * RPC + i;
      if (r >= QW * QV) return;
      const int q3 = r / QV, q2 = r - (r / QV) * QV;
      double x[QU];
      load_row<QU>(a + static_cast<int64_t>(r) * QU, x);
      double ev[Hf], od[Hf];
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        ev[h] = x[h] + x[QU - 1 - h];
        od[h] = x[h] - x[QU - 1 - h];
      }
#pragma unroll
      for (int k1 = 0; k1 < KU; ++k1) {
        double v = 0.0;
#pragma unroll
        for (int h = 0; h < Hf; ++h) v = fma(tu[k1 * H + h], (k1 & 1) ? od[h] : ev[h], v);
        peer[k1 / KC][((k1 % KC) * QW + q3) * S2 + q2] = v;
      }
    });
    cl.sync();  // every T1 complete (and no remote access after this point)
    if (k0 >= KU) return;
  } else {
  if (k0 >= KU) return;
  const double* tu = p.tab + Ls::ttoff(0) + k0 * Ls::H(0);
  // pass u (rows of alpha), outputs k1 = k0 .. k0+KC-1
  for_items<QW * QV, NT>([&](int r) {
    constexpr int Hf = QU / 2, H = (QU + 1) / 2;
    const int q3 = r / QV, q2 = r - (r / QV) * QV;
    double x[QU];
    load_row<QU>(a + static_cast<int64_t>(r) * QU, x);
    double ev[Hf > 0 ? Hf : 1], od[Hf > 0 ? Hf : 1];
#pragma unroll
    for (int h = 0; h < Hf; ++h) {
      ev[h] = x[h] + x[QU - 1 - h];
      od[h] = x[h] - x[QU - 1 - h];
    }
#pragma unroll
    for (int j = 0; j < KC; ++j) {  // k1 = k0 + j, k0 even: parity of j = parity of k1
      double v = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) v = fma(tu[j * H + h], (j & 1) ? od[h] : ev[h], v);
      if constexpr (QU & 1)  // centre node (odd rule): even k only
        if ((j & 1) == 0) v = fma(tu[j * H + Hf], x[Hf], v);
      T1[(j * QW + q3) * S2 + q2] = v;
    }
  });
  __syncthreads();
  }
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

template <class Ls, bool CL = false>
__global__ void __launch_bounds__(P2S_LARGE_MOM_THREADS, Ls::MOM_SMEM <= 110 * 1024 ? P2S_LARGE_MOM_MINB : 1) large_moments_kernel(const __grid_constant__ LMomParams<Ls> p) {
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
    if (s == ss) large_moments_term<Ls, ss, CL>(p, a, Ib + Ls::moff(ss), chunk, sm);
  });
}

// Grouped moments: same CTA = (unit, term, k1 chunk) and the same folded u pass,
// but the v and w passes hand out (row, k group) items -- a group is up to KG
// kernel polynomials of one parity -- instead of one row with all K outputs per
// thread.  (ncu, C5, r2h: a chunk has K_C Q_w = 144 rows in pass v and K_C K_v =
// 124 in pass w for 256 threads, so half the warps idled through two of the
// three passes, each live thread ran a 558-DFMA chain, and 28 % of the executed
// instructions were UMOV / LDC shuffling 62 uniform registers: 21 % FP64 pipe.)
// A thread folds its row to the group's parity with one DFMA per pair (sign as a
// runtime factor: exact, no divergence between groups) and reads its group's
// table rows from shared memory, so lanes of different groups share the code.
#ifndef P2S_LARGE_MOMG_THREADS
#define P2S_LARGE_MOMG_THREADS 288
#endif
#ifndef P2S_LARGE_MOMG_KG
#define P2S_LARGE_MOMG_KG 8
#endif

template <class Ls>
struct LMomG {
  static constexpr int NT = P2S_LARGE_MOMG_THREADS, KG = P2S_LARGE_MOMG_KG;
  static constexpr int hp(int d) { return (Ls::H(d) + 1) & ~1; }  // table row stride: 16-byte rows
  static constexpr int groups(int K) { return ((K + 1) / 2 + KG - 1) / KG + (K / 2 + KG - 1) / KG; }
  static constexpr int T1D = Ls::KC * Ls::Q(2) * Ls::S2, T2D = Ls::KC * Ls::KMAX(1) * Ls::S3;
  static constexpr int TVO = (T1D + T2D + 1) & ~1;                // staged v table, then the w table
  // each table is followed by 2 KG pad rows (zeros): a short last group runs all KG chains
  static constexpr int TWO = TVO + (Ls::KMAX(1) + 2 * KG) * hp(1);
  static constexpr size_t SMEM = sizeof(double) * static_cast<size_t>(TWO + (Ls::KMAX(2) + 2 * KG) * hp(2));
  static constexpr bool FITS = SMEM <= 227 * 1024;
  static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;
};

// outputs of k group g of a[Q] against the staged half table tbs[K][HP]
template <int Q, int K, int KG, int HP, class Out>
__device__ __forceinline__ void fold_contract_group(const double (&a)[Q], const double* tbs, int g, Out&& out) {
  constexpr int Hf = Q / 2, H = (Q + 1) / 2;
  constexpr int NE = (K + 1) / 2, NO = K / 2, GE = (NE + KG - 1) / KG;
  const bool odd = g >= GE;
  const double sg = odd ? -1.0 : 1.0;
  double f[H];
#pragma unroll
  for (int h = 0; h < Hf; ++h) f[h] = fma(sg, a[Q - 1 - h], a[h]);  // a[h] +- a[Q-1-h], one rounding
  if constexpr (Q & 1) f[Hf] = odd ? 0.0 : a[Hf];                    // centre node: even k only
  const int gi = odd ? g - GE : g;
  const int kb = (odd ? 1 : 0) + 2 * KG * gi;
  const int n = (odd ? NO : NE) - KG * gi;
  const double* t = tbs + kb * HP;
  // KG independent accumulation chains (a short last group reads the table's pad rows)
  double v[KG];
#pragma unroll
  for (int i = 0; i < KG; ++i) v[i] = 0.0;
#pragma unroll
  for (int h = 0; h < H; ++h)
#pragma unroll
    for (int i = 0; i < KG; ++i) v[i] = fma(t[i * 2 * HP + h], f[h], v[i]);
#pragma unroll
  for (int i = 0; i < KG; ++i)
    if (i < n) out(kb + 2 * i, v[i]);
}

template <class Ls, int s>
__device__ __forceinline__ void large_moments_g_term(const LMomParams<Ls>& p, const double* a, double* Iout,
                                                     int chunk, double* sm) {
  constexpr int QU = Ls::Q(0), QV = Ls::Q(1), QW = Ls::Q(2);
  constexpr int KU = Ls::K(s, 0), KV = Ls::K(s, 1), KW = Ls::K(s, 2), KC = Ls::KC;
  constexpr int S2 = Ls::S2, S3 = Ls::S3;
  using G = LMomG<Ls>;
  constexpr int NT = G::NT, KG = G::KG;
  const int k0 = chunk * KC;
  if (k0 >= KU) return;
  const int kc = KU - k0 < KC ? KU - k0 : KC;  // live k1 of this chunk
  double* T1 = sm;             // [KC][QW][S2]
  double* T2 = sm + G::T1D;    // [KC*KV][S3]
  const double* tu = p.tab + Ls::ttoff(0) + k0 * Ls::H(0);
  for_items<QW * QV, NT>([&](int r) {
    constexpr int Hf = QU / 2, H = (QU + 1) / 2;
    const int q3 = r / QV, q2 = r - (r / QV) * QV;
    double x[QU];
    load_row<QU>(a + static_cast<int64_t>(r) * QU, x);
    double ev[Hf > 0 ? Hf : 1], od[Hf > 0 ? Hf : 1];
#pragma unroll
    for (int h = 0; h < Hf; ++h) {
      ev[h] = x[h] + x[QU - 1 - h];
      od[h] = x[h] - x[QU - 1 - h];
    }
#pragma unroll
    for (int j = 0; j < KC; ++j) {  // k1 = k0 + j, k0 even: parity of j = parity of k1
      double v = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) v = fma(tu[j * H + h], (j & 1) ? od[h] : ev[h], v);
      if constexpr (QU & 1)
        if ((j & 1) == 0) v = fma(tu[j * H + Hf], x[Hf], v);
      T1[(j * QW + q3) * S2 + q2] = v;
    }
  });
  __syncthreads();  // also orders the table staging of the kernel before its first use
  {
    const double* tvs = sm + G::TVO;
    const int rows = kc * QW;
    for (int it = threadIdx.x; it < rows * G::groups(KV); it += NT) {
      const int g = it / rows, r = it - g * rows;
      const int j = r / QW, q3 = r - j * QW;
      double x[QV];
#pragma unroll
      for (int q = 0; q < QV; ++q) x[q] = T1[r * S2 + q];
      fold_contract_group<QV, KV, KG, G::hp(1)>(x, tvs, g, [&](int k, double v) { T2[(j * KV + k) * S3 + q3] = v; });
    }
  }
  __syncthreads();
  // pass w: the chunk's outputs are one contiguous run of I; they go to shared
  // memory first (T1 is free) and leave in one coalesced sweep when they fit
  constexpr bool kStage = KC * KV * KW <= G::T1D;
  double* Ic = Iout + static_cast<int64_t>(k0) * KV * KW;
  {
    const double* tws = sm + G::TWO;
    const int rows = kc * KV;  // row r = (j, k2)
    for (int it = threadIdx.x; it < rows * G::groups(KW); it += NT) {
      const int g = it / rows, r = it - g * rows;
      double x[QW];
#pragma unroll
      for (int q = 0; q < QW; ++q) x[q] = T2[r * S3 + q];
      fold_contract_group<QW, KW, KG, G::hp(2)>(x, tws, g, [&](int k, double v) {
        if constexpr (kStage)
          T1[r * KW + k] = v;
        else
          Ic[r * KW + k] = v;
      });
    }
    if constexpr (kStage) {
      __syncthreads();
      for (int i = threadIdx.x; i < rows * KW; i += NT) Ic[i] = T1[i];
    }
  }
}

template <class Ls>
__global__ void __launch_bounds__(LMomG<Ls>::NT, LMomG<Ls>::MINB)
    large_moments_g_kernel(const __grid_constant__ LMomParams<Ls> p) {
  extern __shared__ __align__(16) double sm[];
  using G = LMomG<Ls>;
  // half tables of the v and w passes -> shared memory, rows padded to an even length
  for (int d = 1; d <= 2; ++d) {
    const int H = d == 1 ? Ls::H(1) : Ls::H(2), HP = d == 1 ? G::hp(1) : G::hp(2);
    const int K = d == 1 ? Ls::KMAX(1) : Ls::KMAX(2);
    double* dst = sm + (d == 1 ? G::TVO : G::TWO);
    const double* src = p.tab + (d == 1 ? Ls::ttoff(1) : Ls::ttoff(2));
    for (int i = threadIdx.x; i < (K + 2 * G::KG) * HP; i += G::NT) {
      const int k = i / HP, h = i - k * HP;
      dst[i] = (h < H && k < K) ? src[k * H + h] : 0.0;
    }
  }
  const int64_t b = blockIdx.x;
  const int chunk = static_cast<int>(b % Ls::NCH);
  const int64_t us = b / Ls::NCH;               // (unit, term)
  const int s = static_cast<int>(us % Ls::S);
  const int64_t unit = us / Ls::S;
  constexpr int slab = Ls::Q(0) * Ls::Q(1) * Ls::Q(2);
  const double* a = p.alpha + us * slab;
  double* Ib = p.I + unit * Ls::MPP;
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int ss = decltype(sc)::value;
    if (s == ss) large_moments_g_term<Ls, ss>(p, a, Ib + Ls::moff(ss), chunk, sm);
  });
}

// Tiled moments: the three passes as register-tiled contractions.  ncu (r2h) on the
// two kernels above: every DFMA of a one-row-per-thread pass needs its own
// coefficient operand (LDCU / LDS), and both stall on operand delivery at 21 % of
// the FP64 pipe whatever the thread mapping.  Here a thread owns TWO rows -- the
// pair the NEXT pass folds together (q2 / Q_v-1-q2 in pass u, q3 / Q_w-1-q3 in pass
// v) -- so each coefficient feeds two DFMAs, the producer stores the folded sum and
// difference (even / odd tables read only their half), and passes v / w block KG
// kernel polynomials of one parity per thread: 2 x KG accumulators against 2 data +
// KG coefficient loads per quadrature pair.  Same FMA order per output as the
// kernels above (bitwise equal moments).
#ifndef P2S_LARGE_MOMT_THREADS
#define P2S_LARGE_MOMT_THREADS 224
#endif
#ifndef P2S_LARGE_MOMT_KG
#define P2S_LARGE_MOMT_KG 8
#endif

template <class Ls>
struct LMomT {
  static constexpr int NT = P2S_LARGE_MOMT_THREADS, KG = P2S_LARGE_MOMT_KG;
  static constexpr int hp(int d) { return (Ls::H(d) + 1) & ~1; }  // table row stride: 16-byte rows
  // folded-row stride: even (16-byte rows) with stride / 2 odd, so the 16-byte loads
  // of eight consecutive rows fall into eight different bank groups
  static constexpr int rs(int d) {
    const int r = (Ls::H(d) + 1) & ~1;
    return (r / 2) % 2 ? r : r + 2;
  }
  static constexpr int groups(int K) { return ((K + 1) / 2 + KG - 1) / KG + (K / 2 + KG - 1) / KG; }
  static constexpr int T1H = Ls::KC * Ls::Q(2) * rs(1);       // T1 even part, then the odd part
  static constexpr int T2H = Ls::KC * Ls::KMAX(1) * rs(2);    // T2 even part, then the odd part
  static constexpr int TVO = 2 * T1H + 2 * T2H;
  static constexpr int TWO = TVO + (Ls::KMAX(1) + 2 * KG) * hp(1);  // 2 KG zero pad rows per table
  static constexpr int TUO = TWO + (Ls::KMAX(2) + 2 * KG) * hp(2);  // the chunk's KC rows of the u table
  static constexpr size_t SMEM = sizeof(double) * static_cast<size_t>(TUO + Ls::KC * hp(0));
  static constexpr bool FITS = SMEM <= 227 * 1024;
  static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;
};

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// va[i], vb[i] = sum_h t[2 i][h] * fa[h], fb[h]  (two folded rows, KG table rows of one parity)
template <int H, int KG, int HP>
__device__ __forceinline__ void mom_tile2(const double* fa, const double* fb, const double* t,
                                          double (&va)[KG], double (&vb)[KG]) {
#pragma unroll
  for (int i = 0; i < KG; ++i) va[i] = vb[i] = 0.0;
#pragma unroll
  for (int h2 = 0; h2 < H / 2; ++h2) {
    const double2 a = lds2(fa + 2 * h2), b = lds2(fb + 2 * h2);
#pragma unroll
    for (int i = 0; i < KG; ++i) {
      const double2 c = lds2(t + i * 2 * HP + 2 * h2);
      va[i] = fma(c.x, a.x, va[i]);
      vb[i] = fma(c.x, b.x, vb[i]);
      va[i] = fma(c.y, a.y, va[i]);
      vb[i] = fma(c.y, b.y, vb[i]);
    }
  }
  if constexpr (H & 1) {
    const double a = fa[H - 1], b = fb[H - 1];
#pragma unroll
    for (int i = 0; i < KG; ++i) {
      const double c = t[i * 2 * HP + H - 1];
      va[i] = fma(c, a, va[i]);
      vb[i] = fma(c, b, vb[i]);
    }
  }
}

// W adjacent doubles of an alpha row (W = 4: 32-byte, 2: 16-byte, 1), schedulable loads
template <int W>
__device__ __forceinline__ void ld_chunk(const double* p, double (&x)[W]) {
  if constexpr (W == 4) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                 : "l"(p));
  } else if constexpr (W == 2) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    x[0] = v.x;
    x[1] = v.y;
  } else {
    x[0] = __ldg(p);
  }
}

template <class Ls, int s>
__device__ __forceinline__ void large_moments_t_term(const LMomParams<Ls>& p, const double* a, double* Iout,
                                                     int chunk, double* sm) {
  constexpr int QU = Ls::Q(0), QV = Ls::Q(1), QW = Ls::Q(2);
  constexpr int HU = Ls::H(0), HV = Ls::H(1), HW = Ls::H(2);
  constexpr int KU = Ls::K(s, 0), KV = Ls::K(s, 1), KW = Ls::K(s, 2), KC = Ls::KC;
  using G = LMomT<Ls>;
  constexpr int NT = G::NT, KG = G::KG, RS1 = G::rs(1), RS2 = G::rs(2);
  const int k0 = chunk * KC;
  if (k0 >= KU) return;
  const int kc = KU - k0 < KC ? KU - k0 : KC;  // live k1 of this chunk
  double* T1e = sm;                 // [KC][QW][RS1]: sum of the rows q2, Q_v-1-q2 (h = q2 < H_v)
  double* T1o = sm + G::T1H;        //                difference
  double* T2e = sm + 2 * G::T1H;    // [KC * KV][RS2]: sum / difference of q3, Q_w-1-q3
  double* T2o = T2e + G::T2H;
  // ---- pass u: item = (q3, h2): alpha rows (q3, h2) and (q3, Q_v-1-h2), KC outputs each
  {
    constexpr int W = QU % 4 == 0 ? 4 : QU % 2 == 0 ? 2 : 1;
    constexpr int Hf = QU / 2, NCK = (Hf + W - 1) / W;
    constexpr int PD = NCK < 3 ? NCK : 3;  // chunks of loads in flight ahead of the arithmetic
    constexpr int HPU = G::hp(0);
    const double* tu = sm + G::TUO;        // [KC][HPU], staged by the kernel (uniform-address LDS)
    for_items<QW * HV, NT>([&](int item) {
      const int q3 = item / HV, h2 = item - (item / HV) * HV;
      const int q2b = QV - 1 - h2;
      const double* A = a + static_cast<int64_t>(q3 * QV + h2) * QU;
      const double* B = a + static_cast<int64_t>(q3 * QV + q2b) * QU;
      double vA[KC], vB[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j) vA[j] = vB[j] = 0.0;
      // chunk c = the W values from h = W c of both rows and their mirror images
      double af[NCK][W], ab[NCK][W], bf[NCK][W], bb[NCK][W];
      auto issue = [&](auto cc) {
        constexpr int c = decltype(cc)::value;
#ifdef P2S_MOMT_FAKE_COALESCED  // timing experiment only (wrong data): lane-consecutive 32-byte pieces
        const double* F = a + (item % NT) * W + (item / NT) * 36864;
        ld_chunk<W>(F + (4 * c + 0) * 1024, af[c]);
        ld_chunk<W>(F + (4 * c + 1) * 1024, ab[c]);
        ld_chunk<W>(F + (4 * c + 2) * 1024, bf[c]);
        ld_chunk<W>(F + (4 * c + 3) * 1024, bb[c]);
#else
        ld_chunk<W>(A + W * c, af[c]);
        ld_chunk<W>(A + QU - W - W * c, ab[c]);
        ld_chunk<W>(B + W * c, bf[c]);
        ld_chunk<W>(B + QU - W - W * c, bb[c]);
#endif
      };
      static_for<0, PD>([&](auto cc) { issue(cc); });
      static_for<0, NCK>([&](auto cc) {
        constexpr int c = decltype(cc)::value;
        if constexpr (c + PD < NCK) issue(std::integral_constant<int, c + PD>{});
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int h = W * c + w;
          if (h < Hf) {
            const double ae = af[c][w] + ab[c][W - 1 - w], ao = af[c][w] - ab[c][W - 1 - w];
            const double be = bf[c][w] + bb[c][W - 1 - w], bo = bf[c][w] - bb[c][W - 1 - w];
#pragma unroll
            for (int j = 0; j < KC; ++j) {  // k1 = k0 + j, k0 even: parity of j = parity of k1
              const double cf = tu[j * HPU + h];
              vA[j] = fma(cf, (j & 1) ? ao : ae, vA[j]);
              vB[j] = fma(cf, (j & 1) ? bo : be, vB[j]);
            }
          }
        }
      });
      if constexpr (QU & 1) {  // centre node: even k only
        const double ac = __ldg(A + Hf), bc = __ldg(B + Hf);
#pragma unroll
        for (int j = 0; j < KC; j += 2) {
          vA[j] = fma(tu[j * HPU + Hf], ac, vA[j]);
          vB[j] = fma(tu[j * HPU + Hf], bc, vB[j]);
        }
      }
      const double cb = h2 == q2b ? 0.0 : 1.0;  // centre row of an odd rule: the row itself, no partner
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        T1e[(j * QW + q3) * RS1 + h2] = fma(cb, vB[j], vA[j]);
        T1o[(j * QW + q3) * RS1 + h2] = vA[j] - vB[j];
      }
    });
  }
  __syncthreads();  // also orders the kernel's table staging before its first use
  // ---- pass v: item = (j, h3, k2 group): T1 rows q3 = h3 and Q_w-1-h3
  {
    constexpr int NE = (KV + 1) / 2, NO = KV / 2, GE = (NE + KG - 1) / KG, HP = G::hp(1);
    const double* tvs = sm + G::TVO;
    const int rows = kc * HW;
    for (int it = threadIdx.x; it < rows * G::groups(KV); it += NT) {
      const int g = it / rows, r = it - g * rows;
      const int j = r / HW, h3 = r - j * HW;
      const int q3b = QW - 1 - h3;
      const bool odd = g >= GE;
      const int gi = odd ? g - GE : g;
      const int kb = (odd ? 1 : 0) + 2 * KG * gi;
      const int n = (odd ? NO : NE) - KG * gi;
      const double* src = (odd ? T1o : T1e) + j * QW * RS1;
      double va[KG], vb[KG];
      mom_tile2<HV, KG, HP>(src + h3 * RS1, src + q3b * RS1, tvs + kb * HP, va, vb);
      const double cb = h3 == q3b ? 0.0 : 1.0;
#pragma unroll
      for (int i = 0; i < KG; ++i)
        if (i < n) {
          const int o = (j * KV + kb + 2 * i) * RS2 + h3;
          T2e[o] = fma(cb, vb[i], va[i]);
          T2o[o] = va[i] - vb[i];
        }
    }
  }
  __syncthreads();
  // ---- pass w: item = (row pair, k3 group), rows (j, k2) = r and r + ceil(R / 2); the
  // chunk's outputs are one contiguous run of I: through shared memory (T1 is free)
  // and out in one coalesced sweep when they fit
  constexpr bool kStage = KC * KV * KW <= 2 * G::T1H;
  double* Ic = Iout + static_cast<int64_t>(k0) * KV * KW;
  {
    constexpr int NE = (KW + 1) / 2, NO = KW / 2, GE = (NE + KG - 1) / KG, HP = G::hp(2);
    const double* tws = sm + G::TWO;
    const int R = kc * KV, RH = (R + 1) / 2;
    double* dst = kStage ? sm : Ic;
    for (int it = threadIdx.x; it < RH * G::groups(KW); it += NT) {
      const int g = it / RH, ra = it - g * RH;
      const bool live_b = ra + RH < R;
      const int rb = live_b ? ra + RH : ra;
      const bool odd = g >= GE;
      const int gi = odd ? g - GE : g;
      const int kb = (odd ? 1 : 0) + 2 * KG * gi;
      const int n = (odd ? NO : NE) - KG * gi;
      const double* src = odd ? T2o : T2e;
      double va[KG], vb[KG];
      mom_tile2<HW, KG, HP>(src + ra * RS2, src + rb * RS2, tws + kb * HP, va, vb);
#pragma unroll
      for (int i = 0; i < KG; ++i)
        if (i < n) {
          dst[ra * KW + kb + 2 * i] = va[i];
          if (live_b) dst[rb * KW + kb + 2 * i] = vb[i];
        }
    }
    if constexpr (kStage) {
      __syncthreads();
      for (int i = threadIdx.x; i < R * KW; i += NT) Ic[i] = sm[i];
    }
  }
}

template <class Ls>
__global__ void __launch_bounds__(LMomT<Ls>::NT, LMomT<Ls>::MINB)
    large_moments_t_kernel(const __grid_constant__ LMomParams<Ls> p) {
  extern __shared__ __align__(16) double sm[];
  using G = LMomT<Ls>;
  const int64_t b = blockIdx.x;
  const int chunk = static_cast<int>(b % Ls::NCH);
  // half tables of the v and w passes and the chunk's rows of the u table -> shared
  // memory, rows padded to an even length (independent loads: the trip counts are
  // compile-time, so the constant-bank latencies overlap)
  static_for<0, 3>([&](auto dc) {
    constexpr int d = decltype(dc)::value;
    constexpr int H = Ls::H(d), HP = G::hp(d);
    constexpr int K = d == 0 ? Ls::KC : Ls::KMAX(d), ROWS = d == 0 ? Ls::KC : K + 2 * G::KG;
    double* dst = sm + (d == 0 ? G::TUO : d == 1 ? G::TVO : G::TWO);
    const double* src = p.tab + Ls::ttoff(d) + (d == 0 ? chunk * Ls::KC * H : 0);
    const int kmax = d == 0 ? Ls::KMAX(0) - chunk * Ls::KC : K;  // rows past the table: zeros
#pragma unroll
    for (int i0 = 0; i0 < ROWS * HP; i0 += G::NT) {
      const int i = i0 + static_cast<int>(threadIdx.x);
      const int k = i / HP, h = i - k * HP;
      if (i < ROWS * HP) dst[i] = (h < H && k < kmax) ? src[k * H + h] : 0.0;
    }
  });
  __syncthreads();  // pass u reads the staged u rows
  const int64_t us = b / Ls::NCH;               // (unit, term)
  const int s = static_cast<int>(us % Ls::S);
  const int64_t unit = us / Ls::S;
  constexpr int slab = Ls::Q(0) * Ls::Q(1) * Ls::Q(2);
  const double* a = p.alpha + us * slab;
  double* Ib = p.I + unit * Ls::MPP;
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int ss = decltype(sc)::value;
    if (s == ss) large_moments_t_term<Ls, ss>(p, a, Ib + Ls::moff(ss), chunk, sm);
  });
}

// w-first tiled moments: as the tiled kernel, but the first pass contracts the
// SLOWEST direction (q3) and the CTA's chunk is KC kernel polynomials along w.
// Pass u of the kernels above gives every lane its own 288-byte alpha row: each
// 32-byte sector is its own L2 request (ncu r2h: 47.8 M sector requests, 0.8 % L1
// hits, 11.8 wavefronts per load instruction), and four differently organised
// kernels all ran C5 at 1.13-1.29 us per element; the tiled kernel with the same
// sectors read lane-contiguously (wrong data, timing only: -DP2S_MOMT_FAKE_COALESCED)
// ran at 0.85.  Here a thread owns the column pair (q2; q1 = h, Q_u-1-h) and walks
// q3: consecutive lanes read consecutive doubles of an alpha row.  Then pass u
// (over q1, rows folded by the first pass) and pass v (over q2) as tiles; the
// chunk's outputs I[k1][k2][k0..k0+KC) leave through shared memory.  The sums run
// w, u, v instead of u, v, w: same values to rounding (tests: 1e-12), not bitwise.
#ifndef P2S_LARGE_MOMW_PD
#define P2S_LARGE_MOMW_PD 4
#endif

template <class Ls>
struct LMomW {
  static constexpr int KG = P2S_LARGE_MOMT_KG, KC = Ls::KC;
  static constexpr int hp(int d) { return LMomT<Ls>::hp(d); }
  static constexpr int rs(int d) { return LMomT<Ls>::rs(d); }
  static constexpr int groups(int K) { return LMomT<Ls>::groups(K); }
  static constexpr int NCH = (Ls::KMAX(2) + KC - 1) / KC;        // k3 chunks
  static constexpr int T1H = KC * Ls::Q(1) * rs(0);              // [KC][QV][rs(0)]: q1 folded (even, then odd)
  static constexpr int T2H = KC * Ls::KMAX(0) * rs(1);           // [KC * KU][rs(1)]: q2 folded
  static constexpr int TUO = 2 * T1H + 2 * T2H;                  // u table, 2 KG zero pad rows
  static constexpr int TVO = TUO + (Ls::KMAX(0) + 2 * KG) * hp(0);
  static constexpr int TWO = TVO + (Ls::KMAX(1) + 2 * KG) * hp(1);  // the chunk's w rows, [H_w][KC]
  static constexpr size_t SMEM = sizeof(double) * static_cast<size_t>(TWO + Ls::H(2) * KC);
  static constexpr bool FITS = SMEM <= 227 * 1024;
  static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;
  // two CTAs of 224 threads per SM (144-register cap), or one of 352 when the chunk's scratch needs the SM
  static constexpr int NT = MINB == 2 ? P2S_LARGE_MOMT_THREADS : 352;
};

__device__ __forceinline__ double ld_nc_v(const double* p) {  // issue order = source order
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <class Ls, int s>
__device__ __forceinline__ void large_moments_w_term(const LMomParams<Ls>& p, const double* a, double* Iout,
                                                     int chunk, double* sm) {
  constexpr int QU = Ls::Q(0), QV = Ls::Q(1), QW = Ls::Q(2);
  constexpr int HU = Ls::H(0), HV = Ls::H(1);
  constexpr int KU = Ls::K(s, 0), KV = Ls::K(s, 1), KW = Ls::K(s, 2), KC = Ls::KC;
  using G = LMomW<Ls>;
  constexpr int NT = G::NT, KG = G::KG, RS0 = G::rs(0), RS1 = G::rs(1);
  const int k0 = chunk * KC;
  if (k0 >= KW) return;
  const int kc = KW - k0 < KC ? KW - k0 : KC;  // live k3 of this chunk
  double* T1e = sm;
  double* T1o = sm + G::T1H;
  double* T2e = sm + 2 * G::T1H;
  double* T2o = T2e + G::T2H;
  // ---- pass w: item = (q2, h1): columns q1 = h1 and Q_u-1-h1 of alpha row q2, all q3
  {
    constexpr int Hf = QW / 2, PD = Hf < P2S_LARGE_MOMW_PD ? Hf : P2S_LARGE_MOMW_PD;  // q3 pairs in flight
    constexpr int64_t PS = static_cast<int64_t>(QV) * QU;  // plane stride
    const double* tw = sm + G::TWO;                         // [H_w][KC]
    for_items<QV * HU, NT>([&](int item) {
      const int q2 = item / HU, h1 = item - (item / HU) * HU;
      const int q1b = QU - 1 - h1;
      const double* Pa = a + q2 * QU + h1;
      const double* Pb = a + q2 * QU + q1b;
      double wA[KC], wB[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j) wA[j] = wB[j] = 0.0;
      double xa0[Hf > 0 ? Hf : 1], xa1[Hf > 0 ? Hf : 1], xb0[Hf > 0 ? Hf : 1], xb1[Hf > 0 ? Hf : 1];
      auto issue = [&](auto hc) {
        constexpr int h = decltype(hc)::value;
        xa0[h] = ld_nc_v(Pa + h * PS);
        xb0[h] = ld_nc_v(Pb + h * PS);
        xa1[h] = ld_nc_v(Pa + (QW - 1 - h) * PS);
        xb1[h] = ld_nc_v(Pb + (QW - 1 - h) * PS);
      };
      static_for<0, PD>([&](auto hc) { issue(hc); });
      static_for<0, Hf>([&](auto hc) {
        constexpr int h = decltype(hc)::value;
        if constexpr (h + PD < Hf) issue(std::integral_constant<int, h + PD>{});
        const double ea = xa0[h] + xa1[h], oa = xa0[h] - xa1[h];
        const double eb = xb0[h] + xb1[h], ob = xb0[h] - xb1[h];
#pragma unroll
        for (int j = 0; j < KC; ++j) {  // k3 = k0 + j, k0 even: parity of j = parity of k3
          const double cf = tw[h * KC + j];
          wA[j] = fma(cf, (j & 1) ? oa : ea, wA[j]);
          wB[j] = fma(cf, (j & 1) ? ob : eb, wB[j]);
        }
      });
      if constexpr (QW & 1) {  // centre plane: even k only
        const double ac = __ldg(Pa + Hf * PS), bc = __ldg(Pb + Hf * PS);
#pragma unroll
        for (int j = 0; j < KC; j += 2) {
          wA[j] = fma(tw[Hf * KC + j], ac, wA[j]);
          wB[j] = fma(tw[Hf * KC + j], bc, wB[j]);
        }
      }
      const double cb = h1 == q1b ? 0.0 : 1.0;  // centre column of an odd rule: no partner
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        T1e[(j * QV + q2) * RS0 + h1] = fma(cb, wB[j], wA[j]);
        T1o[(j * QV + q2) * RS0 + h1] = wA[j] - wB[j];
      }
    });
  }
  // u and v half tables (rows padded to an even length, 2 KG zero rows behind) -> shared memory
  static_for<0, 2>([&](auto dc) {
    constexpr int d = decltype(dc)::value;
    constexpr int H = Ls::H(d), HP = G::hp(d), K = Ls::KMAX(d), ROWS = K + 2 * G::KG;
    double* dst = sm + (d == 0 ? G::TUO : G::TVO);
    const double* src = p.tab + Ls::ttoff(d);
#pragma unroll
    for (int i0 = 0; i0 < ROWS * HP; i0 += G::NT) {
      const int i = i0 + static_cast<int>(threadIdx.x);
      const int k = i / HP, h = i - k * HP;
      if (i < ROWS * HP) dst[i] = (h < H && k < K) ? src[k * H + h] : 0.0;
    }
  });
  __syncthreads();
  // ---- pass u: item = (j, h2, k1 group): T1 rows q2 = h2 and Q_v-1-h2
  {
    constexpr int NE = (KU + 1) / 2, NO = KU / 2, GE = (NE + KG - 1) / KG, HP = G::hp(0);
    const double* tus = sm + G::TUO;
    const int rows = kc * HV;
    for (int it = threadIdx.x; it < rows * G::groups(KU); it += NT) {
      const int g = it / rows, r = it - g * rows;
      const int j = r / HV, h2 = r - j * HV;
      const int q2b = QV - 1 - h2;
      const bool odd = g >= GE;
      const int gi = odd ? g - GE : g;
      const int kb = (odd ? 1 : 0) + 2 * KG * gi;
      const int n = (odd ? NO : NE) - KG * gi;
      const double* src = (odd ? T1o : T1e) + j * QV * RS0;
      double va[KG], vb[KG];
      mom_tile2<HU, KG, HP>(src + h2 * RS0, src + q2b * RS0, tus + kb * HP, va, vb);
      const double cb = h2 == q2b ? 0.0 : 1.0;
#pragma unroll
      for (int i = 0; i < KG; ++i)
        if (i < n) {
          const int o = (j * KU + kb + 2 * i) * RS1 + h2;
          T2e[o] = fma(cb, vb[i], va[i]);
          T2o[o] = va[i] - vb[i];
        }
    }
  }
  __syncthreads();
  // ---- pass v: item = (row pair, k2 group), rows (j, k1) = r and r + ceil(R / 2); the
  // outputs I[k1][k2][k0 + j] go through shared memory (T1 is free) when they fit
  constexpr bool kStage = KC * KU * KV <= 2 * G::T1H;
  {
    constexpr int NE = (KV + 1) / 2, NO = KV / 2, GE = (NE + KG - 1) / KG, HP = G::hp(1);
    const double* tvs = sm + G::TVO;
    const int R = kc * KU, RH = (R + 1) / 2;
    for (int it = threadIdx.x; it < RH * G::groups(KV); it += NT) {
      const int g = it / RH, ra = it - g * RH;
      const bool live_b = ra + RH < R;
      const int rb = live_b ? ra + RH : ra;
      const bool odd = g >= GE;
      const int gi = odd ? g - GE : g;
      const int kb = (odd ? 1 : 0) + 2 * KG * gi;
      const int n = (odd ? NO : NE) - KG * gi;
      const double* src = odd ? T2o : T2e;
      double va[KG], vb[KG];
      mom_tile2<HV, KG, HP>(src + ra * RS1, src + rb * RS1, tvs + kb * HP, va, vb);
      const int ja = ra / KU, k1a = ra - ja * KU, jb = rb / KU, k1b = rb - jb * KU;
#pragma unroll
      for (int i = 0; i < KG; ++i)
        if (i < n) {
          const int k2 = kb + 2 * i;
          if constexpr (kStage) {
            sm[(k1a * KV + k2) * KC + ja] = va[i];
            if (live_b) sm[(k1b * KV + k2) * KC + jb] = vb[i];
          } else {
            Iout[(k1a * KV + k2) * KW + k0 + ja] = va[i];
            if (live_b) Iout[(k1b * KV + k2) * KW + k0 + jb] = vb[i];
          }
        }
    }
    if constexpr (kStage) {
      __syncthreads();
#pragma unroll 4
      for (int i = threadIdx.x; i < KU * KV * KC; i += NT) {
        const int e = i / KC, j = i - e * KC;
        if (j < kc) Iout[e * KW + k0 + j] = sm[i];
      }
    }
  }
}

template <class Ls>
__global__ void __launch_bounds__(LMomW<Ls>::NT, LMomW<Ls>::MINB)
    large_moments_w_kernel(const __grid_constant__ LMomParams<Ls> p) {
  extern __shared__ __align__(16) double sm[];
  using G = LMomW<Ls>;
  const int64_t b = blockIdx.x;
  const int chunk = static_cast<int>(b % G::NCH);
  // the chunk's rows of the w table, transposed to [h][j], -> shared memory (the u and
  // v tables follow behind pass w, off the start of the CTA)
  {
    constexpr int H = Ls::H(2), KC = Ls::KC;
    const double* src = p.tab + Ls::ttoff(2);
#pragma unroll
    for (int i0 = 0; i0 < H * KC; i0 += G::NT) {
      const int i = i0 + static_cast<int>(threadIdx.x);
      const int h = i / KC, j = i - h * KC;
      if (i < H * KC) sm[G::TWO + i] = chunk * KC + j < Ls::KMAX(2) ? src[(chunk * KC + j) * H + h] : 0.0;
    }
  }
  __syncthreads();  // pass w reads the staged w rows
  const int64_t us = b / G::NCH;                // (unit, term)
  const int s = static_cast<int>(us % Ls::S);
  const int64_t unit = us / Ls::S;
  constexpr int slab = Ls::Q(0) * Ls::Q(1) * Ls::Q(2);
  const double* a = p.alpha + us * slab;
  double* Ib = p.I + unit * Ls::MPP;
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int ss = decltype(sc)::value;
    if (s == ss) large_moments_w_term<Ls, ss>(p, a, Ib + Ls::moff(ss), chunk, sm);
  });
}

// Split moments (default): the u pass of every (unit, term) computes ALL its
// K_u outputs per alpha row at once -- each row is read and folded once, 18 FMAs
// per k1 against 36 loaded values instead of 4 k1 per pass -- into a
// k1-major scratch T1g [K_u][Q_w][Q_v] (L2-resident: the launcher walks the
// batch in sub-batches); then one CTA per (unit, term, k1 chunk) loads its T1
// rows into shared memory and runs the v and w passes as above.  (The fused
// per-chunk kernel re-read and re-folded every alpha row once per k1 chunk:
// 0.33 of the FP64 peak on C5.)
template <class Ls>
struct LMomSplit {
  static constexpr int QU = Ls::Q(0), QV = Ls::Q(1), QW = Ls::Q(2);
  static constexpr int64_t T1U = static_cast<int64_t>(Ls::KMAX(0)) * QW * QV;  // per (unit, term)
  static constexpr int ROWS = 128;  // alpha rows (threads) per u-pass CTA
  static constexpr size_t VW_SMEM = Ls::MOM_SMEM;
};

template <class Ls>
__global__ void __launch_bounds__(LMomSplit<Ls>::ROWS)
    large_mom_u_kernel(const __grid_constant__ LMomParams<Ls> p, double* __restrict__ T1g, int64_t ut0) {
  constexpr int QU = Ls::Q(0), QV = Ls::Q(1), QW = Ls::Q(2), S = Ls::S;
  constexpr int RB = (QW * QV + LMomSplit<Ls>::ROWS - 1) / LMomSplit<Ls>::ROWS;  // row blocks per (unit, term)
  const int64_t ut = blockIdx.x / RB;                 // (unit, term) within the sub-batch
  const int r = static_cast<int>(blockIdx.x % RB) * LMomSplit<Ls>::ROWS + threadIdx.x;
  if (r >= QW * QV) return;
  const int s = static_cast<int>((ut0 + ut) % S);
  constexpr int slab = QU * QV * QW;
  double x[QU];
  load_row<QU>(p.alpha + (ut0 + ut) * slab + static_cast<int64_t>(r) * QU, x);
  constexpr int Hf = QU / 2, H = (QU + 1) / 2;
  double ev[Hf > 0 ? Hf : 1], od[Hf > 0 ? Hf : 1];
#pragma unroll
  for (int h = 0; h < Hf; ++h) {
    ev[h] = x[h] + x[QU - 1 - h];
    od[h] = x[h] - x[QU - 1 - h];
  }
  const double* tu = p.tab + Ls::ttoff(0);
  double* out = T1g + ut * LMomSplit<Ls>::T1U + r;
  static_for<0, S>([&](auto sc) {
    constexpr int ss = decltype(sc)::value;
    if (s == ss) {
#pragma unroll 4
      for (int k = 0; k < Ls::K(ss, 0); ++k) {
        double v = 0.0;
        if (k & 1) {
#pragma unroll
          for (int h = 0; h < Hf; ++h) v = fma(tu[k * H + h], od[h], v);
        } else {
#pragma unroll
          for (int h = 0; h < Hf; ++h) v = fma(tu[k * H + h], ev[h], v);
          if constexpr (QU & 1) v = fma(tu[k * H + Hf], x[Hf], v);
        }
        __stcg(out + static_cast<int64_t>(k) * QW * QV, v);  // L2: read back by the v/w pass
      }
    }
  });
}

template <class Ls, int s>
__device__ __forceinline__ void large_mom_vw_term(const LMomParams<Ls>& p, const double* T1u, double* Iout,
                                                  int chunk, double* sm) {
  constexpr int QV = Ls::Q(1), QW = Ls::Q(2);
  constexpr int KU = Ls::K(s, 0), KV = Ls::K(s, 1), KW = Ls::K(s, 2), KC = Ls::KC;
  constexpr int S2 = Ls::S2, S3 = Ls::S3;
  constexpr int NT = P2S_LARGE_MOM_THREADS;
  const int k0 = chunk * KC;
  if (k0 >= KU) return;
  double* T1 = sm;                         // [KC][QW][S2]
  double* T2 = sm + KC * QW * S2;          // [KC*KV][S3]
  const int nrow = (KU - k0 < KC ? KU - k0 : KC) * QW * QV;
  const double* src = T1u + static_cast<int64_t>(k0) * QW * QV;
  for (int i = threadIdx.x; i < nrow; i += NT) {
    const int jq = i / QV, q2 = i - (i / QV) * QV;
    T1[jq * S2 + q2] = __ldcg(src + i);
  }
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
__global__ void __launch_bounds__(P2S_LARGE_MOM_THREADS, Ls::MOM_SMEM <= 110 * 1024 ? P2S_LARGE_MOM_MINB : 1)
    large_mom_vw_kernel(const __grid_constant__ LMomParams<Ls> p, const double* __restrict__ T1g, int64_t ut0) {
  extern __shared__ __align__(16) double sm[];
  const int64_t b = blockIdx.x;
  const int chunk = static_cast<int>(b % Ls::NCH);
  const int64_t ut = b / Ls::NCH;
  const int64_t us = ut0 + ut;                    // global (unit, term)
  const int s = static_cast<int>(us % Ls::S);
  const int64_t unit = us / Ls::S;
  double* Ib = p.I + unit * Ls::MPP;
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int ss = decltype(sc)::value;
    if (s == ss) large_mom_vw_term<Ls, ss>(p, T1g + ut * LMomSplit<Ls>::T1U, Ib + Ls::moff(ss), chunk, sm);
  });
}

// ------------------------------------------------------------------ v/w stage
// Two steps, both "fiber in registers, compile-time bands, constant-bank
// coefficients, coalesced stores" kernels:
//   w step  Z_s[k1][p1][p2][k2] = sum_k3 Cw[p1 p2 k3] I_s[k1][k2][k3]
//           warp = (unit, term, k1, p1 group {g, N_w-1-g}), lane = k2 with the
//           I row (K_w values) in registers; lanes store consecutive k2
//   v step  X_s[k1][tri(n1,n2)][p1][p2] = sum_k2 Cv[n1 n2 k2] Z_s[k1][p1][p2][k2]
//           CTA = (unit, term, k1), thread = (p1, p2) with its Z fiber (K_v
//           values) in registers; every warp store is 256 contiguous bytes
// (w first: its fibers are the K_v rows of I, the v step's the N_w^2 rows of Z,
// so the wide n1 <= n2 triangle is produced by the step with the most threads.)

template <class Ls>
struct LWParams {
  const double* I;      // [units][MPP]
  double* Z;            // [units][ZPU]
  const double* cg;     // device copy of cw (GC(2): read from global memory)
  int64_t n_units;
  double cw[Ls::cpar(2)];
};

template <class Ls>
struct LVParams {
  const double* Z;
  double* X;            // [units][XPU]
  const double* cg;     // device copy of cv (GC(1))
  int ns;               // n1 slices: CTA blockIdx % ns forms the outputs with n1 % ns == slice
  int64_t n_units;
  double cv[Ls::cpar(1)];
};

// coefficient i of direction D: constant-bank kernel parameter, or global memory
// when the direction's table exceeds the parameter space
// (`glob` is the CTA's shared-memory copy when Ls::GS(D): see stage_coef)
template <class Ls, int D>
__device__ __forceinline__ double lcoef(const double* par, const double* __restrict__ glob, int i) {
  if constexpr (Ls::GS(D))
    return glob[i];
  else if constexpr (Ls::GC(D))
    return __ldg(glob + i);
  else
    return par[i];
}

// Copy direction D's over-size coefficient table into shared memory (all threads of
// the CTA, coalesced; ends with a barrier) and return the pointer lcoef reads.
template <class Ls, int D>
__device__ __forceinline__ const double* stage_coef(const double* __restrict__ glob, double* sh) {
  if constexpr (Ls::GS(D)) {
    for (int i = threadIdx.x; i < Ls::ctot(D); i += blockDim.x) sh[i] = __ldg(glob + i);
    __syncthreads();
    return sh;
  } else {
    return glob;
  }
}

template <class Ls, int s>
__device__ __forceinline__ void large_w_row(const LWParams<Ls>& p, const double* cw, const double* cg,
                                            int64_t unit, int grp, int g, int lane) {
  constexpr int NW = Ls::NW, K2P = Ls::K2P;
  constexpr int KU = Ls::K(s, 0), KV = Ls::K(s, 1), KW = Ls::K(s, 2), kw = Ls::kind(s, 2);
  static_assert(KV <= K2P, "w step maps k2 to lanes");
  // lane = (k1 offset, k2): WR rows of K2S lanes (WR = 1: one row, k2 = lane, lane + 32)
  const int k1 = grp * Ls::WR + lane / Ls::K2S;
  if (k1 >= KU) return;
#pragma unroll 1
  for (int k2 = lane % Ls::K2S; k2 < KV; k2 += Ls::K2S) {
  const double* src = p.I + unit * Ls::MPP + Ls::moff(s) + (k1 * KV + k2) * KW;
  double y[KW];
#pragma unroll
  for (int k3 = 0; k3 < KW; ++k3) y[k3] = src[k3];
  double* Zk = p.Z + unit * Ls::ZPU + Ls::zoff(s) + static_cast<int64_t>(k1) * NW * NW * K2P + k2;
  auto prow = [&](auto p1c) {
    constexpr int a = decltype(p1c)::value;
    static_for<0, NW>([&](auto p2c) {
      constexpr int b = decltype(p2c)::value;
      constexpr int lo = band_lo(kw, a, b), cnt = band_count(kw, a, b);
      constexpr int co = Ls::coff(2, s, a, b);
      double v = 0.0;
      static_for<0, cnt>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        v = fma(lcoef<Ls, 2>(cw, cg, co + j), y[lo + band_step(kw, a, b) * j], v);
      });
      Zk[(a * NW + b) * K2P] = v;
    });
  };
  // rows g and N_w-1-g (one each per group: balanced band work)
  static_for<0, Ls::NGRP>([&](auto gc) {
    constexpr int gg = decltype(gc)::value;
    if (g == gg) {
      prow(std::integral_constant<int, gg>{});
      if constexpr (NW - 1 - gg != gg) prow(std::integral_constant<int, NW - 1 - gg>{});
    }
  });
  }
}

// w step: CTA = 8 warps on 8 consecutive (unit, row) items, all in the same p1
// group, so the CTA's warps read one small coefficient set (the two p1 rows of
// the group) in lockstep -- constant-cache hits.  (Mapping the groups to the
// warps of one row instead put 8 different coefficient regions of the N = 16
// table (26 KB) on an SM at once: LDCU misses, 4 % issue.)
constexpr int kLargeWWarps = 8;

template <class Ls>
__global__ void __launch_bounds__(32 * kLargeWWarps) large_w_kernel(const __grid_constant__ LWParams<Ls> p) {
  extern __shared__ __align__(16) double csh[];
  const double* cg = stage_coef<Ls, 2>(p.cg, csh);
  const int lane = threadIdx.x & 31;
  const int g = static_cast<int>(blockIdx.x % Ls::NGRP);
  const int64_t item = static_cast<int64_t>(blockIdx.x / Ls::NGRP) * kLargeWWarps + threadIdx.x / 32;
  const int row = static_cast<int>(item % Ls::KGTOT());   // (term, group of WR k1 rows)
  const int64_t unit = item / Ls::KGTOT();
  if (unit >= p.n_units) return;
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    if (row >= Ls::kgoff(s) && row < Ls::kgoff(s) + Ls::kgrp(s))
      large_w_row<Ls, s>(p, p.cw, cg, unit, row - Ls::kgoff(s), g, lane);
  });
}

// v-step CTA: VR consecutive (unit, k1) rows of N_w^2 threads each (>= 128
// threads: small N_w would otherwise launch CTAs of a few threads)
template <class Ls>
struct LVRows {
  static constexpr int F = Ls::NW * Ls::NW;
  static constexpr int VR = F >= 128 ? 1 : (128 + F - 1) / F;
};

template <class Ls>
__global__ void __launch_bounds__(LVRows<Ls>::VR * Ls::NW * Ls::NW) large_v_kernel(const __grid_constant__ LVParams<Ls> p) {
  constexpr int NV = Ls::NV, NW = Ls::NW, NQV = Ls::NQV, K2P = Ls::K2P;
  constexpr int F = LVRows<Ls>::F;
  extern __shared__ __align__(16) double csh[];
  const double* cg = stage_coef<Ls, 1>(p.cg, csh);
  const int rl = LVRows<Ls>::VR == 1 ? 0 : static_cast<int>(threadIdx.x) / F;
  const int slice = static_cast<int>(blockIdx.x % p.ns);
  const int64_t b = static_cast<int64_t>(blockIdx.x / p.ns) * LVRows<Ls>::VR + rl;
  const int row = static_cast<int>(b % Ls::KUTOT());
  const int64_t unit = b / Ls::KUTOT();
  if (unit >= p.n_units) return;
  const int t = static_cast<int>(threadIdx.x) - rl * F;  // p1 * N_w + p2
  static_for<0, Ls::S>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    constexpr int KV = Ls::K(s, 1), kv = Ls::kind(s, 1);
    if (row < Ls::kuoff(s) || row >= Ls::kuoff(s) + Ls::K(s, 0)) return;
    const int k1 = row - Ls::kuoff(s);
    // the thread's Z fiber: K2P contiguous doubles (32-B aligned), 32-B loads
    const double* src = p.Z + unit * Ls::ZPU + Ls::zoff(s) + (static_cast<int64_t>(k1) * NW * NW + t) * K2P;
    double z[(KV + 3) & ~3];
#pragma unroll
    for (int q = 0; q < (KV + 3) / 4; ++q) ld_nc4(src + 4 * q, z[4 * q], z[4 * q + 1], z[4 * q + 2], z[4 * q + 3]);
    double* Xk = p.X + unit * Ls::XPU + Ls::xoff(s) + static_cast<int64_t>(k1) * NQV * NW * NW + t;
    static_for<0, NV>([&](auto n1c) {
      constexpr int a = decltype(n1c)::value;
      if (a % p.ns != slice) return;  // CTA-uniform: this n1 row belongs to another slice
      static_for<(Ls::VSYM ? a : 0), NV>([&](auto n2c) {
        constexpr int c = decltype(n2c)::value;
        constexpr int lo = band_lo(kv, a, c), cnt = band_count(kv, a, c);
        constexpr int co = Ls::coff(1, s, a, c);
        double v = 0.0;
        static_for<0, cnt>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          v = fma(lcoef<Ls, 1>(p.cv, cg, co + j), z[lo + band_step(kv, a, c) * j], v);
        });
        Xk[Ls::vidx(a, c) * NW * NW] = v;
      });
    });
  });
}

// ------------------------------------------------------------------ u stage

template <class Ls>
struct LUParams {
  const double* X;
  double* M;
  const double* cu_g;   // device copy of cu (SMEMC: staged into shared memory per CTA)
  int xs;               // XS mode: x classes staged in shared memory by the TMA engine
  int bulk;             // BULK mode: rows written with TMA bulk stores (M rows 16-B aligned)
  int roll;             // XS kernel: runtime row loop (1) or every row unrolled (0)
  int pair;             // PAIR mode: two adjacent fibers per thread, 16-B stores (M rows 16-B aligned)
  int64_t ldM, mat_stride, n_units;
  int nc, P, Nt;
  double cu[Ls::cpar(0)];
};

// PS: the (m1, m2) classes of even and odd m1+m2 run one after the other, each
// holding only the x_s[k1] of its parity (half the registers).
// FIB fibers per thread: thread (n2, p2) of a CTA of N_v N_w / FIB threads also
// owns the fibers n2 + i N_v / FIB; every constant-bank coefficient feeds FIB
// DFMAs (half the LDCU per DFMA at FIB = 2, 3 CTAs of 128 threads per SM).
template <class Ls, bool PS, int FIB, bool SMEMC>
__device__ __forceinline__ void large_u_tile(const LUParams<Ls>& p, const double* cus, int64_t unit0,
                                             int64_t b, int tid) {
  constexpr int NU = Ls::NU, NV = Ls::NV, NW = Ls::NW, S = Ls::S, NQV = Ls::NQV;
  static_assert(NV % FIB == 0, "fibers per thread must divide N_v");
  const int np = static_cast<int>(b % (NV * NW));
  const int64_t unit = unit0 + b / (NV * NW);
  const int n1 = np / NW, p1 = np - (np / NW) * NW;
  const int n2b = tid / NW, p2 = tid - (tid / NW) * NW;
  const int64_t e = unit / p.P;
  const int pair = static_cast<int>(unit - e * p.P);
  const int gci = pair / p.nc, gcj = pair - gci * p.nc;
  const double* Xu[FIB];
#pragma unroll
  for (int f = 0; f < FIB; ++f) {
    const int n2 = n2b + f * (NV / FIB);
    const int qv = Ls::vidx(n1, n2);
    Xu[f] = p.X + (unit - unit0) * Ls::XPU + (static_cast<int64_t>(qv) * NW + p1) * NW + p2;
  }
  double* out = p.M + e * p.mat_stride + static_cast<int64_t>(gci * p.Nt + n1 * NW + p1) * p.ldM +
                gcj * p.Nt + n2b * NW + p2;
  constexpr int FSTEP = (NV / FIB) * NW;  // column offset between a thread's fibers
  const int64_t rowstep = static_cast<int64_t>(NV * NW) * p.ldM;
  auto run = [&](auto parc) {
    constexpr int PAR = decltype(parc)::value;  // -1: every (m1, m2)
    double x[FIB][Ls::KX(PAR)];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
#pragma unroll
      for (int f = 0; f < FIB; ++f) {
        if constexpr (PAR < 0) {
#pragma unroll
          for (int k1 = 0; k1 < Ls::K(s, 0); ++k1)
            x[f][Ls::kuoff(s) + k1] = __ldg(Xu[f] + Ls::xoff(s) + static_cast<int64_t>(k1) * NQV * NW * NW);
        } else {
#pragma unroll
          for (int j = 0; j < Ls::ucnt(s, PAR); ++j)
            x[f][Ls::kpo(s, PAR) + j] = __ldg(
                Xu[f] + Ls::xoff(s) + static_cast<int64_t>(Ls::uk0(s, PAR) + 2 * j) * NQV * NW * NW);
        }
      }
    });
    auto row = [&](auto m1c) {
      constexpr int m1 = decltype(m1c)::value;
      static_for<(Ls::USYM ? m1 : 0), NU>([&](auto m2c) {
        constexpr int m2 = decltype(m2c)::value;
        if constexpr (PAR < 0 || (m1 + m2) % 2 == PAR) {
          double v[FIB];
#pragma unroll
          for (int f = 0; f < FIB; ++f) v[f] = 0.0;
          static_for<0, S>([&](auto sc) {
            constexpr int s = decltype(sc)::value;
            constexpr int ku = Ls::kind(s, 0);
            constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
            constexpr int co = Ls::coff(0, s, m1, m2);
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              constexpr int xi = PAR < 0 ? Ls::kuoff(s) + lo + band_step(ku, m1, m2) * j
                                         : Ls::kpo(s, PAR) + (lo - Ls::uk0(s, PAR)) / 2 + j;
              const double c = SMEMC ? cus[co + j] : lcoef<Ls, 0>(p.cu, p.cu_g, co + j);
#pragma unroll
              for (int f = 0; f < FIB; ++f) v[f] = fma(c, x[f][xi], v[f]);
            });
          });
#pragma unroll
          for (int f = 0; f < FIB; ++f) {
            st_cs(out + m1 * rowstep + m2 * (NV * NW) + f * FSTEP, v[f]);
            if constexpr (Ls::USYM && m2 != m1) st_cs(out + m2 * rowstep + m1 * (NV * NW) + f * FSTEP, v[f]);
          }
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
    // the odd class's x lines go to L1 while the even class computes
#pragma unroll
    for (int f = 0; f < FIB; ++f)
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
#pragma unroll
        for (int j = 0; j < Ls::ucnt(s, 1); ++j)
          prefetch_l1(Xu[f] + Ls::xoff(s) + static_cast<int64_t>(Ls::uk0(s, 1) + 2 * j) * NQV * NW * NW);
      });
    run(std::integral_constant<int, 0>{});
    run(std::integral_constant<int, 1>{});
  } else {
    run(std::integral_constant<int, -1>{});
  }
}

// SMEMC: the coefficients are copied once per (persistent) CTA from global memory
// into shared memory (coalesced) and read as uniform-address LDS; else they are
// constant-bank operands (LDCU).
// tiles per CTA of the plain u stage (one fiber per thread): as LUXs
template <class Ls, int FIB>
struct LUPlain {
  static constexpr int T = Ls::NV * Ls::NW / FIB;
  static constexpr int TPC = (FIB == 1 && T < 128) ? (128 + T - 1) / T : 1;
  static constexpr int THREADS = TPC * T;
  static constexpr int MINB = THREADS <= 96 ? 4 : THREADS <= 170 ? 3 : THREADS <= 256 ? 2 : 1;
};

template <class Ls, bool PS, int FIB, bool SMEMC = false>
__global__ void __launch_bounds__(LUPlain<Ls, FIB>::THREADS,
                                  PS ? (FIB == 1 ? LUPlain<Ls, FIB>::MINB : P2S_LARGE_FIB2_MINB) : 1)
    large_u_kernel(const __grid_constant__ LUParams<Ls> p, int64_t unit0, int64_t ntiles) {
  extern __shared__ __align__(16) double cus[];
  if constexpr (SMEMC) {
    for (int i = threadIdx.x; i < Ls::ctot(0); i += blockDim.x) cus[i] = __ldg(p.cu_g + i);
    __syncthreads();
  }
  // TPC tiles per CTA iteration (group g = tile it * TPC + g), grid-stride over the
  // iterations when the grid is smaller (persistent CTAs); tiles are independent
  constexpr int T = LUPlain<Ls, FIB>::T, TPC = LUPlain<Ls, FIB>::TPC;
  const int g = TPC == 1 ? 0 : static_cast<int>(threadIdx.x) / T;
  const int tid = static_cast<int>(threadIdx.x) - g * T;
  const int64_t nit = (ntiles + TPC - 1) / TPC;
#pragma unroll 1
  for (int64_t it = blockIdx.x; it < nit; it += gridDim.x) {
    const int64_t b = it * TPC + g;
    if (b < ntiles) large_u_tile<Ls, PS, FIB, SMEMC>(p, cus, unit0, b, tid);
  }
}

// XS mode (persistent, parity split, one fiber per thread): each thread's x
// values of the next parity class (of this tile or of the CTA's next tile) are
// copied into its shared-memory slots with cp.async while the current class
// computes, so a class starts with 30 shared-memory loads instead of 30 L2 loads.
// (A first version with one 128-byte TMA bulk copy per (k1, n2) row issued by one
// warp ran at 21.4 k elem/s vs 28.5 k: the TMA engine is slow on tiny copies.)
template <class Ls>
struct LUXs {
  static constexpr int NV = Ls::NV, NW = Ls::NW, T = NV * NW;
  static constexpr int KXM = Ls::KX(0) > Ls::KX(1) ? Ls::KX(0) : Ls::KX(1);
  // tiles per CTA: a tile has only N_v N_w fibers (threads); anisotropic shapes
  // with few (e.g. 17 x 3) would run 2-warp CTAs at a few CTAs per SM, so a CTA
  // takes TPC consecutive tiles (>= 128 threads; 1 for c12 / C5)
  static constexpr int TPC = T >= 128 ? 1 : (128 + T - 1) / T;
  static constexpr int THREADS = TPC * T;
  static constexpr int MINB = THREADS <= 96 ? 4 : THREADS <= 170 ? 3 : THREADS <= 256 ? 2 : 1;
  static constexpr int XDBL = ((KXM * T * TPC + 1) & ~1) + 2;   // x slots (+ pad); the staged u table follows
  static constexpr size_t SMEM = sizeof(double) * static_cast<size_t>(XDBL) + Ls::cs_bytes(0);
};

// Per-thread asynchronous copy (cp.async, 8 bytes) of the thread's own x values
// of one parity class of tile b into its shared-memory slots xbuf[j][tid].
template <class Ls>
__device__ __forceinline__ void large_u_xs_issue(const LUParams<Ls>& p, int64_t unit0, int64_t b, int cls,
                                                 double* xbuf, int tid) {
  constexpr int NV = Ls::NV, NW = Ls::NW, NQV = Ls::NQV, S = Ls::S;
  const int np = static_cast<int>(b % (NV * NW));
  const int64_t unit = unit0 + b / (NV * NW);
  const int n1 = np / NW, p1 = np - (np / NW) * NW;
  const int n2 = tid / NW, p2 = tid - (tid / NW) * NW;
  const int qv = Ls::vidx(n1, n2);
  const double* Xu = p.X + (unit - unit0) * Ls::XPU + (static_cast<int64_t>(qv) * NW + p1) * NW + p2;
  auto go = [&](auto parc) {
    constexpr int PAR = decltype(parc)::value;
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
#pragma unroll
      for (int j = 0; j < Ls::ucnt(s, PAR); ++j) {
        const double* src =
            Xu + Ls::xoff(s) + static_cast<int64_t>(Ls::uk0(s, PAR) + 2 * j) * NQV * NW * NW;
        double* dst = xbuf + (Ls::kpo(s, PAR) + j) * NV * NW + tid;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
      }
    });
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (cls == 0)
    go(std::integral_constant<int, 0>{});
  else
    go(std::integral_constant<int, 1>{});
}

template <class Ls, bool ROLL = true>
__global__ void __launch_bounds__(LUXs<Ls>::THREADS, LUXs<Ls>::MINB)
    large_u_xs_kernel(const __grid_constant__ LUParams<Ls> p, int64_t unit0, int64_t ntiles) {
  constexpr int NU = Ls::NU, NV = Ls::NV, NW = Ls::NW, S = Ls::S, T = NV * NW, TPC = LUXs<Ls>::TPC;
  extern __shared__ __align__(128) double xsm[];
  // thread group g of the CTA works on tile it * TPC + g; tid = its fiber (n2, p2)
  const int g = TPC == 1 ? 0 : static_cast<int>(threadIdx.x) / T;
  const int tid = static_cast<int>(threadIdx.x) - g * T;
  double* xbuf = xsm + g * (LUXs<Ls>::KXM * T);
  const double* cu_g = stage_coef<Ls, 0>(p.cu_g, xsm + LUXs<Ls>::XDBL);
  const int64_t nit = (ntiles + TPC - 1) / TPC;
  int64_t it = blockIdx.x;
  if (it >= nit) return;
  int64_t b = it * TPC + g;
  if (b < ntiles)
    large_u_xs_issue<Ls>(p, unit0, b, 0, xbuf, tid);
  else
    asm volatile("cp.async.commit_group;" ::: "memory");
  const int n2 = tid / NW, p2 = tid - (tid / NW) * NW;
#pragma unroll 1
  for (; it < nit; it += gridDim.x) {
    b = it * TPC + g;
    const bool live = b < ntiles;  // the last CTA iteration's spare groups idle (uniform per group)
    const int64_t bb = live ? b : 0;
    const int np = static_cast<int>(bb % (NV * NW));
    const int64_t unit = unit0 + bb / (NV * NW);
    const int n1 = np / NW, p1 = np - (np / NW) * NW;
    const int64_t e = unit / p.P;
    const int pair = static_cast<int>(unit - e * p.P);
    const int gci = pair / p.nc, gcj = pair - gci * p.nc;
    double* out = p.M + e * p.mat_stride + static_cast<int64_t>(gci * p.Nt + n1 * NW + p1) * p.ldM +
                  gcj * p.Nt + n2 * NW + p2;
    const int64_t rowstep = static_cast<int64_t>(NV * NW) * p.ldM;
    auto run = [&](auto parc) {
      constexpr int PAR = decltype(parc)::value;
      constexpr int KX = Ls::KX(PAR);
      double x[KX];
      asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
      for (int j = 0; j < KX; ++j) x[j] = xbuf[j * T + tid];
      // bar.sync completes the shared-memory loads above before the next class's
      // copies are issued into the same slots
      __syncthreads();
      const int64_t bn = b + static_cast<int64_t>(gridDim.x) * TPC;
      if (PAR == 0 && live)
        large_u_xs_issue<Ls>(p, unit0, b, 1, xbuf, tid);
      else if (PAR == 1 && bn < ntiles)
        large_u_xs_issue<Ls>(p, unit0, bn, 0, xbuf, tid);
      else
        asm volatile("cp.async.commit_group;" ::: "memory");
      auto row = [&](auto m1c) {
        constexpr int m1 = decltype(m1c)::value;
        static_for<(Ls::USYM ? m1 : 0), NU>([&](auto m2c) {
          constexpr int m2 = decltype(m2c)::value;
          if constexpr ((m1 + m2) % 2 == PAR) {
            double v = 0.0;
            static_for<0, S>([&](auto sc) {
              constexpr int s = decltype(sc)::value;
              constexpr int ku = Ls::kind(s, 0);
              constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
              constexpr int co = Ls::coff(0, s, m1, m2);
              static_for<0, cnt>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                constexpr int xi = Ls::kpo(s, PAR) + (lo - Ls::uk0(s, PAR)) / 2 + j;
                v = fma(lcoef<Ls, 0>(p.cu, cu_g, co + j), x[xi], v);
              });
            });
            if (live) {
              st_cs(out + m1 * rowstep + m2 * (NV * NW), v);
              if constexpr (Ls::USYM && m2 != m1) st_cs(out + m2 * rowstep + m1 * (NV * NW), v);
            }
          }
        });
      };
      if constexpr (ROLL) {  // runtime row loop: bounded code and scheduling window (C5)
#pragma unroll 1
        for (int m1 = 0; m1 < NU; ++m1)
          static_for<0, NU>([&](auto m1c) {
            if (m1 == decltype(m1c)::value) row(m1c);
          });
      } else {  // every row unrolled: no per-row dispatch branch
        static_for<0, NU>([&](auto m1c) { row(m1c); });
      }
    };
    run(std::integral_constant<int, 0>{});
    run(std::integral_constant<int, 1>{});
  }
}

// BULK mode (u stage with TMA bulk stores): as the XS kernel, but a row of
// outputs (m1 fixed, every m2 of the parity class) goes to shared memory first --
// one STS per output instead of one (USYM: two) 8-byte STG -- and one thread
// writes each (m1, m2) block (the CTA's N_v N_w contiguous doubles of one matrix
// row) with a bulk copy, and again at (m2, m1) for symmetric u kinds.  Three row
// buffers rotate: after committing row r the issuing thread waits until row
// r-1's copies have read shared memory, so one barrier per row orders the reuse
// of row r-2's buffer by row r+1.
template <class Ls>
struct LUBulk {
  static constexpr int T = Ls::NV * Ls::NW;
  static constexpr int SL = (Ls::NU + 1) / 2;  // outputs of one row in one parity class
  static constexpr int NBUF = 3;
  static constexpr size_t SMEM = sizeof(double) * (static_cast<size_t>(LUXs<Ls>::KXM) * T + NBUF * SL * T) + 16;
};

template <class Ls>
__global__ void __launch_bounds__(Ls::NV * Ls::NW, Ls::UMINB)
    large_u_bulk_kernel(const __grid_constant__ LUParams<Ls> p, int64_t unit0, int64_t ntiles) {
  constexpr int NU = Ls::NU, NV = Ls::NV, NW = Ls::NW, S = Ls::S, T = LUBulk<Ls>::T, SL = LUBulk<Ls>::SL;
  static_assert(T % 2 == 0, "bulk-store rows must be 16-byte multiples");
  extern __shared__ __align__(128) double xbuf[];
  double* obuf = xbuf + LUXs<Ls>::KXM * T;  // [NBUF][SL][T]
  const int tid = threadIdx.x;
  int64_t b = blockIdx.x;
  if (b >= ntiles) return;
  const uint64_t policy = evict_first_policy();
  large_u_xs_issue<Ls>(p, unit0, b, 0, xbuf, tid);
  int ring = 0;
#pragma unroll 1
  for (; b < ntiles; b += gridDim.x) {
    const int np = static_cast<int>(b % (NV * NW));
    const int64_t unit = unit0 + b / (NV * NW);
    const int n1 = np / NW, p1 = np - (np / NW) * NW;
    const int64_t e = unit / p.P;
    const int pair = static_cast<int>(unit - e * p.P);
    const int gci = pair / p.nc, gcj = pair - gci * p.nc;
    double* rowbase = p.M + e * p.mat_stride + static_cast<int64_t>(gci * p.Nt + n1 * NW + p1) * p.ldM + gcj * p.Nt;
    const int64_t rowstep = static_cast<int64_t>(T) * p.ldM;
    auto run = [&](auto parc) {
      constexpr int PAR = decltype(parc)::value;
      constexpr int KX = Ls::KX(PAR);
      double x[KX];
      asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
      for (int j = 0; j < KX; ++j) x[j] = xbuf[j * T + tid];
      __syncthreads();
      if (PAR == 0)
        large_u_xs_issue<Ls>(p, unit0, b, 1, xbuf, tid);
      else if (b + gridDim.x < ntiles)
        large_u_xs_issue<Ls>(p, unit0, b + gridDim.x, 0, xbuf, tid);
      auto row = [&](auto m1c) {
        constexpr int m1 = decltype(m1c)::value;
        constexpr int m2s = Ls::USYM ? m1 : 0;
        constexpr int first = m2s + (((m1 + m2s) % 2 == PAR) ? 0 : 1);
        constexpr int cnt_row = first < NU ? (NU - first + 1) / 2 : 0;
        static_assert(cnt_row <= SL, "row slots");
        if constexpr (cnt_row > 0) {
          double* ob = obuf + ring * (SL * T);
          static_for<first, NU>([&](auto m2c) {
            constexpr int m2 = decltype(m2c)::value;
            if constexpr ((m2 - first) % 2 == 0) {
              double v = 0.0;
              static_for<0, S>([&](auto sc) {
                constexpr int s = decltype(sc)::value;
                constexpr int ku = Ls::kind(s, 0);
                constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
                constexpr int co = Ls::coff(0, s, m1, m2);
                static_for<0, cnt>([&](auto jc) {
                  constexpr int j = decltype(jc)::value;
                  constexpr int xi = Ls::kpo(s, PAR) + (lo - Ls::uk0(s, PAR)) / 2 + j;
                  v = fma(lcoef<Ls, 0>(p.cu, p.cu_g, co + j), x[xi], v);
                });
              });
              ob[((m2 - first) / 2) * T + tid] = v;
            }
          });
          fence_proxy_async_smem();  // this thread's outputs visible to the bulk copies
          __syncthreads();
          if (tid == 0) {
            static_for<first, NU>([&](auto m2c) {
              constexpr int m2 = decltype(m2c)::value;
              if constexpr ((m2 - first) % 2 == 0) {
                const double* src = ob + ((m2 - first) / 2) * T;
                bulk_s2g(rowbase + m1 * rowstep + m2 * T, src, T * 8u, policy);
                if constexpr (Ls::USYM && m2 != m1) bulk_s2g(rowbase + m2 * rowstep + m1 * T, src, T * 8u, policy);
              }
            });
            bulk_commit();
            bulk_wait_read<1>();  // row r-1's copies have read their buffer
          }
          ring = ring == LUBulk<Ls>::NBUF - 1 ? 0 : ring + 1;
        }
      };
#pragma unroll 1
      for (int m1 = 0; m1 < NU; ++m1)
        static_for<0, NU>([&](auto m1c) {
          if (m1 == decltype(m1c)::value) row(m1c);
        });
    };
    run(std::integral_constant<int, 0>{});
    run(std::integral_constant<int, 1>{});
  }
  if (tid == 0) bulk_wait<0>();  // every copy complete before the CTA's shared memory goes away
}

// PAIR mode: a thread owns two adjacent fibers (n2, p2), (n2, p2 + 1) of a tile
// (N_w even), so every constant-bank coefficient feeds two DFMAs, x arrives with
// one 16-B shared-memory load per k1 for both fibers, and each output pair (and
// its USYM mirror) leaves with one 16-B streaming store -- half the LDCU and STG
// instructions of the XS kernel per output.  TPC tiles per CTA keep the CTA a
// whole number of warps (c12: 4 tiles x 72 threads; C5: 1 tile x 128).
constexpr int pair_tpc(int th) {
  int t = 1;
  while ((t * th) % 32 != 0 && t < 32) ++t;
  while (t * th < 96 && t < 32) t *= 2;
  return t;
}

template <class Ls>
struct LUPair {
  static constexpr int T = Ls::NV * Ls::NW, TH = T / 2;
  static constexpr int TPC = pair_tpc(TH);
  static constexpr int THREADS = TPC * TH;
  static constexpr int MINB = 65536 / (THREADS * 136) > 0 ? 65536 / (THREADS * 136) : 1;
  static constexpr size_t SMEM = sizeof(double) * static_cast<size_t>(LUXs<Ls>::KXM) * T * TPC + 16;
};

template <class Ls>
__device__ __forceinline__ void large_u_pair_issue(const LUParams<Ls>& p, int64_t unit0, int64_t b, int cls,
                                                   double* xb, int q) {
  constexpr int NV = Ls::NV, NW = Ls::NW, NQV = Ls::NQV, S = Ls::S, T = NV * NW;
  const int np = static_cast<int>(b % T);
  const int64_t unit = unit0 + b / T;
  const int n1 = np / NW, p1 = np - (np / NW) * NW;
  const int c0 = 2 * q;
  const int n2 = c0 / NW, p2 = c0 - (c0 / NW) * NW;
  const double* Xu = p.X + (unit - unit0) * Ls::XPU + (static_cast<int64_t>(Ls::vidx(n1, n2)) * NW + p1) * NW + p2;
  auto go = [&](auto parc) {
    constexpr int PAR = decltype(parc)::value;
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
#pragma unroll
      for (int j = 0; j < Ls::ucnt(s, PAR); ++j) {
        const double* src = Xu + Ls::xoff(s) + static_cast<int64_t>(Ls::uk0(s, PAR) + 2 * j) * NQV * NW * NW;
        double* dst = xb + (Ls::kpo(s, PAR) + j) * T + c0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
      }
    });
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (cls == 0)
    go(std::integral_constant<int, 0>{});
  else
    go(std::integral_constant<int, 1>{});
}

template <class Ls>
__global__ void __launch_bounds__(LUPair<Ls>::THREADS, LUPair<Ls>::MINB)
    large_u_pair_kernel(const __grid_constant__ LUParams<Ls> p, int64_t unit0, int64_t ntiles) {
  constexpr int NU = Ls::NU, NW = Ls::NW, S = Ls::S, T = LUPair<Ls>::T, TH = LUPair<Ls>::TH;
  constexpr int TPC = LUPair<Ls>::TPC;
  static_assert(NW % 2 == 0, "fiber pairs need an even N_w");
  extern __shared__ __align__(128) double xbuf[];
  const int g = threadIdx.x / TH, q = threadIdx.x - (threadIdx.x / TH) * TH;
  double* xb = xbuf + g * (LUXs<Ls>::KXM * T);
  const int64_t nit = (ntiles + TPC - 1) / TPC;  // CTA iterations: TPC consecutive tiles
  int64_t it = blockIdx.x;
  if (it >= nit) return;
  {
    const int64_t b = it * TPC + g;
    if (b < ntiles) large_u_pair_issue<Ls>(p, unit0, b, 0, xb, q);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
#pragma unroll 1
  for (; it < nit; it += gridDim.x) {
    const int64_t b = it * TPC + g;
    const bool live = b < ntiles;
    const int64_t bb = live ? b : 0;
    const int np = static_cast<int>(bb % T);
    const int64_t unit = unit0 + bb / T;
    const int n1 = np / NW, p1 = np - (np / NW) * NW;
    const int64_t e = unit / p.P;
    const int pair = static_cast<int>(unit - e * p.P);
    const int gci = pair / p.nc, gcj = pair - gci * p.nc;
    double* out = p.M + e * p.mat_stride + static_cast<int64_t>(gci * p.Nt + n1 * NW + p1) * p.ldM + gcj * p.Nt +
                  2 * q;
    const int64_t rowstep = static_cast<int64_t>(T) * p.ldM;
    auto run = [&](auto parc) {
      constexpr int PAR = decltype(parc)::value;
      constexpr int KX = Ls::KX(PAR);
      double xa[KX], xc[KX];
      asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
      for (int j = 0; j < KX; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(xb + j * T + 2 * q);
        xa[j] = v.x;
        xc[j] = v.y;
      }
      __syncthreads();
      if (PAR == 0) {
        if (live) large_u_pair_issue<Ls>(p, unit0, b, 1, xb, q);
        else asm volatile("cp.async.commit_group;" ::: "memory");
      } else {
        const int64_t b2 = b + static_cast<int64_t>(gridDim.x) * TPC;
        if (b2 < ntiles) large_u_pair_issue<Ls>(p, unit0, b2, 0, xb, q);
        else asm volatile("cp.async.commit_group;" ::: "memory");
      }
      auto row = [&](auto m1c) {
        constexpr int m1 = decltype(m1c)::value;
        static_for<(Ls::USYM ? m1 : 0), NU>([&](auto m2c) {
          constexpr int m2 = decltype(m2c)::value;
          if constexpr ((m1 + m2) % 2 == PAR) {
            double va = 0.0, vc = 0.0;
            static_for<0, S>([&](auto sc) {
              constexpr int s = decltype(sc)::value;
              constexpr int ku = Ls::kind(s, 0);
              constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
              constexpr int co = Ls::coff(0, s, m1, m2);
              static_for<0, cnt>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                constexpr int xi = Ls::kpo(s, PAR) + (lo - Ls::uk0(s, PAR)) / 2 + j;
                const double c = lcoef<Ls, 0>(p.cu, p.cu_g, co + j);
                va = fma(c, xa[xi], va);
                vc = fma(c, xc[xi], vc);
              });
            });
            if (live) {
              st_cs2(out + m1 * rowstep + m2 * T, va, vc);
              if constexpr (Ls::USYM && m2 != m1) st_cs2(out + m2 * rowstep + m1 * T, va, vc);
            }
          }
        });
      };
#pragma unroll 1
      for (int m1 = 0; m1 < NU; ++m1)
        static_for<0, NU>([&](auto m1c) {
          if (m1 == decltype(m1c)::value) row(m1c);
        });
    };
    run(std::integral_constant<int, 0>{});
    run(std::integral_constant<int, 1>{});
  }
}

template <class Ls>
cudaError_t large_u_dispatch(const LUParams<Ls>& p, int64_t unit0, int64_t cnt, bool ps, int fib, int64_t max_ctas,
                      bool smemc, int num_sms, cudaStream_t st) {
  const int64_t ntiles = cnt * Ls::NV * Ls::NW;
  // max_ctas > 0: persistent grid of that many CTAs; 0: one CTA per tile; < 0:
  // persistent, as many CTAs as are resident (occupancy x SMs) less -1 - max_ctas
  // slots left free for the next chunk's w / v steps
  auto grid_of = [&](int bps) {
    const int64_t cap = max_ctas < 0 ? std::max<int64_t>(num_sms, static_cast<int64_t>(bps) * num_sms + max_ctas + 1) : max_ctas;
    return static_cast<unsigned>(cap > 0 && cap < ntiles ? cap : ntiles);
  };
  unsigned grid = grid_of(2);
  constexpr int T = Ls::NV * Ls::NW;
  constexpr int F2 = Ls::NV % 2 == 0 ? 2 : 1;
  constexpr size_t cs = sizeof(double) * Ls::ctot(0);
  if constexpr (!Ls::u_conforming()) {
#ifndef P2S_LEAN
    if constexpr (Ls::NW % 2 == 0)
    if (p.pair) {
      int bps = 0;
      cudaError_t e = kernel_prepare(large_u_pair_kernel<Ls>, LUPair<Ls>::SMEM, LUPair<Ls>::THREADS, false, &bps);
      if (e != cudaSuccess) return e;
      const int64_t nit = (ntiles + LUPair<Ls>::TPC - 1) / LUPair<Ls>::TPC;
      const int64_t cap = max_ctas < 0 ? std::max<int64_t>(num_sms, static_cast<int64_t>(bps) * num_sms + max_ctas + 1) : max_ctas;
      const unsigned pg = static_cast<unsigned>(cap > 0 && cap < nit ? cap : nit);
      large_u_pair_kernel<Ls><<<pg, LUPair<Ls>::THREADS, LUPair<Ls>::SMEM, st>>>(p, unit0, ntiles);
      return cudaGetLastError();
    }
    if constexpr (Ls::NW % 2 == 0)
    if (p.bulk) {
      int bps = 0;
      cudaError_t e = kernel_prepare(large_u_bulk_kernel<Ls>, LUBulk<Ls>::SMEM, T, false, &bps);
      if (e != cudaSuccess) return e;
      large_u_bulk_kernel<Ls><<<grid_of(bps), T, LUBulk<Ls>::SMEM, st>>>(p, unit0, ntiles);
      return cudaGetLastError();
    }
#endif
#ifdef P2S_LEAN
    if (true) {
#else
    if (ps && fib == 1 && p.xs) {
#endif
      int bps = 0;
#ifndef P2S_LEAN
      if (!p.roll) {
        cudaError_t e = kernel_prepare(large_u_xs_kernel<Ls, false>, LUXs<Ls>::SMEM, LUXs<Ls>::THREADS, false, &bps);
        if (e != cudaSuccess) return e;
        const int64_t nit = (ntiles + LUXs<Ls>::TPC - 1) / LUXs<Ls>::TPC;
        large_u_xs_kernel<Ls, false><<<static_cast<unsigned>(std::min<int64_t>(nit, int64_t(bps) * num_sms)),
                                       LUXs<Ls>::THREADS, LUXs<Ls>::SMEM, st>>>(p, unit0, ntiles);
        return cudaGetLastError();
      }
#endif
      cudaError_t e = kernel_prepare(large_u_xs_kernel<Ls>, LUXs<Ls>::SMEM, LUXs<Ls>::THREADS, false, &bps);
      if (e != cudaSuccess) return e;
      const int64_t nit = (ntiles + LUXs<Ls>::TPC - 1) / LUXs<Ls>::TPC;
      const int64_t cap = max_ctas < 0 ? std::max<int64_t>(num_sms, static_cast<int64_t>(bps) * num_sms + max_ctas + 1) : max_ctas;
      grid = static_cast<unsigned>(cap > 0 && cap < nit ? cap : nit);
      large_u_xs_kernel<Ls><<<grid, LUXs<Ls>::THREADS, LUXs<Ls>::SMEM, st>>>(p, unit0, ntiles);
      return cudaGetLastError();
    }
  }
#ifdef P2S_LEAN  // generated modules: the default u stage only (no measurement variants)
  (void)smemc;
  (void)fib;
  (void)cs;
  (void)F2;
  (void)ps;
  if constexpr (Ls::u_conforming()) {
    using PL = LUPlain<Ls, 1>;
    int bps = 0;
    // an over-size u table is staged in shared memory per (persistent) CTA
    constexpr bool SC = Ls::GS(0);
    constexpr size_t csm = Ls::cs_bytes(0);
    cudaError_t e = kernel_prepare(large_u_kernel<Ls, true, 1, SC>, csm, PL::THREADS, false, &bps);
    if (e != cudaSuccess) return e;
    const int64_t nit = (ntiles + PL::TPC - 1) / PL::TPC;
    const int64_t cap = max_ctas < 0 ? std::max<int64_t>(num_sms, static_cast<int64_t>(bps) * num_sms + max_ctas + 1) : max_ctas;
    large_u_kernel<Ls, true, 1, SC><<<static_cast<unsigned>(cap > 0 && cap < nit ? cap : nit), PL::THREADS, csm, st>>>(
        p, unit0, ntiles);
  }
#else
  if (ps && smemc && p.cu_g) {
    cudaError_t e = kernel_prepare(large_u_kernel<Ls, true, 1, true>, cs, LUPlain<Ls, 1>::THREADS);
    if (e != cudaSuccess) return e;
    large_u_kernel<Ls, true, 1, true><<<grid, LUPlain<Ls, 1>::THREADS, cs, st>>>(p, unit0, ntiles);
  }
  else if (ps && fib == 2)
    large_u_kernel<Ls, true, F2><<<grid, T / F2, 0, st>>>(p, unit0, ntiles);
  else if (ps) {
    constexpr bool SC = Ls::GS(0);
    cudaError_t e = kernel_prepare(large_u_kernel<Ls, true, 1, SC>, Ls::cs_bytes(0), LUPlain<Ls, 1>::THREADS);
    if (e != cudaSuccess) return e;
    large_u_kernel<Ls, true, 1, SC><<<grid, LUPlain<Ls, 1>::THREADS, Ls::cs_bytes(0), st>>>(p, unit0, ntiles);
  } else
    large_u_kernel<Ls, false, 1><<<grid, LUPlain<Ls, 1>::THREADS, 0, st>>>(p, unit0, ntiles);
#endif
  return cudaGetLastError();
}

}  // namespace p2s
