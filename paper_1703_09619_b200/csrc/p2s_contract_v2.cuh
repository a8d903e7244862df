// p2s_contract_v2.cuh -- shape-specialised contraction kernel (all orders,
// kinds and tile sizes compile-time).  Used for the registered benchmark
// shapes; the runtime-shaped contract_kernel (p2s_kernels.cuh) covers the
// rest.
//
// Persistent CTAs walk (element, pair) units.  Per unit:
//   I  -> smem            one bulk copy (TMA engine, cp.async.bulk) on an
//                         mbarrier; the next unit's copy is issued as soon as
//                         the last stage A of this unit has read I
//   stage A (v):  thread = fiber (k1, k3) of I_s, Kv values in registers;
//                 A_s[n1][k1][n2][k3] = sum_k2 Cv[n1][n2][k2] I_s[k1][k2][k3]
//                 (all n1 at once when AALL, else per n1 tile)
// and per tile of T n1-values:
//   stage B (w):  thread = (fiber (i, k1, n2) of A_s, p1), Kw values in registers;
//                 B_s[i][k1][p1][n2][p2] = sum_k3 Cw[p1][p2][k3] A_s[n1][k1][n2][k3]
//   stage C (u):  thread = FPT fibers (i, p1, n2, p2) of B over all terms;
//                 M[m1 n1 p1][m2 n2 p2] = sum_s sum_k1 Cu[m1][m2][k1] B_s[..k1..]
// Every output loop is unrolled with compile-time bands, every coefficient is
// a constant-bank operand shared by the thread's FPT fibers, every fiber is
// register resident: one DFMA per product-to-sum term and one store per
// element-matrix entry.
#pragma once

#include "p2s_kernels.cuh"
#include "p2s_mma.cuh"

namespace p2s {

// term kinds of a shape: 3 bits per direction (base kind | conforming bit)
constexpr int enc_kind(int ku, int kv, int kw) { return ku | (kv << 3) | (kw << 6); }

// FLAGS bit 0 (AALL): stage A for all n1 once per unit; bit 1 (ROWLOOP): stage C
// walks the m1 rows in a runtime loop (bounds the scheduler's window and
// register pressure for large N_u); FPT: stage-C fibers per thread.
template <int NU_, int NV_, int NW_, int T_, int P1T_, int PG_, int THREADS_, int MINB_, int FLAGS_,
          int FPT_, int... TK>
struct Shape {
  static constexpr int NU = NU_, NV = NV_, NW = NW_, T = T_, THREADS = THREADS_, MINB = MINB_;
  // SYM (bit 2): v- and w-kinds of every term are symmetric (PP / DD), so
  // A is symmetric in (n1, n2) and B in (p1, p2): both are computed and stored
  // for the upper triangle only, A once per unit.
  static constexpr int SYM = (FLAGS_ >> 2) & 1;
  // PERSIST (bit 3): persistent CTAs loop over units (TMA prefetch of the next
  // unit's moments); otherwise one CTA per unit (no outer loop, so ptxas cannot
  // hoist the per-unit constant-bank loads into registers across units).
  static constexpr int PERSIST = (FLAGS_ >> 3) & 1;
  // MMA (bit 4): stage C as FP64 tensor-core GEMMs (p2s_mma.cuh) instead of
  // the banded register form; FPT is unused then.
  static constexpr int MMA = (FLAGS_ >> 4) & 1;
  static constexpr bool WLAST = false;  // u-last contraction (p2s_contract_wl.cuh: w-last)
  // PAIR (bit 5): a thread's stage-C fibers come in adjacent pairs (f, f+1) of
  // one matrix row, written with one 16-B store (half the store instructions)
  static constexpr int PAIR = (FLAGS_ >> 5) & 1;
  static_assert(!PAIR || (FPT_ % 2 == 0 && (NV_ * NW_) % 2 == 0), "PAIR needs even FPT and rows");
  // PSPLIT (bit 6): stage C runs the (m1, m2) classes of even and odd m1+m2
  // one after the other; a class reads only the k1 of one parity, so the
  // register-resident fiber halves
  static constexpr int PSPLIT = (FLAGS_ >> 6) & 1;
  // USYM: every term's u-kind is symmetric in (m1, m2) (PP / DD, either basis),
  // so Cu[m1][m2] = Cu[m2][m1] and M[m1 n1 p1][m2 n2 p2] = M[m2 n1 p1][m1 n2 p2]:
  // stage C forms m2 >= m1 only and stores each value at both (m1, m2) and
  // (m2, m1) -- (N_u + 1) / (2 N_u) of the DFMAs, same stores.  FLAGS bit 7
  // (NOUSYM) turns it off for A/B measurements.
  static constexpr bool u_symmetric() {
    constexpr int k[] = {TK...};
    for (int s = 0; s < static_cast<int>(sizeof...(TK)); ++s)
      if (base_kind(k[s] & 7) != PP && base_kind(k[s] & 7) != DD) return false;
    return true;
  }
  static constexpr bool USYM = u_symmetric() && !((FLAGS_ >> 7) & 1);
  // QUAD (bit 8): a thread's stage-C fibers come in groups of 4 adjacent columns
  // of one row, written with one 32-B store (st.global.v4.f64, sm_100)
  static constexpr int QUAD = (FLAGS_ >> 8) & 1;
  static_assert(!QUAD || (FPT_ % 4 == 0 && (NV_ * NW_) % 4 == 0 && !PAIR),
                "QUAD needs FPT and rows divisible by 4 (and excludes PAIR)");
  static constexpr int VW = QUAD ? 4 : PAIR ? 2 : 1;  // adjacent fibers per vector store
  // NSYM (bit 9, needs SYM): B is symmetric in (n1, n2), so the stage-C fibers
  // (n1, p1, n2, p2) and (n2, p1, n1, p2) hold the same values and give the same
  // outputs: stage C enumerates only n2 >= n1 (compactly, so whole warps retire
  // early) and also stores each value at row (n2, p1), column (n1, p2); stage B
  // skips n2 < n1.  Together with USYM one computed value lands in up to 4 places.
  static constexpr int NSYM = (FLAGS_ >> 9) & 1;
  static_assert(!NSYM || (SYM && !MMA && !QUAD), "NSYM needs SYM (and the banded stage C)");
  static_assert(!NSYM || !PAIR || NW_ % 2 == 0, "NSYM pairs need an even N_w");
  // AL1 (bit 10): the fused kernel's w-first alpha loads allocate in L1 (A/B only)
  static constexpr int AL1 = (FLAGS_ >> 10) & 1;
  static constexpr int AALL = (FLAGS_ & 1) | SYM, ROWLOOP = (FLAGS_ >> 1) & 1;
  static constexpr int NQV = NV_ * (NV_ + 1) / 2, NQW = NW_ * (NW_ + 1) / 2;
  static constexpr int tri(int a, int b, int n) { return a * n - a * (a - 1) / 2 + (b - a); }
  static constexpr int FPT = FPT_, P1T = P1T_, PG = PG_;
  static constexpr int NPG = 1;
  static_assert(PG_ == NW_ && P1T_ == NW_,
                "stage B items cover every (p1, p2) of the tile (no p1 split / sub-tiles)");
  static constexpr int NP1 = NW_ / P1T_;
  static_assert(NW_ % P1T_ == 0, "p1 tile must divide N_w");
  static constexpr int S = sizeof...(TK);
  static constexpr int NT = NV / T;
  static_assert(NV % T == 0, "n1 tile must divide N_v");
  static constexpr int AT = AALL ? NV : T;  // n1 slots held in the A buffer
  static constexpr int N(int d) { return d == 0 ? NU : d == 1 ? NV : NW; }
  static constexpr int kind(int s, int d) {
    const int k[] = {TK...};
    return (k[s] >> (3 * d)) & 7;
  }
  static constexpr int K(int s, int d) { return kernel_count(kind(s, d), N(d)); }
  static constexpr int KTOT_U() {
    int o = 0;
    for (int s = 0; s < S; ++s) o += K(s, 0);
    return o;
  }
  // u-kernels of term s in parity class par (k1 = k0 + 2 idx, k0 = (par + shift) % 2)
  static constexpr int ushift(int s) {
    return (base_kind(kind(s, 0)) == DP || base_kind(kind(s, 0)) == PD) ? 1 : 0;
  }
  static constexpr bool any_conforming() {
    for (int s = 0; s < S; ++s)
      for (int d = 0; d < 3; ++d)
        if (conforming(kind(s, d))) return true;
    return false;
  }
  static constexpr int uk0(int s, int par) { return (par + ushift(s)) % 2; }
  static constexpr int ucnt(int s, int par) { return (K(s, 0) - uk0(s, par) + 1) / 2; }
  static constexpr int kpo(int s, int par) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += ucnt(i, par);
    return o;
  }
  static constexpr int KTOT_PAR(int par) { return par < 0 ? KTOT_U() : kpo(S, par); }
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
  // fiber counts / prefix sums over terms
  static constexpr int fa(int s) { return K(s, 0) * K(s, 2); }                // stage A fibers
  static constexpr int fb(int s) { return SYM ? T * K(s, 0) * NV : T * K(s, 0) * NV * NPG; }
  static constexpr int fa_off(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += fa(i);
    return o;
  }
  static constexpr int fb_off(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += fb(i);
    return o;
  }
  // smem (doubles)
  static constexpr int BSTR = SYM ? (NV * NQW) | 1 : (P1T * NV * NW) | 1;  // odd k1 stride of B
  static constexpr int aks(int s) { return SYM ? (NQV * K(s, 2)) | 1 : (NV * K(s, 2)) | 1; }
  static constexpr int aoff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += (SYM ? 1 : AT) * K(i, 0) * aks(i);
    return o;
  }
  static constexpr bool sym_ok() {
    for (int s = 0; s < S; ++s)
      for (int d = 1; d < 3; ++d)
        if (base_kind(kind(s, d)) != PP && base_kind(kind(s, d)) != DD) return false;
    return true;
  }
  static_assert(!SYM || (sym_ok() && P1T == NW_), "SYM needs symmetric v/w kinds and P1T == N_w");
  static_assert(!(PSPLIT || MMA) || !any_conforming(),
                "parity-split / DMMA stage C need parity bands (modal basis)");
  static constexpr int boff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += T * K(i, 0) * BSTR;
    return o;
  }
  static constexpr int A_DBL = (aoff(S) + 1) & ~1;
  static constexpr int B_DBL = (boff(S) + 1) & ~1;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(MPP + A_DBL + B_DBL) + 16;
};

// stage-C tensor-core operands in shared memory (MMA shapes)
struct MmaSmem {
  const double* A;
  const int2* ctab;
};

template <class Sh>
__device__ __forceinline__ MmaSmem mma_carve(double* base) {
  if constexpr (Sh::MMA)
    return MmaSmem{base, reinterpret_cast<const int2*>(base + MmaMap<Sh>::ATOT)};
  else
    return MmaSmem{nullptr, nullptr};
}

template <class Sh>
struct V2Params {
  const double* I;
  double* M;
  int64_t ldM, mat_stride;
  int64_t n_units;
  int nc, P, Nt;
  int64_t mom_per_elem;
  const double* amma;  // fragment-ordered stage-C A (MMA shapes), else null
  int vec2;            // widest aligned vector store of M rows: 4 (32 B), 2 (16 B) or 1
  int64_t prefetch_stride;  // non-persistent launch: resident CTAs (next unit on this SM slot)
  double cu[Sh::ctot(0)];
  double cv[Sh::ctot(1)];
  double cw[Sh::ctot(2)];
};

// Stage A for the n1 values N1 .. N1+CNT-1 (compile-time), stored at slots
// SLOT0 .. of the A buffer.  Fibers of all terms in one loop.
template <class Sh, int N1, int CNT, int SLOT0>
__device__ __forceinline__ void v2_stage_a(const V2Params<Sh>& p, const double* Ibuf, double* Abuf) {
  constexpr int NV = Sh::NV;
  constexpr int FTOT = Sh::fa_off(Sh::S);
  for_items<FTOT, Sh::THREADS>([&](int f) {
    static_for<0, Sh::S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      if (f >= Sh::fa_off(s) && f < Sh::fa_off(s) + Sh::fa(s)) {
        constexpr int Ku = Sh::K(s, 0), Kv = Sh::K(s, 1), Kw = Sh::K(s, 2);
        constexpr int kv = Sh::kind(s, 1);
        const int g = f - Sh::fa_off(s);
        const int k1 = g / Kw, k3 = g - (g / Kw) * Kw;
        const double* Is = Ibuf + Sh::moff(s);
        double x[Kv];
#pragma unroll
        for (int k2 = 0; k2 < Kv; ++k2) x[k2] = Is[(k1 * Kv + k2) * Kw + k3];
        static_for<0, CNT>([&](auto ic) {
          constexpr int i = decltype(ic)::value;
          constexpr int n1 = N1 + i;
          double* As = Abuf + Sh::aoff(s) + (SLOT0 + i) * (Ku * Sh::aks(s));
          static_for<0, NV>([&](auto n2c) {
            constexpr int n2 = decltype(n2c)::value;
            constexpr int lo = band_lo(kv, n1, n2), cnt = band_count(kv, n1, n2);
            constexpr int co = Sh::coff(1, s, n1, n2);
            double v = 0.0;
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              v = fma(p.cv[co + j], x[lo + band_step(kv, n1, n2) * j], v);
            });
            As[k1 * Sh::aks(s) + n2 * Kw + k3] = v;
          });
        });
      }
    });
  });
}

// Stage B for the current tile: item = (s, (i*Ku + k1)*NV + n2, p1) with p1
// slowest inside a term, so p1 (and its compile-time band) is warp-uniform
// except at boundaries.
template <class Sh>
__device__ __forceinline__ void v2_stage_b(const V2Params<Sh>& p, const double* Abuf, double* Bbuf,
                                           int aslot0, int p1base) {
  constexpr int NV = Sh::NV, NW = Sh::NW, T = Sh::T;
  constexpr int FTOT = Sh::fb_off(Sh::S);
  for_items<FTOT, Sh::THREADS>([&](int f) {
    static_for<0, Sh::S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      if (f >= Sh::fb_off(s) && f < Sh::fb_off(s) + Sh::fb(s)) {
        constexpr int Ku = Sh::K(s, 0), Kw = Sh::K(s, 2);
        constexpr int kw = Sh::kind(s, 2);
        constexpr int NFIB = T * Ku * NV;
        const int g = f - Sh::fb_off(s);
        const int pg = g / NFIB;
        const int fib = g - pg * NFIB;          // n2*(T*Ku) + (i*Ku + k1): k1 fastest
        const int n2 = fib / (T * Ku);
        const int ik = fib - n2 * (T * Ku);     // i*Ku + k1
        const int i = ik / Ku, k1 = ik - i * Ku;
        const double* src =
            Abuf + Sh::aoff(s) + ((aslot0 + i) * Ku + k1) * Sh::aks(s) + n2 * Kw;
        double y[Kw];
#pragma unroll
        for (int k3 = 0; k3 < Kw; ++k3) y[k3] = src[k3];
        double* dst = Bbuf + Sh::boff(s) + ik * Sh::BSTR + n2 * NW;
        auto emit = [&](auto p1c, int p1l) {
          constexpr int pp1 = decltype(p1c)::value;
          static_for<0, NW>([&](auto p2c) {
            constexpr int p2 = decltype(p2c)::value;
            constexpr int lo = band_lo(kw, pp1, p2), cnt = band_count(kw, pp1, p2);
            constexpr int co = Sh::coff(2, s, pp1, p2);
            double v = 0.0;
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              v = fma(p.cw[co + j], y[lo + band_step(kw, pp1, p2) * j], v);
            });
            dst[p1l * NV * NW + p2] = v;
          });
        };
        static_for<0, NW>([&](auto p1c) { emit(p1c, decltype(p1c)::value); });
      }
    });
  });
}

// SYM stage A: A_s[k1][tri(n1, n2)][k3] for n1 <= n2, all n1, once per unit.
template <class Sh>
__device__ __forceinline__ void v2_stage_a_sym(const V2Params<Sh>& p, const double* Ibuf, double* Abuf) {
  constexpr int NV = Sh::NV;
  constexpr int FTOT = Sh::fa_off(Sh::S);
  for_items<FTOT, Sh::THREADS>([&](int f) {
    static_for<0, Sh::S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      if (f >= Sh::fa_off(s) && f < Sh::fa_off(s) + Sh::fa(s)) {
        constexpr int Kv = Sh::K(s, 1), Kw = Sh::K(s, 2);
        constexpr int kv = Sh::kind(s, 1);
        const int g = f - Sh::fa_off(s);
        const int k1 = g / Kw, k3 = g - (g / Kw) * Kw;
        const double* Is = Ibuf + Sh::moff(s);
        double x[Kv];
#pragma unroll
        for (int k2 = 0; k2 < Kv; ++k2) x[k2] = Is[(k1 * Kv + k2) * Kw + k3];
        double* As = Abuf + Sh::aoff(s) + k1 * Sh::aks(s) + k3;
        static_for<0, NV>([&](auto n1c) {
          constexpr int n1 = decltype(n1c)::value;
          static_for<n1, NV>([&](auto n2c) {
            constexpr int n2 = decltype(n2c)::value;
            constexpr int lo = band_lo(kv, n1, n2), cnt = band_count(kv, n1, n2);
            constexpr int co = Sh::coff(1, s, n1, n2);
            double v = 0.0;
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              v = fma(p.cv[co + j], x[lo + band_step(kv, n1, n2) * j], v);
            });
            As[Sh::tri(n1, n2, NV) * Kw] = v;
          });
        });
      }
    });
  });
}

// SYM stage B: item (s, n2, i*Ku + k1) with k1 fastest (conflict-free odd
// stride); B_s[i*Ku + k1][n2][tri(p1, p2)] for p1 <= p2.
template <class Sh>
__device__ __forceinline__ void v2_stage_b_sym(const V2Params<Sh>& p, const double* Abuf, double* Bbuf,
                                               int n1base) {
  constexpr int NV = Sh::NV, NW = Sh::NW, T = Sh::T, NQW = Sh::NQW;
  constexpr int FTOT = Sh::fb_off(Sh::S);
  for_items<FTOT, Sh::THREADS>([&](int f) {
    static_for<0, Sh::S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      if (f >= Sh::fb_off(s) && f < Sh::fb_off(s) + Sh::fb(s)) {
        constexpr int Ku = Sh::K(s, 0), Kw = Sh::K(s, 2);
        constexpr int kw = Sh::kind(s, 2);
        const int g = f - Sh::fb_off(s);
        const int n2 = g / (T * Ku);
        const int ik = g - n2 * (T * Ku);
        const int i = ik / Ku, k1 = ik - i * Ku;
        const int n1 = n1base + i;
        if (Sh::NSYM && n2 < n1) return;  // stage C reads only n2 >= n1
        const int a = n1 < n2 ? n1 : n2, b = n1 < n2 ? n2 : n1;
        const double* src = Abuf + Sh::aoff(s) + k1 * Sh::aks(s) + Sh::tri(a, b, NV) * Kw;
        double y[Kw];
#pragma unroll
        for (int k3 = 0; k3 < Kw; ++k3) y[k3] = src[k3];
        double* dst = Bbuf + Sh::boff(s) + ik * Sh::BSTR + n2 * NQW;
        static_for<0, NW>([&](auto p1c) {
          constexpr int p1 = decltype(p1c)::value;
          static_for<p1, NW>([&](auto p2c) {
            constexpr int p2 = decltype(p2c)::value;
            constexpr int lo = band_lo(kw, p1, p2), cnt = band_count(kw, p1, p2);
            constexpr int co = Sh::coff(2, s, p1, p2);
            double v = 0.0;
            static_for<0, cnt>([&](auto jc) {
              constexpr int j = decltype(jc)::value;
              v = fma(p.cw[co + j], y[lo + band_step(kw, p1, p2) * j], v);
            });
            dst[Sh::tri(p1, p2, NW)] = v;
          });
        });
      }
    });
  });
}

template <class Sh, int PAR = -1>
__device__ __forceinline__ void v2_load_fiber(const double* Bbuf, int i, int p1l, int r,
                                              double (&b)[Sh::KTOT_PAR(PAR)]) {
  constexpr int NV = Sh::NV, NW = Sh::NW;
  int off;
  if constexpr (Sh::SYM) {
    const int n2 = r / NW, p2 = r - n2 * NW;   // p1l == p1 (P1T == NW)
    const int a = p1l < p2 ? p1l : p2, c = p1l < p2 ? p2 : p1l;
    off = n2 * Sh::NQW + Sh::tri(a, c, NW);
  } else {
    off = p1l * NV * NW + r;
  }
  static_for<0, Sh::S>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    constexpr int Ku = Sh::K(s, 0);
    const double* src = Bbuf + Sh::boff(s) + (i * Ku) * Sh::BSTR + off;
    if constexpr (PAR < 0) {
#pragma unroll
      for (int k1 = 0; k1 < Ku; ++k1) b[Sh::kuoff(s) + k1] = src[k1 * Sh::BSTR];
    } else {
      constexpr int k0 = Sh::uk0(s, PAR);
#pragma unroll
      for (int j = 0; j < Sh::ucnt(s, PAR); ++j) b[Sh::kpo(s, PAR) + j] = src[(k0 + 2 * j) * Sh::BSTR];
    }
  });
}

// Contraction of one (element, pair) unit whose moments are in Ibuf.
// after_a() runs once the last stage A has read Ibuf (all threads, after a
// barrier), e.g. to start the next unit's bulk copy into Ibuf.
template <class Sh, class AfterA>
__device__ __forceinline__ void v2_unit(const V2Params<Sh>& p, const double* Ibuf, double* Abuf,
                                        double* Bbuf, double* Mbase, AfterA&& after_a,
                                        MmaSmem mm = MmaSmem{nullptr, nullptr}) {
  constexpr int S = Sh::S, NU = Sh::NU, NV = Sh::NV, NW = Sh::NW, T = Sh::T, FPT = Sh::FPT;
  if constexpr (Sh::SYM) {
    v2_stage_a_sym<Sh>(p, Ibuf, Abuf);
    __syncthreads();
    after_a();
  } else if constexpr (Sh::AALL) {
    v2_stage_a<Sh, 0, NV, 0>(p, Ibuf, Abuf);
    __syncthreads();
    after_a();
  }
  for (int t = 0; t < Sh::NT; ++t) {
    if constexpr (!Sh::AALL) {
      static_for<0, Sh::NT>([&](auto tc) {
        constexpr int tt = decltype(tc)::value;
        if (t == tt) v2_stage_a<Sh, tt * T, T, 0>(p, Ibuf, Abuf);
      });
      __syncthreads();
      if (t == Sh::NT - 1) after_a();
    }
    for (int pt = 0; pt < Sh::NP1; ++pt) {
      if constexpr (Sh::SYM)
        v2_stage_b_sym<Sh>(p, Abuf, Bbuf, t * T);
      else
        v2_stage_b<Sh>(p, Abuf, Bbuf, Sh::AALL ? t * T : 0, pt * Sh::P1T);
      __syncthreads();
      // ---- stage C
      constexpr int NF = T * Sh::P1T * NV * NW;  // fibers of the sub-tile
      // thread items: FPT single fibers, or FPT/2 adjacent pairs (PAIR)
      constexpr int VW = Sh::VW;
      constexpr int NFT = (NF / VW + FPT / VW - 1) / (FPT / VW);
      const int64_t rowstep = static_cast<int64_t>(NV * NW) * p.ldM;
      if constexpr (Sh::MMA) {
        stage_c_mma<Sh>(
            mm.A, mm.ctab, Bbuf, rowstep, p.vec2,
            [&](int f) {
              const int r = f % (NV * NW);
              const int p1l = (f / (NV * NW)) % Sh::P1T;
              if constexpr (Sh::SYM) {
                const int n2 = r / NW, p2 = r - n2 * NW;
                const int a = p1l < p2 ? p1l : p2, c = p1l < p2 ? p2 : p1l;
                return n2 * Sh::NQW + Sh::tri(a, c, NW);
              } else {
                return p1l * NV * NW + r;
              }
            },
            [&](int f) {
              const int r = f % (NV * NW);
              const int ip = f / (NV * NW);
              const int p1l = ip % Sh::P1T, i = ip / Sh::P1T;
              const int n1 = t * T + i, p1 = pt * Sh::P1T + p1l;
              return Mbase + static_cast<int64_t>(n1 * NW + p1) * p.ldM + r;
            });
      } else {
      // NSYM: the tile's canonical (n2 >= n1) fibers, i-major blocks of
      // P1T * (NV - n1) * NW; nf / nft are this tile's fiber / thread-item counts
      int nf = NF;
      if constexpr (Sh::NSYM) {
        nf = 0;
#pragma unroll
        for (int i = 0; i < T; ++i) nf += Sh::P1T * (NV - (t * T + i)) * NW;
      }
      const int nft = Sh::NSYM ? (nf / VW + FPT / VW - 1) / (FPT / VW) : NFT;
      auto stage_c = [&](auto parc) {
      constexpr int PAR = decltype(parc)::value;  // -1: all (m1, m2) at once
      for_items<NFT, Sh::THREADS>([&](int f0) {
        if (Sh::NSYM && f0 >= nft) return;
        double b[FPT][Sh::KTOT_PAR(PAR)];
        double* out[FPT];
        double* outn[Sh::NSYM ? FPT : 1];  // NSYM mirror (row n2, column n1); nullptr when n2 == n1
        (void)outn;
        bool live[FPT];
#pragma unroll
        for (int q = 0; q < FPT; ++q) {
          // f = ((i*P1T + p1l)*NV + n2)*NW + p2  (NSYM: compact canonical index)
          const int f = VW * (f0 + (q / VW) * nft) + (q % VW);
          live[q] = f < nf;
          const int fs = live[q] ? f : 0;
          int r, p1l, i;
          if constexpr (Sh::NSYM) {
            int rem = fs;
            i = 0;
#pragma unroll
            for (int ii = 0; ii < T - 1; ++ii) {
              const int c = Sh::P1T * (NV - (t * T + ii)) * NW;
              if (i == ii && rem >= c) {
                rem -= c;
                i = ii + 1;
              }
            }
            const int w = (NV - (t * T + i)) * NW;
            p1l = rem / w;
            r = (t * T + i) * NW + (rem - p1l * w);  // n2 * NW + p2 with n2 >= n1
          } else {
            r = fs % (NV * NW);
            const int ip = fs / (NV * NW);
            p1l = ip % Sh::P1T;
            i = ip / Sh::P1T;
          }
          const int n1 = t * T + i, p1 = pt * Sh::P1T + p1l;
          v2_load_fiber<Sh, PAR>(Bbuf, i, p1l, r, b[q]);
          out[q] = Mbase + static_cast<int64_t>(n1 * NW + p1) * p.ldM + r;
          if constexpr (Sh::NSYM) {
            const int n2 = r / NW, p2 = r - n2 * NW;
            outn[q] = n2 > n1 ? Mbase + static_cast<int64_t>(n2 * NW + p1) * p.ldM + n1 * NW + p2 : nullptr;
          }
        }
        auto row = [&](auto m1c) {
          constexpr int m1 = decltype(m1c)::value;
          static_for<(Sh::USYM ? m1 : 0), NU>([&](auto m2c) {
            constexpr int m2 = decltype(m2c)::value;
            if constexpr (PAR < 0 || (m1 + m2) % 2 == PAR) {
            constexpr bool mirror = Sh::USYM && m2 != m1;  // also store at (m2, m1)
            double v[FPT];
#pragma unroll
            for (int q = 0; q < FPT; ++q) v[q] = 0.0;
            static_for<0, S>([&](auto sc) {
              constexpr int s = decltype(sc)::value;
              constexpr int ku = Sh::kind(s, 0);
              constexpr int lo = band_lo(ku, m1, m2), cnt = band_count(ku, m1, m2);
              constexpr int co = Sh::coff(0, s, m1, m2);
              constexpr int ko = Sh::kuoff(s);
              static_for<0, cnt>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                const double c = p.cu[co + j];
                constexpr int bi =
                    PAR < 0 ? ko + lo + band_step(ku, m1, m2) * j
                            : Sh::kpo(s, PAR) + (lo - Sh::uk0(s, PAR)) / 2 + j;
#pragma unroll
                for (int q = 0; q < FPT; ++q) v[q] = fma(c, b[q][bi], v[q]);
              });
            });
            if constexpr (Sh::QUAD) {
#pragma unroll
              for (int q = 0; q < FPT; q += 4) {
                double* d = out[q] + m1 * rowstep + m2 * (NV * NW);
                double* dm = out[q] + m2 * rowstep + m1 * (NV * NW);
                if (live[q]) {  // NF % 4 == 0: a group is live as a whole
                  st_cs_n(d, &v[q], p.vec2);
                  if constexpr (mirror) st_cs_n(dm, &v[q], p.vec2);
                }
              }
            } else if constexpr (Sh::PAIR) {
#pragma unroll
              for (int q = 0; q < FPT; q += 2) {
                // the pair shares n2 (even N_w, pairs start at even p2): one mirror row
                double* bases[2] = {out[q], nullptr};
                if constexpr (Sh::NSYM) bases[1] = outn[q];
#pragma unroll
                for (int h = 0; h < (Sh::NSYM ? 2 : 1); ++h) {
                  if (bases[h] == nullptr) continue;
                  double* d = bases[h] + m1 * rowstep + m2 * (NV * NW);
                  double* dm = bases[h] + m2 * rowstep + m1 * (NV * NW);
                  if (p.vec2) {
                    if (live[q]) {
                      st_cs2(d, v[q], v[q + 1]);
                      if constexpr (mirror) st_cs2(dm, v[q], v[q + 1]);
                    }
                  } else {
                    if (live[q]) st_cs(d, v[q]);
                    if (live[q + 1]) st_cs(d + 1, v[q + 1]);
                    if constexpr (mirror) {
                      if (live[q]) st_cs(dm, v[q]);
                      if (live[q + 1]) st_cs(dm + 1, v[q + 1]);
                    }
                  }
                }
              }
            } else {
#pragma unroll
              for (int q = 0; q < FPT; ++q)
                if (live[q]) {
                  st_cs(out[q] + m1 * rowstep + m2 * (NV * NW), v[q]);
                  if constexpr (mirror) st_cs(out[q] + m2 * rowstep + m1 * (NV * NW), v[q]);
                  if constexpr (Sh::NSYM) {
                    if (outn[q] != nullptr) {
                      st_cs(outn[q] + m1 * rowstep + m2 * (NV * NW), v[q]);
                      if constexpr (mirror) st_cs(outn[q] + m2 * rowstep + m1 * (NV * NW), v[q]);
                    }
                  }
                }
            }
            }  // parity class
          });
        };
        if constexpr (Sh::ROWLOOP) {
#pragma unroll 1
          for (int m1 = 0; m1 < NU; ++m1)
            static_for<0, NU>([&](auto m1c) {
              if (m1 == decltype(m1c)::value) row(m1c);
            });
        } else {
          static_for<0, NU>([&](auto m1c) { row(m1c); });
        }
      });
      };
      if constexpr (Sh::PSPLIT) {
        stage_c(std::integral_constant<int, 0>{});
        stage_c(std::integral_constant<int, 1>{});
      } else {
        stage_c(std::integral_constant<int, -1>{});
      }
      }  // banded stage C
      __syncthreads();
    }  // p1 sub-tiles
  }
}

template <class Sh>
constexpr size_t v2_smem() {
  return Sh::SMEM + sizeof(double) * static_cast<size_t>(mma_smem_dbl<Sh>());
}

template <class Sh>
__global__ void __launch_bounds__(Sh::THREADS, Sh::MINB)
    contract_v2_kernel(const __grid_constant__ V2Params<Sh> p) {
  extern __shared__ __align__(16) double sm[];
  double* Ibuf = sm;
  double* Abuf = Ibuf + Sh::MPP;
  double* Bbuf = Abuf + Sh::A_DBL;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bbuf + Sh::B_DBL);
  const int tid = threadIdx.x;
  constexpr uint32_t kIBytes = Sh::MPP * 8u;
  const MmaSmem mm = mma_carve<Sh>(Bbuf + Sh::B_DBL + 2);
  if constexpr (Sh::MMA)
    mma_setup<Sh>(p.amma, const_cast<double*>(mm.A), const_cast<int2*>(mm.ctab));

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
  auto do_unit = [&](auto next_copy) {
    const int64_t e = unit / p.P;
    const int pair = static_cast<int>(unit - e * p.P);
    const int gci = pair / p.nc, gcj = pair - gci * p.nc;
    mbar_wait_parity(bar, phase);
    phase ^= 1u;
    double* Mbase = p.M + e * p.mat_stride + static_cast<int64_t>(gci * p.Nt) * p.ldM + gcj * p.Nt;
    v2_unit<Sh>(p, Ibuf, Abuf, Bbuf, Mbase, next_copy, mm);
  };
  if constexpr (Sh::PERSIST) {
    for (; unit < p.n_units; unit += gridDim.x)
      do_unit([&]() {
        if (tid == 0) {
          const int64_t nxt = unit + gridDim.x;
          if (nxt < p.n_units) {
            const int64_t e2 = nxt / p.P;
            const int pair2 = static_cast<int>(nxt - e2 * p.P);
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bar, kIBytes);
            bulk_g2s(Ibuf, p.I + e2 * p.mom_per_elem + pair2 * Sh::MPP, kIBytes, bar);
          }
        }
      });
  } else {
    if (unit < p.n_units) {
      // warm L2 with the moments of the unit that takes this SM slot next
      const int64_t nxt = unit + p.prefetch_stride;
      if (tid == 0 && p.prefetch_stride > 0 && nxt < p.n_units) {
        const int64_t e2 = nxt / p.P;
        const int pair2 = static_cast<int>(nxt - e2 * p.P);
        prefetch_l2(p.I + e2 * p.mom_per_elem + pair2 * Sh::MPP, kIBytes);
      }
      do_unit([]() {});
    }
  }
}

}  // namespace p2s
