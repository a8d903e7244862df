// p2s_mma.cuh -- stage C (u contraction) as FP64 tensor-core GEMMs
// (mma.sync.aligned.m8n8k4 f64, SASS DMMA; tcgen05 has no f64 kind).
//
//   D[(m1,m2)][fiber] = sum_c A[(m1,m2)][c] B[c][fiber],  c = (term s, k1)
//
// Every product-to-sum band has the parity of m1+m2 (shifted by one for the
// mixed P'P / PP' kinds), so rows and columns split into two parity classes
// and each class is a dense GEMM; 8x4 A tiles that are all zero are skipped
// at compile time.  A = the u-direction coefficients, stored in fragment
// order (32 doubles per 8x4 tile, lane-major: conflict-free shared loads),
// B = the fibers' b_s[k1] straight from the stage-B shared buffer.  Each warp
// owns column tiles of 8 fibers, keeps the accumulators of all row tiles in
// registers and writes its D fragments (2 consecutive fibers = 16 contiguous
// bytes of one matrix row) with streaming 16-B stores.
//
// The banded stage C does sum_k 1 DFMA per in-band term; this form does
// 8x8x4 = 256 FMAs per warp instruction over dense parity tiles (2-2.5x the
// FLOPs for N >= 8) -- it wins where the banded form is issue-bound.
#pragma once

#include <vector>

#include "p2s_kernels.cuh"

namespace p2s {

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Compile-time parity-split layout of stage C (u direction of shape Sh).
template <class Sh>
struct MmaMap {
  static constexpr int NU = Sh::NU, S = Sh::S;
  static constexpr int shift(int s) {
    return (base_kind(Sh::kind(s, 0)) == DP || base_kind(Sh::kind(s, 0)) == PD) ? 1 : 0;
  }
  static constexpr int R(int par) {
    int n = 0;
    for (int a = 0; a < NU; ++a)
      for (int b = 0; b < NU; ++b) n += ((a + b) % 2 == par);
    return n;
  }
  static constexpr int RT(int par) { return (R(par) + 7) / 8; }
  static constexpr int C(int par) {
    int n = 0;
    for (int s = 0; s < S; ++s)
      for (int k = 0; k < Sh::K(s, 0); ++k) n += (k % 2 == (par + shift(s)) % 2);
    return n;
  }
  static constexpr int KT(int par) { return (C(par) + 3) / 4; }
  // i-th row of parity par -> m1 * NU + m2 (row-major order); -1 if padding
  static constexpr int row(int par, int i) {
    int n = 0;
    for (int a = 0; a < NU; ++a)
      for (int b = 0; b < NU; ++b)
        if ((a + b) % 2 == par) {
          if (n == i) return a * NU + b;
          ++n;
        }
    return -1;
  }
  // c-th column of parity par -> s * 64 + k1; -1 if padding
  static constexpr int col(int par, int c) {
    int n = 0;
    for (int s = 0; s < S; ++s)
      for (int k = 0; k < Sh::K(s, 0); ++k)
        if (k % 2 == (par + shift(s)) % 2) {
          if (n == c) return s * 64 + k;
          ++n;
        }
    return -1;
  }
  static constexpr bool in_band(int par, int i, int c) {
    const int rc = row(par, i), cc = col(par, c);
    if (rc < 0 || cc < 0) return false;
    const int a = rc / NU, b = rc % NU, s = cc / 64, k = cc % 64;
    const int kd = Sh::kind(s, 0);
    return band_count(kd, a, b) > 0 && k >= band_lo(kd, a, b) && k <= band_hi(kd, a, b);
  }
  static constexpr bool tile_nz(int par, int rt, int kt) {
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 4; ++c)
        if (in_band(par, rt * 8 + r, kt * 4 + c)) return true;
    return false;
  }
  static constexpr int n_dmma() {
    int n = 0;
    for (int par = 0; par < 2; ++par)
      for (int rt = 0; rt < RT(par); ++rt)
        for (int kt = 0; kt < KT(par); ++kt) n += tile_nz(par, rt, kt);
    return n;
  }
  // fragment-ordered A: tile (par, rt, kt) at 32 * tile index, lane-major
  static constexpr int tile(int par, int rt, int kt) {
    return (par == 0 ? 0 : RT(0) * KT(0)) + rt * KT(par) + kt;
  }
  static constexpr int ATOT = (RT(0) * KT(0) + RT(1) * KT(1)) * 32;
  static constexpr int CMAX = (KT(0) > KT(1) ? KT(0) : KT(1)) * 4;
  // shared footprint (doubles): A fragments + column table (2 ints per entry)
  static constexpr int SMEM_DBL = ATOT + 2 * CMAX;
};

template <class Sh>
constexpr int mma_smem_dbl() {
  if constexpr (Sh::MMA)
    return MmaMap<Sh>::SMEM_DBL;
  else
    return 0;
}

// Host: fragment-ordered A from the dense u tables dense[s] = [NU][NU][K_s].
template <class Sh>
std::vector<double> build_mma_a(const std::vector<double>* const* dense) {
  using Mp = MmaMap<Sh>;
  std::vector<double> A(static_cast<size_t>(Mp::ATOT), 0.0);
  for (int par = 0; par < 2; ++par)
    for (int rt = 0; rt < Mp::RT(par); ++rt)
      for (int kt = 0; kt < Mp::KT(par); ++kt)
        for (int lane = 0; lane < 32; ++lane) {
          const int i = rt * 8 + (lane >> 2), c = kt * 4 + (lane & 3);
          if (!Mp::in_band(par, i, c)) continue;
          const int rc = Mp::row(par, i), cc = Mp::col(par, c);
          const int a = rc / Sh::NU, b = rc % Sh::NU, s = cc / 64, k = cc % 64;
          A[static_cast<size_t>(Mp::tile(par, rt, kt) * 32 + lane)] =
              (*dense[s])[(static_cast<size_t>(a) * Sh::NU + b) * Sh::K(s, 0) + k];
        }
  return A;
}

// Per CTA: A fragments global -> shared, column table: ctab[par*CMAX + c] =
// {B-buffer row offset of (s, k1) for tile slot 0 (-1 for padding),
//  offset step per tile slot (K_s * BSTR)}.
template <class Sh>
__device__ __forceinline__ void mma_setup(const double* __restrict__ gA, double* sA, int2* ctab) {
  using Mp = MmaMap<Sh>;
  for (int i = threadIdx.x; i < Mp::ATOT; i += blockDim.x) sA[i] = __ldg(gA + i);
  for (int i = threadIdx.x; i < 2 * Mp::CMAX; i += blockDim.x) {
    const int par = i / Mp::CMAX, c = i - par * Mp::CMAX;
    const int cc = Mp::col(par, c);
    int2 v = make_int2(-1, 0);
    if (cc >= 0) {
      const int s = cc / 64, k = cc % 64;
      v = make_int2(Sh::boff(s) + k * Sh::BSTR, Sh::K(s, 0) * Sh::BSTR);
    }
    ctab[i] = v;
  }
}

// Stage C of one sub-tile with DMMA.  fiber_off(f) = the fiber's offset inside
// a B-buffer row, out_of(f) = its output pointer for m1 = m2 = 0; fibers are
// numbered ((slot * P1T + p1l) * NV + n2) * NW + p2.
template <class Sh, class FiberOff, class OutOf>
__device__ __forceinline__ void stage_c_mma(const double* sA, const int2* ctab, const double* Bbuf,
                                            int64_t rowstep, int vec2, FiberOff&& fiber_off,
                                            OutOf&& out_of) {
  using Mp = MmaMap<Sh>;
  constexpr int NVW = Sh::NV * Sh::NW;
  constexpr int NF = Sh::T * Sh::P1T * NVW;
  // fiber pairs of a D fragment share one matrix row when rows are even
  constexpr bool PAIRED = NVW % 2 == 0;
  constexpr int CT = (NF + 7) / 8;
  constexpr int NWARP = Sh::THREADS / 32;
  constexpr int RT0 = Mp::RT(0) > 0 ? Mp::RT(0) : 1, RT1 = Mp::RT(1) > 0 ? Mp::RT(1) : 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int lr = lane >> 2, lc = lane & 3;
  for (int ct = warp; ct < CT; ct += NWARP) {
    // B fragment: fiber ct*8 + (lane >> 2), column c = kt*4 + (lane & 3)
    const int fb = (ct * 8 + lr) < NF ? ct * 8 + lr : NF - 1;  // columns past NF: not stored
    const int fslot = fb / (Sh::P1T * NVW);
    const int boff = fiber_off(fb);
    double acc0[RT0][2], acc1[RT1][2];
#pragma unroll
    for (int r = 0; r < RT0; ++r) acc0[r][0] = acc0[r][1] = 0.0;
#pragma unroll
    for (int r = 0; r < RT1; ++r) acc1[r][0] = acc1[r][1] = 0.0;
    static_for<0, 2>([&](auto pc) {
      constexpr int par = decltype(pc)::value;
      static_for<0, Mp::KT(par)>([&](auto kc) {
        constexpr int kt = decltype(kc)::value;
        const int2 cr = ctab[par * Mp::CMAX + kt * 4 + lc];
        const double bv = cr.x >= 0 ? Bbuf[cr.x + fslot * cr.y + boff] : 0.0;
        static_for<0, Mp::RT(par)>([&](auto rc) {
          constexpr int rt = decltype(rc)::value;
          if constexpr (Mp::tile_nz(par, rt, kt)) {
            const double av = sA[Mp::tile(par, rt, kt) * 32 + lane];
            if constexpr (par == 0)
              dmma884(acc0[rt][0], acc0[rt][1], av, bv);
            else
              dmma884(acc1[rt][0], acc1[rt][1], av, bv);
          }
        });
      });
    });
    // D fragment: row (lane >> 2) of each row tile, fibers ct*8 + (lane & 3)*2 + {0, 1}
    const int fd = ct * 8 + lc * 2;
    const bool live0 = fd < NF, live1 = fd + 1 < NF;
    double* o = out_of(live0 ? fd : 0);
    double* o1 = PAIRED ? o + 1 : out_of(live1 ? fd + 1 : 0);
    static_for<0, 2>([&](auto pc) {
      constexpr int par = decltype(pc)::value;
      static_for<0, Mp::RT(par)>([&](auto rc) {
        constexpr int rt = decltype(rc)::value;
        // (m1, m2) of row rt*8 + lr, selected among 8 compile-time rows
        int moff = -1;
        static_for<0, 8>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          constexpr int code = Mp::row(par, rt * 8 + j);
          if (lr == j) moff = code;
        });
        if (moff >= 0) {
          const int m1 = moff / Sh::NU, m2 = moff - (moff / Sh::NU) * Sh::NU;
          const double v0 = par == 0 ? acc0[rt][0] : acc1[rt][0];
          const double v1 = par == 0 ? acc0[rt][1] : acc1[rt][1];
          const int64_t d = m1 * rowstep + m2 * NVW;
          if (PAIRED && NF % 8 == 0 && vec2) {
            __stcs(reinterpret_cast<double2*>(o + d), make_double2(v0, v1));
          } else {
            if (live0) st_cs(o + d, v0);
            if (live1) st_cs(o1 + d, v1);
          }
        }
      });
    });
  }
}

}  // namespace p2s
