// p2s_moments_v2.cuh -- shape-specialised moment kernel.
//
// I_s[k1][k2][k3] = sum_q alpha_s(q) phi_k1(u_q1) phi_k2(v_q2) phi_k3(w_q3),
// phi_k(x_q) = w_q P_k(x_q), by three 1-D passes.  The Gauss-Legendre rule is
// symmetric (x_{n-1-h} = -x_h, w_{n-1-h} = w_h) and P_k(-x) = (-1)^k P_k(x),
// so every pass first folds a fiber into its even part a_h + a_{n-1-h} and odd
// part a_h - a_{n-1-h}; even k then contract the even part and odd k the odd
// part over half the nodes: half the FMAs of the plain sum factorisation.
// Sizes are compile-time, tables are constant-bank operands, fibers live in
// registers:
//   pass u: thread = alpha row (q_w, q_v), 16-B global loads    -> T1[k1][q_w][q_v]
//   pass v: thread = fiber (k1, q_w) of T1                      -> T2[k1 k2][q_w]
//   pass w: thread = fiber (k1, k2) of T2                       -> I (global or smem)
#pragma once

#include "p2s_kernels.cuh"

namespace p2s {

template <int NU_, int NV_, int NW_, int QU_, int QV_, int QW_, int THREADS_, int... TK>
struct MShape {
  static constexpr int NU = NU_, NV = NV_, NW = NW_, THREADS = THREADS_;
  static constexpr int S = sizeof...(TK);
  static constexpr int N(int d) { return d == 0 ? NU : d == 1 ? NV : NW; }
  static constexpr int Q(int d) { return d == 0 ? QU_ : d == 1 ? QV_ : QW_; }
  static constexpr int H(int d) { return (Q(d) + 1) / 2; }  // half rule incl. centre
  static constexpr int kind(int s, int d) {
    const int k[] = {TK...};
    return (k[s] >> (3 * d)) & 7;
  }
  static constexpr int K(int s, int d) { return kernel_count(kind(s, d), N(d)); }
  static constexpr int toff(int s, int d) {  // half-table offsets in the param block
    int o = 0;
    for (int t = 0; t <= s; ++t)
      for (int e = 0; e < 3; ++e) {
        if (t == s && e == d) return o;
        o += K(t, e) * H(e);
      }
    return o;
  }
  static constexpr int TTOT = toff(S - 1, 2) + K(S - 1, 2) * H(2);
  // shared per-direction half tables (rows 0..KMAX(d)-1) used by moments_all_terms
  static constexpr int KMAX(int d) {
    int m = 0;
    for (int s = 0; s < S; ++s) m = K(s, d) > m ? K(s, d) : m;
    return m;
  }
  static constexpr int ttoff(int d) {
    int o = TTOT;  // appended after the per-term tables
    for (int e = 0; e < d; ++e) o += KMAX(e) * H(e);
    return o;
  }
  static constexpr int TALL = ttoff(3);
  static constexpr int t1off(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0) * Q(2) * (Q(1) | 1);
    return o;
  }
  static constexpr int t2off(int s) {
    int o = t1off(S);
    for (int i = 0; i < s; ++i) o += K(i, 0) * K(i, 1) * (Q(2) | 1);
    return o;
  }
  // w-first pass order (moments_all_terms_wfirst)
  static constexpr int w1off(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 2) * Q(1) * (Q(0) | 1);
    return o;
  }
  static constexpr int w2off(int s) {
    int o = w1off(S);
    for (int i = 0; i < s; ++i) o += K(i, 2) * K(i, 1) * (Q(0) | 1);
    return o;
  }
  // pass order: w first when it is the direction with the fewest kernel polynomials
  static constexpr bool WFIRST = KMAX(2) < KMAX(0);
  static constexpr int scratch_all_dbl() {
    return WFIRST ? (w2off(S) + 1) & ~1 : (t2off(S) + 1) & ~1;
  }
  static constexpr int moff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += K(i, 0) * K(i, 1) * K(i, 2);
    return o;
  }
  static constexpr int MPP = (moff(S) + 3) & ~3;
  static constexpr int S2 = Q(1) | 1, S3 = Q(2) | 1;
  static constexpr int t1_dbl(int s) { return K(s, 0) * Q(2) * S2; }
  static constexpr int t2_dbl(int s) { return K(s, 0) * K(s, 1) * S3; }
  static constexpr int scratch_dbl() {
    int m = 0;
    for (int s = 0; s < S; ++s) {
      const int v = t1_dbl(s) + t2_dbl(s);
      m = v > m ? v : m;
    }
    return (m + 1) & ~1;
  }
  static constexpr size_t SMEM = sizeof(double) * (size_t)scratch_dbl();
};

template <class Ms>
struct MV2Params {
  const double* alpha;
  double* I;
  int64_t n_units;     // E * P * S
  int P;
  int64_t mom_per_elem;
  double tab[Ms::TALL];  // per (s, d): [K][H] = w_h P_k(x_h), h < H (x_h <= 0); then shared
                         // per-direction tables [KMAX][H]
};

// One alpha row (QU contiguous doubles) into registers with the widest loads the
// row length allows: 32-B (LDG.256, sm_100) when QU % 4 == 0 -- every sector is
// touched by exactly one load -- else 16-B.  Rows start at multiples of QU
// doubles from a 32-B aligned slab.
template <int QU>
__device__ __forceinline__ void load_row(const double* __restrict__ row, double (&x)[QU]) {
  if constexpr (QU % 4 == 0) {
#pragma unroll
    for (int q = 0; q < QU / 4; ++q) ld_nc4(row + 4 * q, x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
  } else if constexpr (QU % 2 == 0) {
#pragma unroll
    for (int q = 0; q < QU / 2; ++q) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(row) + q);
      x[2 * q] = v.x;
      x[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < QU; ++q) x[q] = __ldg(row + q);
  }
}

// Even/odd folded contraction of one register fiber a[Q] against the half
// table tb[K][H]; out(k, value) receives each result.
template <int Q, int K, class Out>
__device__ __forceinline__ void fold_contract(const double (&a)[Q], const double* tb, Out&& out) {
  constexpr int Hf = Q / 2;
  constexpr int H = (Q + 1) / 2;
  double ev[Hf > 0 ? Hf : 1], od[Hf > 0 ? Hf : 1];
#pragma unroll
  for (int h = 0; h < Hf; ++h) {
    ev[h] = a[h] + a[Q - 1 - h];
    od[h] = a[h] - a[Q - 1 - h];
  }
  static_for<0, K>([&](auto kc) {
    constexpr int k = decltype(kc)::value;
    double v = 0.0;
    if constexpr ((k & 1) == 0) {
#pragma unroll
      for (int h = 0; h < Hf; ++h) v = fma(tb[k * H + h], ev[h], v);
      if constexpr (Q & 1) v = fma(tb[k * H + Hf], a[Hf], v);
    } else {
#pragma unroll
      for (int h = 0; h < Hf; ++h) v = fma(tb[k * H + h], od[h], v);
    }
    out(k, v);
  });
}

// Moments of one (alpha slab, term) into Iout (global or shared), using the
// smem scratch T1/T2.  All threads of the CTA participate; ends with a
// __syncthreads().
template <class Ms, int s, int NTHR = Ms::THREADS>
__device__ __forceinline__ void moments_unit(const double* __restrict__ a, const double* tab,
                                             double* scratch, double* Iout) {
  constexpr int QU = Ms::Q(0), QV = Ms::Q(1), QW = Ms::Q(2);
  constexpr int KU = Ms::K(s, 0), KV = Ms::K(s, 1), KW = Ms::K(s, 2);
  constexpr int S2 = Ms::S2, S3 = Ms::S3;
  double* T1 = scratch;                    // [KU][QW][S2]
  double* T2 = scratch + Ms::t1_dbl(s);    // [KU*KV][S3]
  const double* tu = tab + Ms::toff(s, 0);
  const double* tv = tab + Ms::toff(s, 1);
  const double* tw = tab + Ms::toff(s, 2);

  for_items<QW * QV, NTHR>([&](int r) {
    const int q3 = r / QV, q2 = r - (r / QV) * QV;
    double x[QU];
    load_row<QU>(a + static_cast<int64_t>(r) * QU, x);
    fold_contract<QU, KU>(x, tu, [&](int k, double v) { T1[(k * QW + q3) * S2 + q2] = v; });
  });
  __syncthreads();
  for_items<KU * QW, NTHR>([&](int r) {
    const int k1 = r / QW, q3 = r - (r / QW) * QW;
    const double* src = T1 + (k1 * QW + q3) * S2;
    double x[QV];
#pragma unroll
    for (int q = 0; q < QV; ++q) x[q] = src[q];
    fold_contract<QV, KV>(x, tv, [&](int k, double v) { T2[(k1 * KV + k) * S3 + q3] = v; });
  });
  __syncthreads();
  // pass w: the thread's KW outputs are one contiguous run of I; they go to shared
  // memory first (T1 is free after pass v) and leave in one coalesced sweep --
  // unless the I tile is larger than T1 (fewer quadrature points than kernel
  // polynomials along w), then straight to Iout
  constexpr bool kStage = KU * KV * KW <= KU * QW * S2;
  for_items<KU * KV, NTHR>([&](int r) {
    const double* src = T2 + r * S3;
    double x[QW];
#pragma unroll
    for (int q = 0; q < QW; ++q) x[q] = src[q];
    fold_contract<QW, KW>(x, tw, [&](int k, double v) {
      if constexpr (kStage)
        T1[r * KW + k] = v;
      else
        Iout[r * KW + k] = v;
    });
  });
  __syncthreads();
  if constexpr (kStage) {
    for (int i = threadIdx.x; i < KU * KV * KW; i += NTHR) Iout[i] = T1[i];
    __syncthreads();
  }
}

// Element geometry for coupling factors computed in place of loaded alpha
// (p2s_fill_geometry): the trilinear map in polynomial form (A[m][c], monomial
// bit d = factor r_d), the material (a, b, c, phi) and the unit's component pair.
struct GeoUnit {
  double A[8][3];
  double mat[4];
  int gi, gj;
  int* bad;  // set when a Jacobian determinant is <= 0 (GeometryError, assembly.cpp:95-99)
};

// Per CTA: record (include/p2s_b200.h layout) -> GeoUnit in shared memory.
__device__ __forceinline__ void geo_unit_setup(const double* __restrict__ rec, int gi, int gj, GeoUnit* g,
                                               int* bad) {
  if (threadIdx.x < 24) {
    const int m = threadIdx.x / 3, comp = threadIdx.x % 3;
    double acc = 0.0;
    for (int c = 0; c < 8; ++c) {
      double sgn = 1.0;
      for (int d = 0; d < 3; ++d)
        if ((m >> d) & 1) sgn *= ((c >> d) & 1) ? 1.0 : -1.0;
      acc += sgn * __ldg(rec + c * 3 + comp);
    }
    g->A[m][comp] = 0.125 * acc;
  } else if (threadIdx.x < 28) {
    g->mat[threadIdx.x - 24] = __ldg(rec + threadIdx.x);
  } else if (threadIdx.x == 28) {
    g->gi = gi;
    g->gj = gj;
    g->bad = bad;
  }
}

// Coupling factors of one row (v, w) at the u nodes xu[], folded like a loaded
// alpha row: even terms alpha_mat detJ (J^T J)^-1_{gi gj}, odd terms
// alpha_mat (J^T J)_{gi gj} / detJ.  Along a row the Jacobian is linear in u.
template <int S, int QU>
__device__ __forceinline__ void geo_row(const GeoUnit& g, double v, double w, const double* xu,
                                        double (&ev)[S][QU / 2 > 0 ? QU / 2 : 1],
                                        double (&od)[S][QU / 2 > 0 ? QU / 2 : 1], double (&mid)[S]) {
  constexpr int Hf = QU / 2;
  double J0[3], J1a[3], J1b[3], J2a[3], J2b[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    J0[c] = g.A[1][c] + v * g.A[3][c] + w * g.A[5][c] + v * w * g.A[7][c];
    J1a[c] = g.A[2][c] + w * g.A[6][c];
    J1b[c] = g.A[3][c] + w * g.A[7][c];
    J2a[c] = g.A[4][c] + v * g.A[6][c];
    J2b[c] = g.A[5][c] + v * g.A[7][c];
  }
  const double sarg = g.mat[1] * v + g.mat[2] * w + g.mat[3];
  // pair code 3 gi + gj -> (G / cofactor) entry; G symmetric
  const int pc = g.gi * 3 + g.gj;
  auto at = [&](double u, double& mass, double& curl) {
    double J[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      J[c][0] = J0[c];
      J[c][1] = J1a[c] + u * J1b[c];
      J[c][2] = J2a[c] + u * J2b[c];
    }
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(det > 0.0)) atomicOr(g.bad, 1);
    const double G00 = J[0][0] * J[0][0] + J[1][0] * J[1][0] + J[2][0] * J[2][0];
    const double G11 = J[0][1] * J[0][1] + J[1][1] * J[1][1] + J[2][1] * J[2][1];
    const double G22 = J[0][2] * J[0][2] + J[1][2] * J[1][2] + J[2][2] * J[2][2];
    const double G01 = J[0][0] * J[0][1] + J[1][0] * J[1][1] + J[2][0] * J[2][1];
    const double G02 = J[0][0] * J[0][2] + J[1][0] * J[1][2] + J[2][0] * J[2][2];
    const double G12 = J[0][1] * J[0][2] + J[1][1] * J[1][2] + J[2][1] * J[2][2];
    double gsel, csel;
    switch (pc) {  // warp-uniform
      case 0: gsel = G00; csel = G11 * G22 - G12 * G12; break;
      case 4: gsel = G11; csel = G00 * G22 - G02 * G02; break;
      case 8: gsel = G22; csel = G00 * G11 - G01 * G01; break;
      case 1: case 3: gsel = G01; csel = G02 * G12 - G01 * G22; break;
      case 2: case 6: gsel = G02; csel = G01 * G12 - G02 * G11; break;
      default: gsel = G12; csel = G02 * G01 - G00 * G12; break;
    }
    const double am = (1.0 + 0.3 * sin(g.mat[0] * u + sarg)) / det;
    mass = am * csel;  // alpha_mat detJ cof(G) / det(G), det(G) = detJ^2
    curl = am * gsel;
  };
#pragma unroll
  for (int h = 0; h < Hf; ++h) {
    double m1, c1, m2, c2;
    at(xu[h], m1, c1);
    at(xu[QU - 1 - h], m2, c2);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      ev[s][h] = (s % 2 == 0) ? m1 + m2 : c1 + c2;
      od[s][h] = (s % 2 == 0) ? m1 - m2 : c1 - c2;
    }
  }
  if constexpr ((QU & 1) != 0) {
    double m, c;
    at(xu[Hf], m, c);
#pragma unroll
    for (int s = 0; s < S; ++s) mid[s] = (s % 2 == 0) ? m : c;
  } else {
#pragma unroll
    for (int s = 0; s < S; ++s) mid[s] = 0.0;
  }
}

// All terms of one (element, pair) at once: the kernel polynomials of every
// term are the same Legendre P_k (only the count K differs), so one half-table
// row (loaded once per thread) feeds every term that uses it, and the three
// passes need three barriers for all terms.  alpha_s slabs are consecutive
// (a + s * slab); Iout + moff(s) receives I_s.  Requires every term's tables
// to be row prefixes of term kmax_term(d)'s table (true for Legendre kernels).
// SRC: 0 alpha in global memory (read-only path), 1 coupling factors computed
// from the unit's geometry (geo, xq), 2 alpha in shared memory (cluster mode)
template <class Ms, int NTHR, int SRC = 0>
__device__ __forceinline__ void moments_all_terms(const double* __restrict__ a, const double* tab,
                                                  double* scratch, double* Iout,
                                                  const GeoUnit* geo = nullptr,
                                                  const double* xq = nullptr) {
  constexpr int S = Ms::S;
  constexpr int QU = Ms::Q(0), QV = Ms::Q(1), QW = Ms::Q(2);
  constexpr int S2 = Ms::S2, S3 = Ms::S3;
  constexpr int slab = QU * QV * QW;
  // per-term scratch: T1_s [KU_s][QW][S2] then T2_s [KU_s*KV_s][S3]
  auto t1 = [&](int s) { return scratch + Ms::t1off(s); };
  auto t2 = [&](int s) { return scratch + Ms::t2off(s); };
  // ---- pass u: thread = row (q_w, q_v) of every term
  for_items<QW * QV, NTHR>([&](int r) {
    const int q3 = r / QV, q2 = r - (r / QV) * QV;
    constexpr int Hf = QU / 2, H = (QU + 1) / 2;
    double ev[S][Hf > 0 ? Hf : 1], od[S][Hf > 0 ? Hf : 1], mid[S];
    if constexpr (SRC == 1) {  // coupling factors from the element geometry (xq = u, v, w nodes)
      geo_row<S, QU>(*geo, xq[QU + q2], xq[QU + QV + q3], xq, ev, od, mid);
    } else
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      double x[QU];
      const double* row = a + s * slab + static_cast<int64_t>(r) * QU;
      if constexpr (SRC == 2) {  // alpha in shared memory (cluster mode)
        if constexpr ((QU & 1) == 0) {
#pragma unroll
          for (int q = 0; q < QU / 2; ++q) {
            const double2 v = reinterpret_cast<const double2*>(row)[q];
            x[2 * q] = v.x;
            x[2 * q + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < QU; ++q) x[q] = row[q];
        }
      } else {
        load_row<QU>(row, x);
      }
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        ev[s][h] = x[h] + x[QU - 1 - h];
        od[s][h] = x[h] - x[QU - 1 - h];
      }
      mid[s] = (QU & 1) ? x[Hf] : 0.0;
    });
    const double* tb = tab + Ms::ttoff(0);
    static_for<0, Ms::KMAX(0)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      double v[S];
#pragma unroll
      for (int s = 0; s < S; ++s) v[s] = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        const double c = tb[k * H + h];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 0)) v[s] = fma(c, (k & 1) ? od[s][h] : ev[s][h], v[s]);
        });
      }
      if constexpr ((QU & 1) && (k & 1) == 0) {
        const double c = tb[k * H + Hf];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 0)) v[s] = fma(c, mid[s], v[s]);
        });
      }
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        if constexpr (k < Ms::K(s, 0)) t1(s)[(k * QW + q3) * S2 + q2] = v[s];
      });
    });
  });
  __syncthreads();
  // ---- pass v: thread = (k1, q_w) for every term with k1 < KU_s
  for_items<Ms::KMAX(0) * QW, NTHR>([&](int r) {
    const int k1 = r / QW, q3 = r - (r / QW) * QW;
    constexpr int Hf = QV / 2, H = (QV + 1) / 2;
    double ev[S][Hf > 0 ? Hf : 1], od[S][Hf > 0 ? Hf : 1], mid[S];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      const int kk = k1 < Ms::K(s, 0) ? k1 : 0;
      const double* src = t1(s) + (kk * QW + q3) * S2;
      double x[QV];
#pragma unroll
      for (int q = 0; q < QV; ++q) x[q] = src[q];
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        ev[s][h] = x[h] + x[QV - 1 - h];
        od[s][h] = x[h] - x[QV - 1 - h];
      }
      mid[s] = (QV & 1) ? x[Hf] : 0.0;
    });
    const double* tb = tab + Ms::ttoff(1);
    static_for<0, Ms::KMAX(1)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      double v[S];
#pragma unroll
      for (int s = 0; s < S; ++s) v[s] = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        const double c = tb[k * H + h];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 1)) v[s] = fma(c, (k & 1) ? od[s][h] : ev[s][h], v[s]);
        });
      }
      if constexpr ((QV & 1) && (k & 1) == 0) {
        const double c = tb[k * H + Hf];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 1)) v[s] = fma(c, mid[s], v[s]);
        });
      }
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        if constexpr (k < Ms::K(s, 1))
          if (k1 < Ms::K(s, 0)) t2(s)[(k1 * Ms::K(s, 1) + k) * S3 + q3] = v[s];
      });
    });
  });
  __syncthreads();
  // ---- pass w: thread = (k1, k2) over the largest term's (K_u, K_v) grid
  for_items<Ms::KMAX(0) * Ms::KMAX(1), NTHR>([&](int r) {
    const int k1 = r / Ms::KMAX(1), k2 = r - (r / Ms::KMAX(1)) * Ms::KMAX(1);
    constexpr int Hf = QW / 2, H = (QW + 1) / 2;
    double ev[S][Hf > 0 ? Hf : 1], od[S][Hf > 0 ? Hf : 1], mid[S];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      const bool in = k1 < Ms::K(s, 0) && k2 < Ms::K(s, 1);
      const double* src = t2(s) + (in ? (k1 * Ms::K(s, 1) + k2) : 0) * S3;
      double x[QW];
#pragma unroll
      for (int q = 0; q < QW; ++q) x[q] = src[q];
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        ev[s][h] = x[h] + x[QW - 1 - h];
        od[s][h] = x[h] - x[QW - 1 - h];
      }
      mid[s] = (QW & 1) ? x[Hf] : 0.0;
    });
    const double* tb = tab + Ms::ttoff(2);
    static_for<0, Ms::KMAX(2)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      double v[S];
#pragma unroll
      for (int s = 0; s < S; ++s) v[s] = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        const double c = tb[k * H + h];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 2)) v[s] = fma(c, (k & 1) ? od[s][h] : ev[s][h], v[s]);
        });
      }
      if constexpr ((QW & 1) && (k & 1) == 0) {
        const double c = tb[k * H + Hf];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 2)) v[s] = fma(c, mid[s], v[s]);
        });
      }
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        if constexpr (k < Ms::K(s, 2))
          if (k1 < Ms::K(s, 0) && k2 < Ms::K(s, 1))
            Iout[Ms::moff(s) + (k1 * Ms::K(s, 1) + k2) * Ms::K(s, 2) + k] = v[s];
      });
    });
  });
  __syncthreads();
}

// Same as moments_all_terms with the passes in the order w, v, u (cheaper and
// a smaller scratch when K_w < K_u, e.g. C4's (10, 6, 4)):
//   pass w: thread = (q_v, q_u) column, fiber along q_w (lanes read
//           consecutive q_u: every load instruction is 256 contiguous bytes)
//   pass v: thread = (k3, q_u), fiber along q_v of W1[k3][q_v][q_u]
//   pass u: thread = (k3, k2), fiber along q_u of W2[k3*KV + k2][q_u]
template <class Ms, int NTHR, bool NA = false>
__device__ __forceinline__ void moments_all_terms_wfirst(const double* __restrict__ a,
                                                         const double* tab, double* scratch,
                                                         double* Iout) {
  constexpr int S = Ms::S;
  constexpr int QU = Ms::Q(0), QV = Ms::Q(1), QW = Ms::Q(2);
  constexpr int SU = QU | 1;  // odd row stride over q_u
  constexpr int slab = QU * QV * QW;
  auto w1 = [&](int s) { return scratch + Ms::w1off(s); };   // [KW_s][QV][SU]
  auto w2 = [&](int s) { return scratch + Ms::w2off(s); };   // [KW_s*KV_s][SU]
  // ---- pass w
  for_items<QV * QU, NTHR>([&](int r) {
    constexpr int Hf = QW / 2, H = (QW + 1) / 2;
    const int q2 = r / QU, q1 = r - (r / QU) * QU;
    double ev[S][Hf > 0 ? Hf : 1], od[S][Hf > 0 ? Hf : 1], mid[S];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      const double* col = a + s * slab + r;
      double x[QW];
#pragma unroll
      for (int q = 0; q < QW; ++q)
        x[q] = NA ? ld_nc_na(col + q * (QU * QV)) : __ldg(col + q * (QU * QV));
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        ev[s][h] = x[h] + x[QW - 1 - h];
        od[s][h] = x[h] - x[QW - 1 - h];
      }
      mid[s] = (QW & 1) ? x[Hf] : 0.0;
    });
    const double* tb = tab + Ms::ttoff(2);
    static_for<0, Ms::KMAX(2)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      double v[S];
#pragma unroll
      for (int s = 0; s < S; ++s) v[s] = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        const double c = tb[k * H + h];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 2)) v[s] = fma(c, (k & 1) ? od[s][h] : ev[s][h], v[s]);
        });
      }
      if constexpr ((QW & 1) && (k & 1) == 0) {
        const double c = tb[k * H + Hf];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 2)) v[s] = fma(c, mid[s], v[s]);
        });
      }
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        if constexpr (k < Ms::K(s, 2)) w1(s)[(k * QV + q2) * SU + q1] = v[s];
      });
    });
  });
  __syncthreads();
  // ---- pass v
  for_items<Ms::KMAX(2) * QU, NTHR>([&](int r) {
    constexpr int Hf = QV / 2, H = (QV + 1) / 2;
    const int k3 = r / QU, q1 = r - (r / QU) * QU;
    double ev[S][Hf > 0 ? Hf : 1], od[S][Hf > 0 ? Hf : 1], mid[S];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      const int kk = k3 < Ms::K(s, 2) ? k3 : 0;
      const double* src = w1(s) + kk * QV * SU + q1;
      double x[QV];
#pragma unroll
      for (int q = 0; q < QV; ++q) x[q] = src[q * SU];
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        ev[s][h] = x[h] + x[QV - 1 - h];
        od[s][h] = x[h] - x[QV - 1 - h];
      }
      mid[s] = (QV & 1) ? x[Hf] : 0.0;
    });
    const double* tb = tab + Ms::ttoff(1);
    static_for<0, Ms::KMAX(1)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      double v[S];
#pragma unroll
      for (int s = 0; s < S; ++s) v[s] = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        const double c = tb[k * H + h];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 1)) v[s] = fma(c, (k & 1) ? od[s][h] : ev[s][h], v[s]);
        });
      }
      if constexpr ((QV & 1) && (k & 1) == 0) {
        const double c = tb[k * H + Hf];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 1)) v[s] = fma(c, mid[s], v[s]);
        });
      }
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        if constexpr (k < Ms::K(s, 1))
          if (k3 < Ms::K(s, 2)) w2(s)[(k3 * Ms::K(s, 1) + k) * SU + q1] = v[s];
      });
    });
  });
  __syncthreads();
  // ---- pass u
  for_items<Ms::KMAX(2) * Ms::KMAX(1), NTHR>([&](int r) {
    constexpr int Hf = QU / 2, H = (QU + 1) / 2;
    const int k3 = r / Ms::KMAX(1), k2 = r - (r / Ms::KMAX(1)) * Ms::KMAX(1);
    double ev[S][Hf > 0 ? Hf : 1], od[S][Hf > 0 ? Hf : 1], mid[S];
    static_for<0, S>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      const bool in = k3 < Ms::K(s, 2) && k2 < Ms::K(s, 1);
      const double* src = w2(s) + (in ? (k3 * Ms::K(s, 1) + k2) : 0) * SU;
      double x[QU];
#pragma unroll
      for (int q = 0; q < QU; ++q) x[q] = src[q];
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        ev[s][h] = x[h] + x[QU - 1 - h];
        od[s][h] = x[h] - x[QU - 1 - h];
      }
      mid[s] = (QU & 1) ? x[Hf] : 0.0;
    });
    const double* tb = tab + Ms::ttoff(0);
    static_for<0, Ms::KMAX(0)>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      double v[S];
#pragma unroll
      for (int s = 0; s < S; ++s) v[s] = 0.0;
#pragma unroll
      for (int h = 0; h < Hf; ++h) {
        const double c = tb[k * H + h];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 0)) v[s] = fma(c, (k & 1) ? od[s][h] : ev[s][h], v[s]);
        });
      }
      if constexpr ((QU & 1) && (k & 1) == 0) {
        const double c = tb[k * H + Hf];
        static_for<0, S>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          if constexpr (k < Ms::K(s, 0)) v[s] = fma(c, mid[s], v[s]);
        });
      }
      static_for<0, S>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        if constexpr (k < Ms::K(s, 0))
          if (k3 < Ms::K(s, 2) && k2 < Ms::K(s, 1))
            Iout[Ms::moff(s) + (k * Ms::K(s, 1) + k2) * Ms::K(s, 2) + k3] = v[s];
      });
    });
  });
  __syncthreads();
}

// one CTA per (element, pair, term)
template <class Ms>
__global__ void __launch_bounds__(Ms::THREADS) moments_v2_kernel(const __grid_constant__ MV2Params<Ms> p) {
  extern __shared__ __align__(16) double sm[];
  const int64_t unit = blockIdx.x;
  const int ps = static_cast<int>(unit % (p.P * Ms::S));
  const int64_t e = unit / (p.P * Ms::S);
  const int pair = ps / Ms::S, s = ps - pair * Ms::S;
  constexpr int slab = Ms::Q(0) * Ms::Q(1) * Ms::Q(2);
  const double* a = p.alpha + unit * slab;
  double* base = p.I + e * p.mom_per_elem + static_cast<int64_t>(pair) * Ms::MPP;
  static_for<0, Ms::S>([&](auto sc) {
    constexpr int ss = decltype(sc)::value;
    if (s == ss) moments_unit<Ms, ss>(a, p.tab, sm, base + Ms::moff(ss));
  });
}

}  // namespace p2s
