// p2s_tables.hpp -- host-side coefficient-table builder (built once per
// context, uploaded once).  Replaces the reference's per-element table work:
// gauss_legendre (quadrature.cpp:27-53), poly_table (assembly.cpp:41-49,
// 110-117) and the product_to_sum / FlatTable expansions (chebyshev.cpp:
// 156-178, assembly.cpp:332-352), generalised to Legendre kernels in 3-D.
#pragma once

#include <cstdint>
#include <vector>

namespace p2s {

enum Kind : int { PP = 0, DD = 1, DP = 2, PD = 3 };

// Bit 2 of a kind selects the conforming (hierarchical) basis in place of the
// modal P_0..P_{N-1} on both sides:  phi_0 = (P_0 - P_1)/2, phi_1 = (P_0 + P_1)/2,
// phi_n = P_n - P_{n mod 2} (n >= 2) -- the reference's conforming_matrix /
// apply_conforming_transform change of basis (assembly.cpp:476-574), phi_m =
// sum_a R[a][m] P_a.  Folding R into the product-to-sum tables makes the
// transform free inside the contraction.
constexpr int kConforming = 4;
constexpr int base_kind(int kind) { return kind & 3; }
constexpr bool conforming(int kind) { return (kind & kConforming) != 0; }

// R[a][m] of the conforming change of basis (2 nonzeros per column)
constexpr int conf_sup(int m, int i) { return m >= 2 ? (i == 0 ? m : m % 2) : i; }
constexpr double conf_r(int m, int i) {  // coefficient of P_{conf_sup(m, i)} in phi_m
  return m >= 2 ? (i == 0 ? 1.0 : -1.0) : (m == 0 ? (i == 0 ? 0.5 : -0.5) : 0.5);
}

// Number of kernel polynomials for an operator pair (paper Eq. (3)).
constexpr int kernel_count(int kind, int N) {
  const int b = base_kind(kind);
  const int K = b == PP ? 2 * N - 1 : b == DD ? 2 * N - 3 : 2 * N - 2;
  return K < 1 ? 1 : K;
}

// Nonzero band of the Legendre product-to-sum expansion of the modal pair
// (a, b): k = lo, lo+2, ..., hi (empty when hi < lo).
//   PP:  P_a P_b   -> k in [|a-b|, a+b]
//   DP:  P'_a P_b  -> k in [b >= a ? b-a+1 : (a+b-1)%2, a+b-1]   (a >= 1)
//   PD:  P_a P'_b  -> mirror of DP
//   DD:  P'_a P'_b -> k in [(a+b)%2, a+b-2]                       (a, b >= 1)
constexpr int modal_lo(int kind, int a, int b) {
  return kind == PP ? (a > b ? a - b : b - a)
         : kind == DD ? (a + b) % 2
         : kind == DP ? (b >= a ? b - a + 1 : (a + b - 1) % 2)
                      : (a >= b ? a - b + 1 : (a + b - 1) % 2);
}
constexpr int modal_hi(int kind, int a, int b) {
  return kind == PP ? a + b
         : kind == DD ? ((a >= 1 && b >= 1) ? a + b - 2 : -1)
         : kind == DP ? (a >= 1 ? a + b - 1 : -1)
                      : (b >= 1 ? a + b - 1 : -1);
}
// Conforming pair (m1, m2): the union of the modal bands of the (<= 4) modal
// pairs it combines; step 2 when they share one parity (always for m1, m2 >= 2),
// else 1 (rows / columns 0 and 1 mix parities).
constexpr int conf_band(int kind, int m1, int m2, int what) {  // 0 lo, 1 hi, 2 step
  int lo = 1 << 20, hi = -1, par = -1;
  bool mixed = false;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      const int a = conf_sup(m1, i), b = conf_sup(m2, j);
      const int l = modal_lo(kind, a, b), h = modal_hi(kind, a, b);
      if (h < l) continue;
      lo = l < lo ? l : lo;
      hi = h > hi ? h : hi;
      if (par < 0) par = l % 2;
      else if (par != l % 2) mixed = true;
    }
  return what == 0 ? (hi < 0 ? 0 : lo) : what == 1 ? hi : (mixed ? 1 : 2);
}
constexpr int band_lo(int kind, int a, int b) {
  return conforming(kind) ? conf_band(base_kind(kind), a, b, 0) : modal_lo(kind, a, b);
}
constexpr int band_hi(int kind, int a, int b) {
  return conforming(kind) ? conf_band(base_kind(kind), a, b, 1) : modal_hi(kind, a, b);
}
constexpr int band_step(int kind, int a, int b) {
  return conforming(kind) ? conf_band(base_kind(kind), a, b, 2) : 2;
}
constexpr int band_count(int kind, int a, int b) {
  return band_hi(kind, a, b) >= band_lo(kind, a, b)
             ? (band_hi(kind, a, b) - band_lo(kind, a, b)) / band_step(kind, a, b) + 1
             : 0;
}

// Gauss-Legendre rule, Newton iteration in long double.
void gauss_legendre_ld(int n, std::vector<double>& nodes, std::vector<double>& weights);

// P_k(x) and P'_k(x) for k < K in long double.
void legendre_ld(int K, long double x, long double* P, long double* dP);

// C[a][b][k], a, b < N, k < K: f_a g_b = sum_k C P_k with f, g in {P, P'}
// per kind; computed by exact Gauss-Legendre projection in long double,
// entries outside the band set to exactly zero.  Conforming kinds: the same
// projection of the transformed basis functions phi_m (R folded in).
std::vector<double> product_to_sum_table(int kind, int N);

// phi[k][q] = w_q P_k(x_q), k < K.
std::vector<double> weighted_kernel_table(int K, const std::vector<double>& nodes,
                                          const std::vector<double>& weights);

// ---------------------------------------------------------------- 2-D Chebyshev mode
// The reference's own specialisation (chebyshev.hpp / assembly.cpp):
// families T_n, U_n and the nonsingular T^ns_n, and their <= 2-term exact
// product-to-sum identities (Eq. (16)).
enum ChebFamily : int { CHEB_T = 0, CHEB_U = 1, CHEB_TNS = 2 };

// value of family fam, degree n at x (long-double recurrences; T^ns by
// Clenshaw over its integer T-coefficients, finite at x = +-1)
long double cheb_eval(int fam, int n, long double x);

struct ChebTerm {
  double coeff;
  int fam, deg;
};
// product of two T/U polynomials rewritten as <= 2 terms (equal terms merged,
// zero coefficients dropped); U_{-1} = 0, U_{-k} = -U_{k-2}
int cheb_product(int fam_a, int a, int fam_b, int b, ChebTerm out[2]);

}  // namespace p2s
