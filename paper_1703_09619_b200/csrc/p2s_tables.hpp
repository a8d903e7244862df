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

// Number of kernel polynomials for an operator pair (paper Eq. (3)).
constexpr int kernel_count(int kind, int N) {
  const int K = kind == PP ? 2 * N - 1 : kind == DD ? 2 * N - 3 : 2 * N - 2;
  return K < 1 ? 1 : K;
}

// Nonzero band of the Legendre product-to-sum expansion of the pair (a, b):
// k = lo, lo+2, ..., hi (empty when hi < lo).
//   PP:  P_a P_b   -> k in [|a-b|, a+b]
//   DP:  P'_a P_b  -> k in [b >= a ? b-a+1 : (a+b-1)%2, a+b-1]   (a >= 1)
//   PD:  P_a P'_b  -> mirror of DP
//   DD:  P'_a P'_b -> k in [(a+b)%2, a+b-2]                       (a, b >= 1)
constexpr int band_lo(int kind, int a, int b) {
  return kind == PP ? (a > b ? a - b : b - a)
         : kind == DD ? (a + b) % 2
         : kind == DP ? (b >= a ? b - a + 1 : (a + b - 1) % 2)
                      : (a >= b ? a - b + 1 : (a + b - 1) % 2);
}
constexpr int band_hi(int kind, int a, int b) {
  return kind == PP ? a + b
         : kind == DD ? ((a >= 1 && b >= 1) ? a + b - 2 : -1)
         : kind == DP ? (a >= 1 ? a + b - 1 : -1)
                      : (b >= 1 ? a + b - 1 : -1);
}
constexpr int band_count(int kind, int a, int b) {
  return band_hi(kind, a, b) >= band_lo(kind, a, b)
             ? (band_hi(kind, a, b) - band_lo(kind, a, b)) / 2 + 1
             : 0;
}

// Gauss-Legendre rule, Newton iteration in long double.
void gauss_legendre_ld(int n, std::vector<double>& nodes, std::vector<double>& weights);

// P_k(x) and P'_k(x) for k < K in long double.
void legendre_ld(int K, long double x, long double* P, long double* dP);

// C[a][b][k], a, b < N, k < K: f_a g_b = sum_k C P_k with f, g in {P, P'}
// per kind; computed by exact Gauss-Legendre projection in long double,
// entries outside the band set to exactly zero.
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
