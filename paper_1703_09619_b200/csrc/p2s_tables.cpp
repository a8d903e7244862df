// p2s_tables.cpp -- see p2s_tables.hpp.
#include "p2s_tables.hpp"

#include <cmath>

namespace p2s {

namespace {
constexpr long double kPiL = 3.141592653589793238462643383279502884L;
}

void legendre_ld(int K, long double x, long double* P, long double* dP) {
  if (K <= 0) return;
  P[0] = 1.0L;
  dP[0] = 0.0L;
  if (K == 1) return;
  P[1] = x;
  dP[1] = 1.0L;
  for (int k = 1; k + 1 < K; ++k) {
    P[k + 1] = ((2 * k + 1) * x * P[k] - k * P[k - 1]) / (k + 1);
    dP[k + 1] = dP[k - 1] + (2 * k + 1) * P[k];
  }
}

void gauss_legendre_ld(int n, std::vector<double>& nodes, std::vector<double>& weights) {
  nodes.assign(static_cast<size_t>(n), 0.0);
  weights.assign(static_cast<size_t>(n), 0.0);
  std::vector<long double> P(static_cast<size_t>(n) + 2), dP(static_cast<size_t>(n) + 2);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    long double x = cosl(kPiL * (i + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 200; ++it) {
      legendre_ld(n + 1, x, P.data(), dP.data());
      const long double dx = P[n] / dP[n];
      x -= dx;
      if (fabsl(dx) < 1e-19L) break;
    }
    if (n % 2 == 1 && i == (n + 1) / 2 - 1) x = 0.0L;
    legendre_ld(n + 1, x, P.data(), dP.data());
    const long double w = 2.0L / ((1.0L - x * x) * dP[n] * dP[n]);
    nodes[static_cast<size_t>(n - 1 - i)] = static_cast<double>(x);
    nodes[static_cast<size_t>(i)] = static_cast<double>(-x);
    weights[static_cast<size_t>(n - 1 - i)] = static_cast<double>(w);
    weights[static_cast<size_t>(i)] = static_cast<double>(w);
  }
}

std::vector<double> product_to_sum_table(int kind, int N) {
  const int K = kernel_count(kind, N);
  // projection rule exact for degree (2N-2) + (K-1) <= 4N
  const int nq = 2 * N + 2;
  std::vector<long double> x(static_cast<size_t>(nq)), w(static_cast<size_t>(nq));
  {
    // long-double rule (nodes kept in extended precision here)
    std::vector<long double> P(static_cast<size_t>(nq) + 2), dP(static_cast<size_t>(nq) + 2);
    for (int i = 0; i < (nq + 1) / 2; ++i) {
      long double t = cosl(kPiL * (i + 0.75L) / (nq + 0.5L));
      for (int it = 0; it < 200; ++it) {
        legendre_ld(nq + 1, t, P.data(), dP.data());
        const long double dx = P[nq] / dP[nq];
        t -= dx;
        if (fabsl(dx) < 1e-19L) break;
      }
      if (nq % 2 == 1 && i == (nq + 1) / 2 - 1) t = 0.0L;
      legendre_ld(nq + 1, t, P.data(), dP.data());
      const long double wt = 2.0L / ((1.0L - t * t) * dP[nq] * dP[nq]);
      x[static_cast<size_t>(nq - 1 - i)] = t;
      x[static_cast<size_t>(i)] = -t;
      w[static_cast<size_t>(nq - 1 - i)] = wt;
      w[static_cast<size_t>(i)] = wt;
    }
  }
  const int KP = (N > K ? N : K) + 1;
  std::vector<long double> P(static_cast<size_t>(nq) * KP), dP(static_cast<size_t>(nq) * KP);
  for (int q = 0; q < nq; ++q) legendre_ld(KP, x[q], &P[q * KP], &dP[q * KP]);
  if (conforming(kind)) {  // phi_m = sum_i conf_r(m, i) P_{conf_sup(m, i)}: fold R into the basis
    std::vector<long double> Pc(P.size(), 0.0L), dPc(dP.size(), 0.0L);
    for (int q = 0; q < nq; ++q)
      for (int m = 0; m < N; ++m)
        for (int i = 0; i < 2; ++i) {
          const int a = conf_sup(m, i);
          Pc[q * KP + m] += conf_r(m, i) * P[q * KP + a];
          dPc[q * KP + m] += conf_r(m, i) * dP[q * KP + a];
        }
    // the kernel polynomials (index k) stay modal: P_k below
    std::vector<double> C(static_cast<size_t>(N) * N * K, 0.0);
    const int bk = base_kind(kind);
    const bool da = (bk == DD || bk == DP), db = (bk == DD || bk == PD);
    for (int a = 0; a < N; ++a)
      for (int b = 0; b < N; ++b) {
        const int lo = band_lo(kind, a, b), hi = band_hi(kind, a, b), st = band_step(kind, a, b);
        for (int k = lo; k <= hi && k < K; k += st) {
          long double s = 0.0L;
          for (int q = 0; q < nq; ++q) {
            const long double fa = da ? dPc[q * KP + a] : Pc[q * KP + a];
            const long double gb = db ? dPc[q * KP + b] : Pc[q * KP + b];
            s += w[q] * fa * gb * P[q * KP + k];
          }
          C[(static_cast<size_t>(a) * N + b) * K + k] = static_cast<double>(s * (2 * k + 1) / 2);
        }
      }
    return C;
  }
  const bool da = (kind == DD || kind == DP);
  const bool db = (kind == DD || kind == PD);
  std::vector<double> C(static_cast<size_t>(N) * N * K, 0.0);
  for (int a = 0; a < N; ++a)
    for (int b = 0; b < N; ++b) {
      const int lo = band_lo(kind, a, b), hi = band_hi(kind, a, b);
      for (int k = lo; k <= hi && k < K; k += 2) {
        long double s = 0.0L;
        for (int q = 0; q < nq; ++q) {
          const long double fa = da ? dP[q * KP + a] : P[q * KP + a];
          const long double gb = db ? dP[q * KP + b] : P[q * KP + b];
          s += w[q] * fa * gb * P[q * KP + k];
        }
        C[(static_cast<size_t>(a) * N + b) * K + k] = static_cast<double>(s * (2 * k + 1) / 2);
      }
    }
  return C;
}

std::vector<double> weighted_kernel_table(int K, const std::vector<double>& nodes,
                                          const std::vector<double>& weights) {
  const int nq = static_cast<int>(nodes.size());
  std::vector<double> phi(static_cast<size_t>(K) * nq);
  std::vector<long double> P(static_cast<size_t>(K)), dP(static_cast<size_t>(K));
  for (int q = 0; q < nq; ++q) {
    legendre_ld(K, nodes[q], P.data(), dP.data());
    for (int k = 0; k < K; ++k)
      phi[static_cast<size_t>(k) * nq + q] =
          static_cast<double>(static_cast<long double>(weights[q]) * P[k]);
  }
  return phi;
}

long double cheb_eval(int fam, int n, long double x) {
  if (fam == CHEB_T || fam == CHEB_U) {
    if (n == 0) return 1.0L;
    long double p = 1.0L, q = (fam == CHEB_T) ? x : 2.0L * x;
    for (int k = 1; k < n; ++k) {
      const long double r = 2.0L * x * q - p;
      p = q;
      q = r;
    }
    return q;
  }
  // T^ns_n = (T_n - T_{n mod 2}) / (2 (1 - x^2)) as a T-series:
  // T^ns_{2s} = -(s T_0 + sum_{m<s} 2(s-m) T_{2m}),  T^ns_{2s+1} = -sum_{q<s} 2(s-q) T_{2q+1}
  if (n < 2) return 0.0L;
  std::vector<long double> c(static_cast<size_t>(n - 1), 0.0L);
  if (n % 2 == 0) {
    const int s = n / 2;
    c[0] = -static_cast<long double>(s);
    for (int m = 1; m < s; ++m) c[static_cast<size_t>(2 * m)] = -2.0L * (s - m);
  } else {
    const int s = (n - 1) / 2;
    for (int q = 0; q < s; ++q) c[static_cast<size_t>(2 * q + 1)] = -2.0L * (s - q);
  }
  long double b1 = 0.0L, b2 = 0.0L;
  for (int k = static_cast<int>(c.size()) - 1; k >= 1; --k) {
    const long double b = c[static_cast<size_t>(k)] + 2.0L * x * b1 - b2;
    b2 = b1;
    b1 = b;
  }
  return c[0] + x * b1 - b2;
}

namespace {
void add_term(ChebTerm out[2], int& n, double coeff, int fam, int deg) {
  if (coeff == 0.0) return;
  for (int i = 0; i < n; ++i)
    if (out[i].fam == fam && out[i].deg == deg) {
      out[i].coeff += coeff;
      if (out[i].coeff == 0.0) {
        out[i] = out[n - 1];
        --n;
      }
      return;
    }
  out[n++] = ChebTerm{coeff, fam, deg};
}
}  // namespace

int cheb_product(int fa, int a, int fb, int b, ChebTerm out[2]) {
  int n = 0;
  if (fa == CHEB_U && fb == CHEB_U) {
    // U_a U_b = T^ns_|a-b| - T^ns_{a+b+2}
    add_term(out, n, 1.0, CHEB_TNS, a > b ? a - b : b - a);
    add_term(out, n, -1.0, CHEB_TNS, a + b + 2);
  } else if (fa == CHEB_T && fb == CHEB_T) {
    // T_a T_b = (T_|a-b| + T_{a+b}) / 2
    add_term(out, n, 0.5, CHEB_T, a > b ? a - b : b - a);
    add_term(out, n, 0.5, CHEB_T, a + b);
  } else {
    // U_u T_t = (U_{u-t} + U_{u+t}) / 2 with signed U indices
    const int u = (fa == CHEB_U) ? a : b, t = (fa == CHEB_U) ? b : a;
    const int k = u - t;
    if (k >= 0)
      add_term(out, n, 0.5, CHEB_U, k);
    else if (k <= -2)
      add_term(out, n, -0.5, CHEB_U, -k - 2);
    add_term(out, n, 0.5, CHEB_U, u + t);
  }
  return n;
}

}  // namespace p2s
