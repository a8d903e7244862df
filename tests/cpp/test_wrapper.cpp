// tests/cpp/test_wrapper.cpp -- the reference-shaped C++ API (include/p2s_b200.hpp)
// on a B200.  Built by tests/test_capi_cpu.py (compile only, CPU) and run by
// tests/test_gpu_cxx.py (GPU).  Known answers need no oracle:
//   * alpha = 1, PP term: the element matrix is the Legendre mass matrix,
//     diagonal with entries 8 / ((2m+1)(2n+1)(2p+1));
//   * fill_elements == compute_kernel_tables + assemble_p2s_element, bitwise;
//   * assemble_p2s_element with tables of other orders throws
//     std::invalid_argument (assembly.cpp:376-378).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "p2s_b200.hpp"

#define REQUIRE(c)                                                   \
  do {                                                               \
    if (!(c)) {                                                      \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                      \
    }                                                                \
  } while (0)

int main() {
  p2s::Problem pb;
  pb.n_comp = 1;
  pb.orders = {4, 4, 4};
  pb.terms = {p2s::Term{}};
  pb.nq = {8, 8, 8};
  p2s::Context ctx(pb, 0);
  const int64_t n = 3;
  std::vector<double> alpha(static_cast<size_t>(n * ctx.alpha_per_elem()), 1.0);
  p2s::KernelTable kt = p2s::compute_kernel_tables(ctx, alpha);
  REQUIRE(kt.n_elem == n);
  p2s::ElementMatrices em = p2s::assemble_p2s_element(ctx, kt);
  REQUIRE(em.n_tot == 64);
  double worst = 0.0;
  for (int64_t e = 0; e < n; ++e)
    for (int i = 0; i < 64; ++i)
      for (int j = 0; j < 64; ++j) {
        const int m = i / 16, nn = (i / 4) % 4, p = i % 4;
        const double expect = (i == j) ? 8.0 / ((2 * m + 1) * (2 * nn + 1) * (2 * p + 1)) : 0.0;
        worst = std::fmax(worst, std::fabs(em(e, i, j) - expect));
      }
  REQUIRE(worst <= 1e-14);

  p2s::ElementMatrices f = p2s::fill_elements(pb, alpha, 1);
  REQUIRE(f.M == em.M);

  p2s::Problem other = pb;
  other.orders = {4, 4, 3};
  p2s::Context ctx2(other, 0);
  bool threw = false;
  try {
    p2s::assemble_p2s_element(ctx2, kt);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);
  std::printf("cxx wrapper ok (max |M - mass| = %.3g, path: %s)\n", worst, ctx.kernel_path().c_str());
  return 0;
}
