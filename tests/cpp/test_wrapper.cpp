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

#include <cuda_runtime_api.h>

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

  // counters (assembly.cpp:291-310, 665-666): 7^3 moments of the single PP term
  REQUIRE(kt.n_integrals == 343 * n && kt.n_mass_uu_integrals == 343 * n);
  REQUIRE(f.n_integrals == kt.n_integrals && em.n_mass_uu_integrals == kt.n_mass_uu_integrals);
  // nq <= 0: the reference's default_quad_points (4 + 1 + 6 = 11 per direction)
  p2s::Problem dq = pb;
  dq.nq = {0, 0, 0};
  REQUIRE(dq.c().nq[0] == 11 && dq.c().nq[2] == 11);
  p2s::Context ctx3(dq, 0);
  REQUIRE(ctx3.alpha_per_elem() == 11 * 11 * 11);

  // every device of the box (the reference's thread pool, assembly.cpp:676-698):
  // the result is independent of the device count
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 1) {
    std::vector<double> a2(static_cast<size_t>(37 * ctx.alpha_per_elem()));
    for (size_t i = 0; i < a2.size(); ++i) a2[i] = 1.0 + 0.25 * std::sin(0.001 * static_cast<double>(i));
    p2s::ElementMatrices one = p2s::fill_elements(pb, a2, 1);
    p2s::ElementMatrices all = p2s::fill_elements(pb, a2, ndev);
    REQUIRE(one.M == all.M);
    std::printf("fill_elements on %d devices == 1 device\n", ndev);
  } else {
    std::printf("fill_elements multi-device check skipped (%d device)\n", ndev);
  }
  std::printf("cxx wrapper ok (max |M - mass| = %.3g, path: %s)\n", worst, ctx.kernel_path().c_str());
  return 0;
}
