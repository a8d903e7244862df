// tests/cpp/test_wrapper_cpu.cpp -- host logic of the C++ API that needs no
// GPU (run by tests/test_capi_cpu.py): the element partition of the multi-GPU
// fill_elements, the first-exception rethrow of its worker pool (reference
// fill_elements, assembly.cpp:676-698: workers catch, the first exception is
// rethrown on the caller after every worker joined), sizes without a device
// and the nq <= 0 default (assembly.cpp:23-25).
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
  // contiguous partition: covers [0, n) exactly once, sizes differ by <= 1
  for (int64_t n : {0, 1, 7, 8, 1000, 262144})
    for (int g : {1, 2, 3, 4, 8}) {
      int64_t next = 0, lo = n, hi = 0;
      for (int w = 0; w < g; ++w) {
        const auto r = p2s::element_range(n, w, g);
        REQUIRE(r.first == next && r.second >= r.first);
        next = r.second;
        lo = std::min(lo, r.second - r.first);
        hi = std::max(hi, r.second - r.first);
      }
      REQUIRE(next == n && hi - lo <= 1);
    }

  p2s::Problem pb;
  pb.orders = {4, 3, 2};
  pb.terms = {p2s::Term{}, p2s::Term{p2s::Kind::DD, p2s::Kind::DD, p2s::Kind::DD}};
  pb.nq = {0, 5, 0};
  const p2s_problem c = pb.c();
  REQUIRE(c.nq[0] == 11 && c.nq[1] == 5 && c.nq[2] == 11);
  p2s_sizes sz{};
  p2s::check(p2s_problem_sizes(&c, &sz));
  REQUIRE(sz.n_tot == 24 && sz.alpha_per_elem == 2 * 11 * 5 * 11);
  REQUIRE(sz.K[0][0] == 7 && sz.K[1][0] == 5 && sz.K[1][2] == 1);

  // bad arguments: std::invalid_argument before any device work
  bool threw = false;
  try {
    p2s::fill_elements(pb, std::vector<double>(7, 1.0), 2);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);

  // without a device every worker fails; exactly one exception (the first) reaches
  // the caller, after all workers joined, with the CUDA error type
  std::vector<double> alpha(static_cast<size_t>(5 * sz.alpha_per_elem), 1.0);
  int ndev = 0;
  threw = false;
  try {
    p2s::fill_elements(pb, alpha, 4);
  } catch (const p2s::CudaError& e) {
    threw = true;
    std::printf("rethrown: %s\n", e.what());
  } catch (const std::invalid_argument& e) {  // a box with fewer than 4 devices
    threw = true;
    std::printf("rethrown: %s\n", e.what());
  }
  (void)ndev;
  REQUIRE(threw);
  std::printf("cxx host logic ok\n");
  return 0;
}
