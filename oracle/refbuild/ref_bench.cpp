// ref_bench.cpp -- runs the REFERENCE's own 2-D timing study, chebfem::bench_fill
// (bench.cpp:75-140), on its Fig.-1 benchmark domain (16 curved order-4
// quadrilaterals, generate_benchmark_domain(4, 4, 4) as acceptance.cpp:220-225)
// at the orders given on the command line; prints one JSON object.  Test /
// measurement infrastructure only (bench.py's context line); built by the
// Makefile in this directory into oracle/_ref/ from the reference's sources.
//   ref_bench <threads> <reps> <M=N> [<M=N> ...]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chebfem/bench.hpp"
#include "chebfem/mesh.hpp"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: ref_bench <threads> <reps> <order> [<order> ...]\n");
    return 2;
  }
  chebfem::BenchOptions opt;
  opt.threads = std::atoi(argv[1]);
  opt.reps = std::atoi(argv[2]);
  for (int i = 3; i < argc; ++i) opt.orders.push_back(std::atoi(argv[i]));
  const chebfem::Mesh mesh = chebfem::generate_benchmark_domain(4, 4, 4);
  const chebfem::BenchReport r = chebfem::bench_fill(mesh, opt);
  std::printf("{\"elements\": %zu, \"threads\": %d, \"reps\": %d, \"rows\": [", mesh.elements.size(),
              opt.threads, opt.reps);
  for (size_t i = 0; i < r.rows.size(); ++i) {
    const chebfem::BenchRow& w = r.rows[i];
    std::printf("%s{\"M\": %d, \"N\": %d, \"fill_p2s_s\": %.6g, \"fill_direct_s\": %.6g, "
                "\"p2s_elem_per_s\": %.6g, \"measured_reduction\": %.4g, \"predicted_reduction\": %.4g}",
                i ? ", " : "", w.M, w.N, w.fill_p2s_s, w.fill_direct_s,
                static_cast<double>(mesh.elements.size()) / w.fill_p2s_s, w.measured_reduction,
                w.predicted_reduction);
  }
  std::printf("]}\n");
  return 0;
}
