// ref_probe.cpp -- golden-vector generator linked against the REFERENCE
// library compiled from /root/reference/proj/src (see oracle/refbuild/Makefile).
// Runs only in the build container (the GPU box has no /root/reference); its
// JSON output is converted by tests/golden/make_ref2d_golden.py into the
// committed fixtures tests/golden/ref2d_*.npz.
//
// Everything it calls is the reference's public API:
//   gauss_legendre            (quadrature.hpp:25)
//   eval_T/eval_U/eval_Tns, product_to_sum (chebyshev.hpp:18-66)
//   map_and_jacobian, eval_expr (mesh.hpp:67, expr.hpp:66)
//   random_single_element_mesh (bench.hpp:105; verify.cpp:25-77)
//   compute_kernel_tables, assemble_p2s_element, assemble_direct_element
//   (assembly.hpp:50-56)
// The coupling grids are recomputed with the formulas of build_element_quad
// (assembly.cpp:77-107), which is internal to the reference.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "chebfem/assembly.hpp"
#include "chebfem/bench.hpp"
#include "chebfem/chebyshev.hpp"
#include "chebfem/quadrature.hpp"

using namespace chebfem;

namespace {

void put_vec(const char* name, const std::vector<double>& v, bool comma = true) {
  std::printf("\"%s\":[", name);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? "," : "", v[i]);
  std::printf("]%s", comma ? "," : "");
}

void put_mat(const char* name, const Mat& m, bool comma = true) {
  std::printf("\"%s\":{\"rows\":%d,\"cols\":%d,", name, m.rows(), m.cols());
  put_vec("data", m.data(), false);
  std::printf("}%s", comma ? "," : "");
}

Mesh identity_mesh() {
  Mesh mesh;
  mesh.nodes = {{-1, -1}, {1, -1}, {-1, 1}, {1, 1}};
  CurvedQuadElement e;
  e.order = 1;
  e.nodes = {0, 1, 2, 3};
  mesh.elements = {e};
  mesh.boundary_edges = {{0, 0}, {0, 1}, {0, 2}, {0, 3}};
  mesh.materials.eps_r_text = "1";
  mesh.materials.mu_r_text = "1";
  mesh.materials.eps_r = parse_expr("1");
  mesh.materials.mu_r = parse_expr("1");
  return mesh;
}

// build_element_quad (assembly.cpp:77-107) through the public map.
void coupling_grids(const Mesh& mesh, int nq, Mat& ws, Mat& wuu, Mat& wuv, Mat& wvv) {
  const QuadRule1D rule = gauss_legendre(nq);
  ws = Mat(nq, nq);
  wuu = Mat(nq, nq);
  wuv = Mat(nq, nq);
  wvv = Mat(nq, nq);
  for (int j = 0; j < nq; ++j) {
    for (int i = 0; i < nq; ++i) {
      const MapSample s = map_and_jacobian(mesh.elements[0], mesh.nodes, rule.nodes[i], rule.nodes[j]);
      const double eps = eval_expr(mesh.materials.eps_r, s.x, s.y);
      const double mu = eval_expr(mesh.materials.mu_r, s.x, s.y);
      const double w2 = rule.weights[i] * rule.weights[j];
      ws(i, j) = w2 / (mu * s.J);
      wuu(i, j) = w2 * eps * (s.x_v * s.x_v + s.y_v * s.y_v) / s.J;
      wuv(i, j) = w2 * eps * (s.x_u * s.x_v + s.y_u * s.y_v) / s.J;
      wvv(i, j) = w2 * eps * (s.x_u * s.x_u + s.y_u * s.y_u) / s.J;
    }
  }
}

void put_case(const char* tag, const Mesh& mesh, const Orders& o, int nq, bool comma) {
  Mat ws, wuu, wuv, wvv;
  coupling_grids(mesh, nq, ws, wuu, wuv, wvv);
  const KernelTable kt = compute_kernel_tables(mesh, 0, o, nq);
  const ElementMatrices p2s = assemble_p2s_element(kt, o);
  const ElementMatrices dir = assemble_direct_element(mesh, 0, o, nq);
  const QuadRule1D rule = gauss_legendre(nq);
  std::printf("{\"tag\":\"%s\",\"M\":%d,\"N\":%d,\"nq\":%d,\"geom_order\":%d,", tag, o.M, o.N, nq,
              mesh.elements[0].order);
  std::printf("\"eps\":\"%s\",\"mu\":\"%s\",", mesh.materials.eps_r_text.c_str(),
              mesh.materials.mu_r_text.c_str());
  std::printf("\"n_integrals\":%ld,\"n_mass_uu_integrals\":%ld,\"direct_n_integrals\":%ld,",
              kt.n_integrals, kt.n_mass_uu_integrals, dir.n_integrals);
  put_vec("nodes", rule.nodes);
  put_mat("ws", ws);
  put_mat("wuu", wuu);
  put_mat("wuv", wuv);
  put_mat("wvv", wvv);
  put_mat("Ks", kt.Ks);
  put_mat("Kuu", kt.Kuu);
  put_mat("Kuv", kt.Kuv);
  put_mat("Kvv", kt.Kvv);
  const char* names[8] = {"Suu", "Suv", "Svu", "Svv", "Muu", "Muv", "Mvu", "Mvv"};
  const Mat* pb[8] = {&p2s.Suu, &p2s.Suv, &p2s.Svu, &p2s.Svv, &p2s.Muu, &p2s.Muv, &p2s.Mvu, &p2s.Mvv};
  const Mat* db[8] = {&dir.Suu, &dir.Suv, &dir.Svu, &dir.Svv, &dir.Muu, &dir.Muv, &dir.Mvu, &dir.Mvv};
  for (int b = 0; b < 8; ++b) put_mat((std::string("p2s_") + names[b]).c_str(), *pb[b]);
  for (int b = 0; b < 8; ++b) put_mat((std::string("direct_") + names[b]).c_str(), *db[b]);
  // conforming change of basis applied to the p2s blocks (apply_conforming_transform)
  ElementMatrices conf = p2s;
  apply_conforming_transform(conf);
  const Mat* cb[8] = {&conf.Suu, &conf.Suv, &conf.Svu, &conf.Svv, &conf.Muu, &conf.Muv, &conf.Mvu, &conf.Mvv};
  for (int b = 0; b < 8; ++b) put_mat((std::string("conf_") + names[b]).c_str(), *cb[b], b < 7);
  std::printf("}%s\n", comma ? "," : "");
}

}  // namespace

int main() {
  std::printf("{\n\"quadrature\":[");
  for (int n = 1; n <= 48; ++n) {
    const QuadRule1D r = gauss_legendre(n);
    std::printf("{\"n\":%d,", n);
    put_vec("nodes", r.nodes);
    put_vec("weights", r.weights, false);
    std::printf("}%s", n < 48 ? "," : "");
  }
  std::printf("],\n");

  // product_to_sum expansions (chebyshev.cpp:156-178), degrees <= 20
  std::printf("\"p2s\":[");
  bool first = true;
  const PolyFamily fams[2] = {PolyFamily::T, PolyFamily::U};
  for (PolyFamily fa : fams)
    for (PolyFamily fb : fams)
      for (int a = 0; a <= 20; ++a)
        for (int b = 0; b <= 20; ++b) {
          const SumExpansion e = product_to_sum(fa, a, fb, b);
          std::printf("%s[%d,%d,%d,%d", first ? "" : ",", static_cast<int>(fa), a,
                      static_cast<int>(fb), b);
          for (const SumTerm& t : e)
            std::printf(",%.17g,%d,%d", t.coeff, static_cast<int>(t.family), t.degree);
          std::printf("]");
          first = false;
        }
  std::printf("],\n");

  // family values incl. u = +-1 (test_chebyshev.cpp:131-152 pattern)
  std::mt19937 rng(2024);
  std::uniform_real_distribution<double> unit(-1.0, 1.0);
  std::vector<double> pts{-1.0, 1.0, 0.0};
  for (int i = 0; i < 29; ++i) pts.push_back(unit(rng));
  std::printf("\"points\":[");
  for (std::size_t i = 0; i < pts.size(); ++i) std::printf("%s%.17g", i ? "," : "", pts[i]);
  std::printf("],\n\"family_values\":[");
  first = true;
  for (int fam = 0; fam < 3; ++fam)
    for (int n = 0; n <= 40; ++n) {
      std::printf("%s[", first ? "" : ",");
      for (std::size_t i = 0; i < pts.size(); ++i)
        std::printf("%s%.17g", i ? "," : "", eval_poly(static_cast<PolyFamily>(fam), n, pts[i]));
      std::printf("]");
      first = false;
    }
  std::printf("],\n\"conforming\":[");
  for (int d = 1; d <= 16; ++d) {
    const Mat r = conforming_matrix(d);
    std::printf("%s[", d > 1 ? "," : "");
    for (int i = 0; i < r.rows(); ++i)
      for (int j = 0; j < r.cols(); ++j) std::printf("%s%.17g", i + j ? "," : "", r(i, j));
    std::printf("]");
  }
  std::printf("],\n\"cases\":[\n");

  // known-answer element (test_assembly.cpp:96-140)
  put_case("identity_2x2_nq10", identity_mesh(), Orders{2, 2}, 10, true);

  // seeded curved elements (test_assembly.cpp:142-158 pattern, seed 57)
  std::mt19937 r57(57);
  std::uniform_int_distribution<int> order_dist(1, 4);
  for (int trial = 0; trial < 3; ++trial) {
    const Mesh mesh = random_single_element_mesh(r57, order_dist(r57));
    for (int mn : {1, 2, 4}) {
      const Orders o{mn, mn};
      const int nq = default_quad_points(o, mesh.elements[0].order);
      const std::string tag = "seed57_t" + std::to_string(trial) + "_mn" + std::to_string(mn);
      put_case(tag.c_str(), mesh, o, nq, true);
    }
  }
  // anisotropic orders (test_assembly.cpp:160-172, seed 91)
  std::mt19937 r91(91);
  const Mesh mesh91 = random_single_element_mesh(r91, 3);
  const int aniso[3][2] = {{1, 4}, {5, 2}, {3, 7}};
  for (int c = 0; c < 3; ++c) {
    const Orders o{aniso[c][0], aniso[c][1]};
    const int nq = default_quad_points(o, 3);
    const std::string tag = "seed91_M" + std::to_string(o.M) + "_N" + std::to_string(o.N);
    put_case(tag.c_str(), mesh91, o, nq, c < 2);
  }
  std::printf("]\n}\n");
  return 0;
}
