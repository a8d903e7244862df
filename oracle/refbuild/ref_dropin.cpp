// ref_dropin.cpp -- the reference (chebfem, compiled from /root/reference/proj/src
// by oracle/refbuild/Makefile) calling the B200 fill through the C-ABI, exactly as
// a maintainer would wire it: for seeded curved elements
// (random_single_element_mesh, verify.cpp:25-77; seeds 57 / 91 / 4242 as in
// test_assembly.cpp:142-172 and acceptance.cpp:84-121) the coupling grids of
// build_element_quad (assembly.cpp:77-107) go to p2s_cheb2d_kernel_tables /
// p2s_cheb2d_assemble on the GPU, and the reference's OWN comparator
// element_matrices_close (verify.cpp:103-113) checks the GPU matrices against
// compute_kernel_tables + assemble_p2s_element at rtol 1e-12.
// Built in the container (links the static reference library), run on the B200
// by tests/test_gpu_reference2d.py.  Exit 0 = every element passed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "chebfem/assembly.hpp"
#include "chebfem/bench.hpp"
#include "chebfem/dof_map.hpp"
#include "chebfem/mesh.hpp"
#include "chebfem/quadrature.hpp"
#include "p2s_b200.h"

using namespace chebfem;

namespace {

std::vector<double> coupling_grids(const Mesh& mesh, int nq) {
  const QuadRule1D rule = gauss_legendre(nq);
  std::vector<double> g(static_cast<size_t>(4) * nq * nq);
  for (int j = 0; j < nq; ++j)
    for (int i = 0; i < nq; ++i) {
      const MapSample s = map_and_jacobian(mesh.elements[0], mesh.nodes, rule.nodes[i], rule.nodes[j]);
      const double eps = eval_expr(mesh.materials.eps_r, s.x, s.y);
      const double mu = eval_expr(mesh.materials.mu_r, s.x, s.y);
      const double w2 = rule.weights[i] * rule.weights[j];
      const size_t q = static_cast<size_t>(i) * nq + j;
      g[0 * nq * nq + q] = w2 / (mu * s.J);
      g[1 * nq * nq + q] = w2 * eps * (s.x_v * s.x_v + s.y_v * s.y_v) / s.J;
      g[2 * nq * nq + q] = w2 * eps * (s.x_u * s.x_v + s.y_u * s.y_v) / s.J;
      g[3 * nq * nq + q] = w2 * eps * (s.x_u * s.x_u + s.y_u * s.y_u) / s.J;
    }
  return g;
}

Mat block(const std::vector<double>& flat, const p2s_cheb2d_sizes& sz, int b) {
  Mat m(sz.block_rows[b], sz.block_cols[b]);
  for (int i = 0; i < m.rows(); ++i)
    for (int j = 0; j < m.cols(); ++j)
      m(i, j) = flat[static_cast<size_t>(sz.block_offset[b] + static_cast<int64_t>(i) * m.cols() + j)];
  return m;
}

// conforming: the GPU folds apply_conforming_transform into its fill; the
// reference applies it to its own p2s matrices afterwards
bool check_element(const Mesh& mesh, const Orders& o, const char* tag, bool conforming) {
  const int nq = default_quad_points(o, mesh.elements[0].order);
  p2s_cheb2d_problem pb{o.M, o.N, nq, conforming ? 1 : 0};
  p2s_cheb2d_ctx* ctx = nullptr;
  if (p2s_cheb2d_create(&pb, 0, &ctx) != P2S_OK) {
    std::printf("FAIL %s: create: %s\n", tag, p2s_last_error());
    return false;
  }
  p2s_cheb2d_sizes sz{};
  p2s_cheb2d_get_sizes(ctx, &sz);
  const std::vector<double> grids = coupling_grids(mesh, nq);
  double *dg = nullptr, *dt = nullptr, *db = nullptr;
  cudaMalloc(&dg, sizeof(double) * grids.size());
  cudaMalloc(&dt, sizeof(double) * sz.tables_per_elem);
  cudaMalloc(&db, sizeof(double) * sz.blocks_per_elem);
  cudaMemcpy(dg, grids.data(), sizeof(double) * grids.size(), cudaMemcpyHostToDevice);
  bool ok = p2s_cheb2d_kernel_tables(ctx, dg, dt, 1, nullptr) == P2S_OK &&
            p2s_cheb2d_assemble(ctx, dt, db, 1, nullptr) == P2S_OK;
  std::vector<double> blocks(static_cast<size_t>(sz.blocks_per_elem));
  ok = ok && cudaMemcpy(blocks.data(), db, sizeof(double) * blocks.size(), cudaMemcpyDeviceToHost) == cudaSuccess;
  cudaFree(dg);
  cudaFree(dt);
  cudaFree(db);
  p2s_cheb2d_destroy(ctx);
  if (!ok) {
    std::printf("FAIL %s: GPU call failed: %s\n", tag, p2s_last_error());
    return false;
  }
  ElementMatrices gpu;
  gpu.orders = o;
  gpu.Suu = block(blocks, sz, 0);
  gpu.Suv = block(blocks, sz, 1);
  gpu.Svu = block(blocks, sz, 2);
  gpu.Svv = block(blocks, sz, 3);
  gpu.Muu = block(blocks, sz, 4);
  gpu.Muv = block(blocks, sz, 5);
  gpu.Mvu = block(blocks, sz, 6);
  gpu.Mvv = block(blocks, sz, 7);
  ElementMatrices ref = assemble_p2s_element(compute_kernel_tables(mesh, 0, o, nq), o);
  if (conforming) apply_conforming_transform(ref);
  std::string msg;
  if (!element_matrices_close(ref, gpu, 1e-12, &msg)) {
    std::printf("FAIL %s M=%d N=%d conforming=%d: %s\n", tag, o.M, o.N, conforming, msg.c_str());
    return false;
  }
  return true;
}

// The reference's assemble_system (assembly.cpp:702-711) with the fill, the
// conforming transform and the global scatter on the GPU: connectivity from the
// reference's build_connectivity, every element's grids in one batched
// p2s_cheb2d_kernel_tables / p2s_cheb2d_assemble (conforming = 1) call, then
// p2s_cheb2d_scatter; compared with the reference's global S and M.
bool check_system(const Mesh& mesh, const Orders& o, const char* tag) {
  int geom = 1;
  for (const auto& el : mesh.elements) geom = std::max(geom, el.order);
  const int nq = default_quad_points(o, geom);
  const DofMap dm = build_connectivity(mesh, o.M, o.N);
  const int E = static_cast<int>(mesh.elements.size());
  p2s_cheb2d_problem pb{o.M, o.N, nq, 1};
  p2s_cheb2d_ctx* ctx = nullptr;
  if (p2s_cheb2d_create(&pb, 0, &ctx) != P2S_OK) return false;
  p2s_cheb2d_sizes sz{};
  p2s_cheb2d_get_sizes(ctx, &sz);
  const int n_local = sz.n_eu + sz.n_ev;
  std::vector<double> grids;
  std::vector<int32_t> fr;
  std::vector<double> sg;
  for (int e = 0; e < E; ++e) {
    Mesh one = mesh;
    one.elements = {mesh.elements[static_cast<size_t>(e)]};
    const std::vector<double> g = coupling_grids(one, nq);
    grids.insert(grids.end(), g.begin(), g.end());
    for (int i = 0; i < n_local; ++i) {
      const DofMap::LocalDof& d = dm.element_dofs[static_cast<size_t>(e)][static_cast<size_t>(i)];
      fr.push_back(dm.free_index[static_cast<size_t>(d.global)]);
      sg.push_back(d.sign);
    }
  }
  const int nf = dm.n_free;
  double *dg, *dt, *db, *dS, *dM, *dsg;
  int32_t* dfr;
  cudaMalloc(&dg, sizeof(double) * grids.size());
  cudaMalloc(&dt, sizeof(double) * sz.tables_per_elem * E);
  cudaMalloc(&db, sizeof(double) * sz.blocks_per_elem * E);
  cudaMalloc(&dS, sizeof(double) * nf * nf);
  cudaMalloc(&dM, sizeof(double) * nf * nf);
  cudaMalloc(&dfr, sizeof(int32_t) * fr.size());
  cudaMalloc(&dsg, sizeof(double) * sg.size());
  cudaMemcpy(dg, grids.data(), sizeof(double) * grids.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dfr, fr.data(), sizeof(int32_t) * fr.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dsg, sg.data(), sizeof(double) * sg.size(), cudaMemcpyHostToDevice);
  cudaMemset(dS, 0, sizeof(double) * nf * nf);
  cudaMemset(dM, 0, sizeof(double) * nf * nf);
  bool ok = p2s_cheb2d_kernel_tables(ctx, dg, dt, E, nullptr) == P2S_OK &&
            p2s_cheb2d_assemble(ctx, dt, db, E, nullptr) == P2S_OK &&
            p2s_cheb2d_scatter(ctx, db, dfr, dsg, E, dS, dM, nf, nullptr) == P2S_OK;
  ElementMatrices gpu, ref;
  gpu.orders = ref.orders = o;
  gpu.Suu = Mat(nf, nf);
  gpu.Muu = Mat(nf, nf);
  ok = ok &&
       cudaMemcpy(gpu.Suu.data().data(), dS, sizeof(double) * nf * nf, cudaMemcpyDeviceToHost) == cudaSuccess &&
       cudaMemcpy(gpu.Muu.data().data(), dM, sizeof(double) * nf * nf, cudaMemcpyDeviceToHost) == cudaSuccess;
  for (void* p : {static_cast<void*>(dg), static_cast<void*>(dt), static_cast<void*>(db),
                  static_cast<void*>(dS), static_cast<void*>(dM), static_cast<void*>(dfr),
                  static_cast<void*>(dsg)})
    cudaFree(p);
  p2s_cheb2d_destroy(ctx);
  if (!ok) {
    std::printf("FAIL system %s: GPU call failed: %s\n", tag, p2s_last_error());
    return false;
  }
  const GlobalSystem sys = assemble_system(mesh, o, Backend::p2s, nq, 1);
  ref.Suu = sys.S;
  ref.Muu = sys.M;
  std::string msg;
  // the reference's own comparator on (S, M) carried in the Suu / Muu slots
  if (!element_matrices_close(ref, gpu, 1e-12, &msg)) {
    std::printf("FAIL system %s M=%d N=%d: %s\n", tag, o.M, o.N, msg.c_str());
    return false;
  }
  return true;
}

}  // namespace

int main() {
  int n_ok = 0, n = 0;
  for (unsigned seed : {57u, 91u, 4242u}) {
    std::mt19937 rng(seed);
    std::uniform_int_distribution<int> order_dist(1, 4);
    for (int trial = 0; trial < 6; ++trial) {
      const Mesh mesh = random_single_element_mesh(rng, order_dist(rng));
      for (int mn = 1; mn <= 8; ++mn) {
        const std::string tag = "seed" + std::to_string(seed) + "/t" + std::to_string(trial);
        for (bool conf : {false, true}) {
          ++n;
          n_ok += check_element(mesh, Orders{mn, mn}, tag.c_str(), conf);
        }
      }
      for (const auto& mn : {std::pair<int, int>{1, 4}, {5, 2}, {3, 7}})
        for (bool conf : {false, true}) {
          ++n;
          n_ok += check_element(mesh, Orders{mn.first, mn.second}, "aniso", conf);
        }
    }
  }
  // the 16 elements of the paper's Fig.-1 benchmark domain at M = N = 4 and 8
  const Mesh dom = generate_benchmark_domain(4, 4, 4);
  for (size_t e = 0; e < dom.elements.size(); ++e) {
    Mesh one = dom;
    one.elements = {dom.elements[e]};
    for (int mn : {4, 8})
      for (bool conf : {false, true}) {
        ++n;
        n_ok += check_element(one, Orders{mn, mn}, "fig1", conf);
      }
  }
  // full pipeline: connectivity + GPU fill + conforming + GPU scatter vs assemble_system
  int s_ok = 0, s_n = 0;
  for (int nx : {2, 4})
    for (int mn : {2, 4, 6}) {
      ++s_n;
      s_ok += check_system(generate_benchmark_domain(nx, nx, 4), Orders{mn, mn}, "benchmark");
    }
  ++s_n;
  s_ok += check_system(generate_benchmark_domain(3, 2, 3), Orders{3, 5}, "benchmark-aniso");
  std::printf("ref_dropin: %d / %d global systems (assemble_system on GPU) pass\n", s_ok, s_n);
  std::printf("ref_dropin: %d / %d elements (modal and conforming) pass "
              "element_matrices_close(reference, gpu, 1e-12)\n",
              n_ok, n);
  return (n_ok == n && s_ok == s_n) ? 0 : 1;
}
