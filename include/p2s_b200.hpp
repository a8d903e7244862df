// p2s_b200.hpp -- C++ host API over the C-ABI (header-only), keeping the
// shape of the reference's fill interface (include/chebfem/assembly.hpp):
//
//   chebfem::compute_kernel_tables(mesh, e, orders, nq)    -> p2s::compute_kernel_tables
//   chebfem::assemble_p2s_element(kernels, orders)         -> p2s::assemble_p2s_element
//   chebfem::fill_elements(mesh, orders, Backend, nq, thr) -> p2s::fill_elements (gpus)
//
// Value semantics as in the reference (owning std::vector results), the same
// exception types for the same failures (std::invalid_argument for bad
// orders / buffers, assembly.cpp:20,376-378), and a multi-GPU fill_elements
// that runs one host thread per GPU over contiguous element ranges and
// rethrows the first worker exception on the caller (assembly.cpp:676-698).
// The GPU is the implementation; there is no CPU backend behind this API.
#pragma once

#include <array>
#include <cstdint>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "p2s_b200.h"

namespace p2s {

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class UnsupportedShape : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class GeometryError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(p2s_status st) {
  if (st == P2S_OK) return;
  const std::string msg = p2s_last_error();
  switch (st) {
    case P2S_INVALID_ARG: throw std::invalid_argument(msg);
    case P2S_UNSUPPORTED_SHAPE: throw UnsupportedShape(msg);
    case P2S_GEOMETRY_ERROR: throw GeometryError(msg);
    default: throw CudaError(msg);
  }
}

enum class Kind : int { PP = P2S_PP, DD = P2S_DD, DP = P2S_DP, PD = P2S_PD };

struct Term {
  Kind u = Kind::PP, v = Kind::PP, w = Kind::PP;
};

// Orders per direction (the 3-D counterpart of chebfem::Orders, dof_map.hpp:13-20).
struct Orders {
  int Nu = 1, Nv = 1, Nw = 1;
  int n_local() const { return Nu * Nv * Nw; }
  bool operator==(const Orders& o) const { return Nu == o.Nu && Nv == o.Nv && Nw == o.Nw; }
};

// Quadrature points per direction when the caller passes nq <= 0: the
// reference's policy max(M, N) + geometric order + 6 (default_quad_points,
// assembly.cpp:23-25, applied by assemble_system at :704-706), here over the
// three orders; geometric order 1 = the trilinear hexahedron.
inline int default_quad_points(const Orders& o, int geometric_order = 1) {
  int m = o.Nu > o.Nv ? o.Nu : o.Nv;
  m = m > o.Nw ? m : o.Nw;
  return m + geometric_order + 6;
}

struct Problem {
  int n_comp = 1;
  Orders orders;
  std::vector<Term> terms{Term{}};
  std::array<int, 3> nq{0, 0, 0};  // <= 0: default_quad_points(orders, geometric_order)
  int geometric_order = 1;
  bool conforming = false;  // conforming basis (reference apply_conforming_transform)

  int resolved_nq(int d) const { return nq[d] > 0 ? nq[d] : default_quad_points(orders, geometric_order); }

  p2s_problem c() const {
    p2s_problem p{};
    p.n_comp = n_comp;
    p.order[0] = orders.Nu;
    p.order[1] = orders.Nv;
    p.order[2] = orders.Nw;
    p.n_terms = static_cast<int32_t>(terms.size());
    for (size_t s = 0; s < terms.size() && s < P2S_MAX_TERMS; ++s) {
      p.kind[s][0] = static_cast<int>(terms[s].u);
      p.kind[s][1] = static_cast<int>(terms[s].v);
      p.kind[s][2] = static_cast<int>(terms[s].w);
    }
    for (int d = 0; d < 3; ++d) p.nq[d] = resolved_nq(d);
    p.basis = conforming ? P2S_BASIS_CONFORMING : P2S_BASIS_MODAL;
    return p;
  }
  bool same_shape(const Problem& o) const {
    if (n_comp != o.n_comp || !(orders == o.orders) || terms.size() != o.terms.size() ||
        conforming != o.conforming)
      return false;
    for (int d = 0; d < 3; ++d)
      if (resolved_nq(d) != o.resolved_nq(d)) return false;
    for (size_t s = 0; s < terms.size(); ++s)
      if (terms[s].u != o.terms[s].u || terms[s].v != o.terms[s].v || terms[s].w != o.terms[s].w)
        return false;
    return true;
  }
};

// RAII owner of one p2s_ctx (tables uploaded once, immutable).
class Context {
 public:
  Context(const Problem& pb, int device = 0) : problem_(pb) {
    const p2s_problem c = pb.c();
    check(p2s_create(&c, device, &h_));
    check(p2s_get_sizes(h_, &sizes_));
  }
  ~Context() {
    if (h_) p2s_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  Context(Context&& o) noexcept : h_(std::exchange(o.h_, nullptr)), sizes_(o.sizes_), problem_(o.problem_) {}

  p2s_ctx* handle() const { return h_; }
  const p2s_sizes& sizes() const { return sizes_; }
  const Problem& problem() const { return problem_; }
  int64_t alpha_per_elem() const { return sizes_.alpha_per_elem; }
  int64_t moments_per_elem() const { return sizes_.moments_per_elem; }
  int n_tot() const { return sizes_.n_tot; }
  std::string kernel_path() const { return p2s_kernel_path(h_); }

  // device-pointer entry points (caller-owned buffers, asynchronous on stream)
  void moments(const double* d_alpha, double* d_I, int64_t n, void* stream = nullptr) {
    check(p2s_moments(h_, d_alpha, d_I, n, stream));
  }
  void contract(const double* d_I, double* d_M, int64_t ld, int64_t n, void* stream = nullptr) {
    check(p2s_contract(h_, d_I, d_M, ld, n, stream));
  }
  void fill(const double* d_alpha, double* d_M, int64_t ld, int64_t n, void* stream = nullptr) {
    check(p2s_fill(h_, d_alpha, d_M, ld, n, stream));
  }

 private:
  p2s_ctx* h_ = nullptr;
  p2s_sizes sizes_{};
  Problem problem_;
};

// RAII owner of one p2s_direct_ctx: the direct-quadrature fill (reference
// assemble_direct_element, assembly.hpp:50), device buffers, same layouts.
class DirectContext {
 public:
  DirectContext(const Problem& pb, int device = 0) {
    const p2s_problem c = pb.c();
    check(p2s_direct_create(&c, device, &h_));
  }
  ~DirectContext() {
    if (h_) p2s_direct_destroy(h_);
  }
  DirectContext(const DirectContext&) = delete;
  DirectContext& operator=(const DirectContext&) = delete;
  void fill(const double* d_alpha, double* d_M, int64_t ld, int64_t n, void* stream = nullptr) {
    check(p2s_direct_fill(h_, d_alpha, d_M, ld, n, stream));
  }

 private:
  p2s_direct_ctx* h_ = nullptr;
};

// Moment integrals of a batch of elements (reference: KernelTable, assembly.hpp:35-40).
// Counters as the reference's (assembly.cpp:291-310): n_integrals = moment
// entries computed (one tensor quadrature each), n_mass_uu_integrals = those of
// the mass term (term 0) of the (0, 0) component pair -- the Kuu table's count.
struct KernelTable {
  Problem problem;
  int64_t n_elem = 0;
  std::vector<double> I;   // [n_elem][moments_per_elem]
  long n_integrals = 0;
  long n_mass_uu_integrals = 0;
};

// Element matrices of a batch (reference: ElementMatrices, assembly.hpp:20-26);
// matrix e occupies M[e * n_tot * n_tot ...], row-major.  The counters are the
// kernel tables' (set by fill_elements like fill_one, assembly.cpp:665-666).
struct ElementMatrices {
  Problem problem;
  int64_t n_elem = 0;
  int n_tot = 0;
  std::vector<double> M;
  long n_integrals = 0;
  long n_mass_uu_integrals = 0;
  double operator()(int64_t e, int i, int j) const {
    return M[static_cast<size_t>((e * n_tot + i) * n_tot + j)];
  }
};

// moment entries per element, all terms and pairs / the mass term of pair (0, 0)
inline void integral_counts(const p2s_sizes& sz, int n_terms, long* all, long* mass_uu) {
  long per = 0;
  for (int s = 0; s < n_terms; ++s) per += static_cast<long>(sz.K[s][0]) * sz.K[s][1] * sz.K[s][2];
  *all = per * sz.n_pairs;
  *mass_uu = static_cast<long>(sz.K[0][0]) * sz.K[0][1] * sz.K[0][2];
}

inline KernelTable compute_kernel_tables(Context& ctx, const std::vector<double>& alpha) {
  if (alpha.size() % static_cast<size_t>(ctx.alpha_per_elem()) != 0)
    throw std::invalid_argument("compute_kernel_tables: alpha size is not a whole number of elements");
  KernelTable kt;
  kt.problem = ctx.problem();
  kt.n_elem = static_cast<int64_t>(alpha.size()) / ctx.alpha_per_elem();
  kt.I.assign(static_cast<size_t>(kt.n_elem * ctx.moments_per_elem()), 0.0);
  check(p2s_moments_host(ctx.handle(), alpha.data(), kt.I.data(), kt.n_elem));
  long all = 0, muu = 0;
  integral_counts(ctx.sizes(), static_cast<int>(kt.problem.terms.size()), &all, &muu);
  kt.n_integrals = all * kt.n_elem;
  kt.n_mass_uu_integrals = muu * kt.n_elem;
  return kt;
}

inline ElementMatrices assemble_p2s_element(Context& ctx, const KernelTable& kt) {
  if (!kt.problem.same_shape(ctx.problem()))
    throw std::invalid_argument("assemble_p2s_element: kernel table was built for other orders");
  ElementMatrices em;
  em.problem = ctx.problem();
  em.n_elem = kt.n_elem;
  em.n_tot = ctx.n_tot();
  em.M.assign(static_cast<size_t>(em.n_elem) * em.n_tot * em.n_tot, 0.0);
  check(p2s_contract_host(ctx.handle(), kt.I.data(), em.M.data(), em.n_tot, em.n_elem));
  em.n_integrals = kt.n_integrals;
  em.n_mass_uu_integrals = kt.n_mass_uu_integrals;
  return em;
}

// Partition of n elements over g workers: worker w owns [n w / g, n (w+1) / g).
inline std::pair<int64_t, int64_t> element_range(int64_t n, int w, int g) {
  return {n * w / g, n * (w + 1) / g};
}

// Batch fill on `gpus` devices: contiguous element ranges, one host thread
// (and one context) per GPU, first exception rethrown after all workers joined;
// the result is independent of the GPU count (elements are independent).
inline ElementMatrices fill_elements(const Problem& pb, const std::vector<double>& alpha, int gpus = 1) {
  if (gpus < 1) throw std::invalid_argument("fill_elements: gpus must be >= 1");
  const p2s_problem cp = pb.c();
  p2s_sizes sz{};
  check(p2s_problem_sizes(&cp, &sz));  // no device, no context
  const int64_t ape = sz.alpha_per_elem;
  if (alpha.size() % static_cast<size_t>(ape) != 0)
    throw std::invalid_argument("fill_elements: alpha size is not a whole number of elements");
  ElementMatrices em;
  em.problem = pb;
  em.n_elem = static_cast<int64_t>(alpha.size()) / ape;
  em.n_tot = sz.n_tot;
  long all = 0, muu = 0;
  integral_counts(sz, cp.n_terms, &all, &muu);
  em.n_integrals = all * em.n_elem;
  em.n_mass_uu_integrals = muu * em.n_elem;
  const int64_t mel = static_cast<int64_t>(em.n_tot) * em.n_tot;
  em.M.assign(static_cast<size_t>(em.n_elem * mel), 0.0);
  if (em.n_elem == 0) return em;
  if (gpus == 1 || em.n_elem <= 1) {
    Context ctx(pb, 0);
    check(p2s_fill_host(ctx.handle(), alpha.data(), em.M.data(), em.n_tot, em.n_elem));
    return em;
  }
  std::exception_ptr error;
  std::mutex error_mutex;
  std::vector<std::thread> pool;
  for (int g = 0; g < gpus; ++g) {
    pool.emplace_back([&, g] {
      try {
        const auto r = element_range(em.n_elem, g, gpus);
        const int64_t e0 = r.first, e1 = r.second;
        if (e1 <= e0) return;
        Context ctx(pb, g);
        check(p2s_fill_host(ctx.handle(), alpha.data() + e0 * ape, em.M.data() + e0 * mel, em.n_tot,
                            e1 - e0));
      } catch (...) {
        std::lock_guard<std::mutex> lock(error_mutex);
        if (!error) error = std::current_exception();
      }
    });
  }
  for (std::thread& t : pool) t.join();
  if (error) std::rethrow_exception(error);
  return em;
}

}  // namespace p2s
