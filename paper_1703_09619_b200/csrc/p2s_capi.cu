// p2s_capi.cu -- C-ABI (include/p2s_b200.h): context, kernel registry and the
// element-batch scheduler.  The scheduler replaces fill_elements
// (assembly.cpp:654-700): elements are processed in chunks whose moment
// scratch stays L2-resident; p2s_fill_host pipelines H2D / fill / D2H over a
// two-slot device ring on three streams.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/p2s_b200.h"
#include "p2s_jit.hpp"
#include "p2s_launch.cuh"
#include "p2s_registry.hpp"
#include "p2s_tables.hpp"

namespace p2s {
cudaError_t launch_geometry(double* geom, double lo, double hi, uint64_t seed, int64_t e0, int64_t n,
                            cudaStream_t stream);
cudaError_t launch_alpha_geometry_fast(double* alpha, const double* geom, const double* const x[3],
                                       const int nq[3], int nc, int S, int64_t n, int64_t per_elem,
                                       int* bad, cudaStream_t stream);
cudaError_t launch_alpha(double* alpha, const double* const x[3], const int nq[3], int nc, int S,
                         int kind, double lo, double hi, uint64_t seed, int64_t e0, int64_t n,
                         int64_t per_elem, cudaStream_t stream);
}

namespace {

thread_local std::string g_last_error;

p2s_status fail(p2s_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

p2s_status cuda_fail(cudaError_t err, const char* where) {
  return fail(P2S_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(err));
}

#define P2S_CUDA(call)                                   \
  do {                                                   \
    cudaError_t err__ = (call);                          \
    if (err__ != cudaSuccess) return cuda_fail(err__, #call); \
  } while (0)

using namespace p2s;
using namespace p2s::reg;

// ------------------------------------------------------------ options
// Test and tuning hooks, passed explicitly to p2s_create_ex as "KEY=VALUE"
// pairs (';' / ',' / whitespace separated).  The production library never
// reads them from the environment (a tuning build, -DP2S_TUNING, falls back to
// environment variables of the same names for the sweep scripts in tools/).
const char* const kOptionKeys[] = {
    "P2S_NO_FUSED",         // 1: two-stage path even where a fused kernel exists
    "P2S_FUSED_VARIANT",    // k: the k-th registered fused variant of the shape
    "P2S_V2_VARIANT",       // k: the k-th registered contract_v2 variant
    "P2S_MV2_VARIANT",      // k: the k-th registered moments_v2 variant
    "P2S_FORCE_GENERIC",    // 1: runtime-shaped generic kernels (where compiled)
    "P2S_JIT",              // 0: never use a generated module
    "P2S_FORCE_JIT",        // 1: a generated module even for registered shapes
    "P2S_JIT_FAMILY",       // planner overrides: fused / large
    "P2S_JIT_T", "P2S_JIT_FLAGS", "P2S_JIT_FPT", "P2S_JIT_MINB", "P2S_JIT_THREADS", "P2S_JIT_KC",
    "P2S_GEO_MODE",         // geometry fill mode 0 / 1 / 2
    "P2S_XCHUNK_MB",        // large path: intermediate chunk (MB)
    "P2S_LARGE_PS", "P2S_LARGE_OVERLAP", "P2S_LARGE_PRIO", "P2S_LARGE_USTREAMS", "P2S_LARGE_UPERSIST", "P2S_LARGE_URESERVE", "P2S_LARGE_VSPLIT",
    "P2S_LARGE_XS", "P2S_LARGE_UBULK", "P2S_LARGE_UROLL", "P2S_LARGE_UPAIR", "P2S_LARGE_MSPLIT", "P2S_LARGE_MOMCL", "P2S_LARGE_MOMG", "P2S_LARGE_MOMT", "P2S_LARGE_MOMW", "P2S_LARGE_USMEM", "P2S_LARGE_FIB",
    "P2S_CHUNK_MB",         // two-stage scheduler chunk (MB of moments)
    "P2S_TWO_STAGE_OVERLAP", "P2S_MOM_PRIO",
    "P2S_HOST_CHUNK_MB",    // p2s_fill_host ring slot (MB of matrices)
    "P2S_GEO_CHUNK_MB",     // p2s_fill_geometry alpha buffer (MB)
    "P2S_GRAPH",            // 0: large-path fills are never replayed from a CUDA graph
};

struct Options {
  std::map<std::string, std::string> kv;
  const char* get(const char* k) const {
    auto it = kv.find(k);
    if (it != kv.end()) return it->second.c_str();
    return tuning_env(k);
  }
};

bool parse_options(const char* text, Options* o, std::string* err) {
  if (!text) return true;
  std::string tok;
  auto flush = [&]() -> bool {
    if (tok.empty()) return true;
    const size_t eq = tok.find('=');
    const std::string k = tok.substr(0, eq), v = eq == std::string::npos ? "1" : tok.substr(eq + 1);
    bool known = false;
    for (const char* kk : kOptionKeys) known = known || k == kk;
    if (!known) {
      *err = "unknown option '" + k + "'";
      return false;
    }
    o->kv[k] = v;
    tok.clear();
    return true;
  };
  for (const char* p = text; *p; ++p) {
    if (*p == ';' || *p == ',' || std::isspace(static_cast<unsigned char>(*p))) {
      if (!flush()) return false;
    } else {
      tok.push_back(*p);
    }
  }
  return flush();
}

jit::Overrides overrides_of(const Options& opt) {
  jit::Overrides ov;
  auto num = [&](const char* k, int* dst) {
    if (const char* v = opt.get(k)) *dst = std::atoi(v);
  };
  if (const char* v = opt.get("P2S_JIT_FAMILY"))
    ov.family = std::string(v) == "large" ? jit::kFamilyLarge : jit::kFamilyFused;
  num("P2S_JIT_T", &ov.T);
  num("P2S_JIT_FLAGS", &ov.flags);
  num("P2S_JIT_FPT", &ov.fpt);
  num("P2S_JIT_MINB", &ov.minb);
  num("P2S_JIT_THREADS", &ov.threads);
  num("P2S_JIT_KC", &ov.kc);
  return ov;
}

// ------------------------------------------------------------ registry lookup

const RegEntry* find_entry(const p2s_problem& pb) {
  for (const RegEntry& r : registry()) {
    if (r.NU != pb.order[0] || r.S != pb.n_terms) continue;
    bool ok = true;
    for (int s = 0; s < r.S; ++s) ok = ok && (r.kinds[s] == pb.kind[s][0]);
    if (ok) return &r;
  }
  return nullptr;
}


const V2Entry* find_v2(const p2s_problem& pb, const Options& o) {
  int want = 0, seen = 0;
  if (const char* v = o.get("P2S_V2_VARIANT")) want = std::atoi(v);
  const V2Entry* first = nullptr;
  for (const V2Entry& r : v2_registry()) {
    bool ok = r.S == pb.n_terms;
    for (int d = 0; d < 3; ++d) ok = ok && r.order[d] == pb.order[d];
    for (int s = 0; ok && s < r.S; ++s)
      for (int d = 0; d < 3; ++d) ok = ok && r.kinds[s][d] == pb.kind[s][d];
    if (!ok) continue;
    if (!first) first = &r;
    if (seen++ == want) return &r;
  }
  return first;
}


const MV2Entry* find_mv2(const p2s_problem& pb, const Options& o) {
  int want = 0, seen = 0;
  if (const char* v = o.get("P2S_MV2_VARIANT")) want = std::atoi(v);
  const MV2Entry* first = nullptr;
  for (const MV2Entry& r : mv2_registry()) {
    bool ok = r.S == pb.n_terms;
    for (int d = 0; d < 3; ++d) ok = ok && r.order[d] == pb.order[d] && r.nq[d] == pb.nq[d];
    for (int s = 0; ok && s < r.S; ++s)
      for (int d = 0; d < 3; ++d) ok = ok && r.kinds[s][d] == base_kind(pb.kind[s][d]);
    if (!ok) continue;  // moments do not depend on the basis
    if (!first) first = &r;
    if (seen++ == want) return &r;
  }
  return first;
}


const FusedEntry* find_fused(const p2s_problem& pb, const Options& o) {
  if (const char* v = o.get("P2S_NO_FUSED"))
    if (v[0] == '1') return nullptr;
  int want = 0, seen = 0;
  const char* var = o.get("P2S_FUSED_VARIANT");
  if (var) want = std::atoi(var);
  const FusedEntry* first = nullptr;
  for (const FusedEntry& r : fused_registry()) {
    bool ok = r.S == pb.n_terms;
    for (int d = 0; d < 3; ++d) ok = ok && r.order[d] == pb.order[d] && r.nq[d] == pb.nq[d];
    for (int s = 0; ok && s < r.S; ++s)
      for (int d = 0; d < 3; ++d) ok = ok && r.kinds[s][d] == pb.kind[s][d];
    if (!ok) continue;
    if (!first) {
      if (r.prefer_two_stage && !var) return nullptr;
      first = &r;
    }
    if (seen++ == want) return &r;
  }
  return first;
}


const LargeEntry* find_large(const p2s_problem& pb) {
  for (const LargeEntry& r : large_registry()) {
    bool ok = r.S == pb.n_terms;
    for (int d = 0; d < 3; ++d) ok = ok && r.order[d] == pb.order[d] && r.nq[d] == pb.nq[d];
    for (int s = 0; ok && s < r.S; ++s)
      for (int d = 0; d < 3; ++d) ok = ok && r.kinds[s][d] == pb.kind[s][d];
    if (ok) return &r;
  }
  return nullptr;
}


}  // namespace

// ------------------------------------------------------------ context

struct p2s_ctx {
  p2s_problem pb{};
  int device = 0;
  Options opt;
  const reg::JitEntries* jit = nullptr;  // generated module (shapes without a registered kernel)
  std::string jit_desc;
  p2s_sizes sz{};
  std::vector<double> x[3], w[3];
  std::vector<double> phi[kMaxTerms][3];   // [K][nq]
  std::vector<double> coef[kMaxTerms][3];  // [N][N][K]
  int Kpad[kMaxTerms][3]{};
  double* d_phiT[kMaxTerms][3]{};          // [nq][Kpad]
  double* d_coef[kMaxTerms][3]{};          // [N][N][K]
  double* d_x[3]{};
  const RegEntry* entry = nullptr;
  const V2Entry* v2 = nullptr;
  const MV2Entry* mv2 = nullptr;
  const LargeEntry* large = nullptr;
  LargePack lpack;
  double* d_X = nullptr;
  int64_t xchunk = 1;
  const FusedEntry* fused = nullptr;
  std::vector<double> fused_cpack, fused_mpack;
  double* d_amma_fused = nullptr;  // stage-C tensor-core A (MMA shapes)
  double* d_amma_v2 = nullptr;
  std::vector<double> mv2_packed;
  std::vector<double> v2_packed;
  int num_sms = 148;
  bool force_generic = false;
  std::vector<double> cu_packed;
  Plan plan{};
  int kmax = 8;
  size_t mom_smem = 0;
  int S2 = 1, S3 = 1;
  // scheduler
  int64_t chunk = 1;
  double* d_scratch = nullptr;             // chunk * moments_per_elem
  // host pipeline
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  int64_t host_chunk = 0;
  // two-stage fill: moments of the next chunk on s_mom (double-buffered scratch)
  cudaStream_t s_mom = nullptr;
  cudaEvent_t ev_fill_start = nullptr, ev_mom_done[2]{}, ev_con_done[2]{};
  double* d_ring_alpha[2]{};
  double* d_ring_M[2]{};
  cudaEvent_t ev_h2d[2]{}, ev_comp[2]{}, ev_d2h[2]{};
  // geometry fill: alpha of a chunk of elements generated into an L2-sized
  // double buffer on s_geo while the fill consumes the other buffer
  int64_t geo_chunk = 0;
  int geo_mode = 0;  // P2S_GEO_MODE: 0 alpha via the L2 double buffer (default, fastest);
                     // 1 per-unit recomputation inside the fused kernel; 2 one cluster per
                     // element sharing the per-point geometry through DSMEM
  double* d_geo_alpha[2]{};
  int* d_bad = nullptr;  // non-positive Jacobian flag of the geometry entry points
  int* h_bad = nullptr;  // (pinned host copy)
  cudaStream_t s_geo = nullptr;
  cudaEvent_t ev_geo_start = nullptr, ev_ga[2]{}, ev_gf[2]{};
  // context scratch (two-stage moment buffers, large-path X / Z, host ring,
  // geometry buffers): calls that use it are ordered on the device through
  // ev_scratch whatever stream they come on; scratch_mu orders the host side
  std::mutex scratch_mu;
  cudaEvent_t ev_scratch = nullptr;
  // large path: the launch sequence of a fill (hundreds of short w / v / u kernels
  // with up to 30 KB of parameters each, ordered by events over three streams)
  // costs the host about as long as the GPU needs to run it (c12: 9.4 ms of launch
  // code for 10.6 ms of device time).  A fill that comes back with the same buffers
  // is captured once into a CUDA graph and replayed (P2S_GRAPH=0: never).
  struct FillGraph {
    const double* alpha;
    double* M;
    int64_t ldM, n;
    cudaGraphExec_t exec;  // null until the second call with this key
    bool failed;           // capture / instantiation failed once: direct launches
    uint64_t stamp;
  };
  std::vector<FillGraph> graphs;
  cudaStream_t s_cap = nullptr;  // capture origin (the caller's stream may be the legacy stream)
  uint64_t graph_clock = 0;
  bool use_graphs = true;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_mom, ev_con;
  double ms_mom = 0.0, ms_con = 0.0;
  int64_t n_mom = 0, n_con = 0, n_fused = 0;
};

namespace {

cudaEvent_t take_event(p2s_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void harvest(p2s_ctx* c) {
  for (auto& pr : c->ev_mom) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    c->ms_mom += ms;
    c->ev_pool.push_back(pr.first);
    c->ev_pool.push_back(pr.second);
  }
  for (auto& pr : c->ev_con) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    c->ms_con += ms;
    c->ev_pool.push_back(pr.first);
    c->ev_pool.push_back(pr.second);
  }
  c->ev_mom.clear();
  c->ev_con.clear();
}

p2s_status validate(const p2s_problem* pb) {
  if (!pb) return fail(P2S_INVALID_ARG, "p2s_create: null problem");
  if (pb->n_comp < 1 || pb->n_comp > 3) return fail(P2S_INVALID_ARG, "n_comp must be 1..3");
  if (pb->n_terms < 1 || pb->n_terms > P2S_MAX_TERMS)
    return fail(P2S_INVALID_ARG, "n_terms must be 1..4");
  for (int d = 0; d < 3; ++d) {
    if (pb->order[d] < 1 || pb->order[d] > 32) return fail(P2S_INVALID_ARG, "order must be 1..32");
    if (pb->nq[d] < 1 || pb->nq[d] > 64) return fail(P2S_INVALID_ARG, "nq must be 1..64");
  }
  for (int s = 0; s < pb->n_terms; ++s)
    for (int d = 0; d < 3; ++d)
      if (pb->kind[s][d] < 0 || pb->kind[s][d] > 3) return fail(P2S_INVALID_ARG, "bad kind");
  if (pb->basis != P2S_BASIS_MODAL && pb->basis != P2S_BASIS_CONFORMING)
    return fail(P2S_INVALID_ARG, "basis must be P2S_BASIS_MODAL or P2S_BASIS_CONFORMING");
  if (pb->basis == P2S_BASIS_CONFORMING)
    for (int d = 0; d < 3; ++d)
      if (pb->order[d] < 2)  // conforming_matrix needs degree >= 1 (assembly.cpp:478)
        return fail(P2S_INVALID_ARG, "conforming basis needs order >= 2 in every direction");
  return P2S_OK;
}

// internal problem: the basis travels as bit 2 of every kind
p2s_problem effective(const p2s_problem& pb) {
  p2s_problem e = pb;
  if (pb.basis == P2S_BASIS_CONFORMING)
    for (int s = 0; s < pb.n_terms; ++s)
      for (int d = 0; d < 3; ++d) e.kind[s][d] |= kConforming;
  return e;
}

p2s_status run_moments(p2s_ctx* c, const double* alpha, double* I, int64_t n, cudaStream_t st) {
  MomentParams p;
  std::memset(&p, 0, sizeof(p));
  p.alpha = alpha;
  p.I = I;
  p.P = c->sz.n_pairs;
  p.S = c->pb.n_terms;
  p.n_units = n * p.P * p.S;
  for (int d = 0; d < 3; ++d) p.nq[d] = c->pb.nq[d];
  for (int s = 0; s < p.S; ++s)
    for (int d = 0; d < 3; ++d) {
      p.K[s][d] = c->sz.K[s][d];
      p.Kpad[s][d] = c->Kpad[s][d];
      p.phiT[s][d] = c->d_phiT[s][d];
    }
  p.mom_per_elem = c->sz.moments_per_elem;
  p.mom_per_pair = c->sz.moments_per_pair;
  for (int s = 0; s < p.S; ++s) p.mom_off[s] = c->sz.moment_offset[s];
  p.S2 = c->S2;
  p.S3 = c->S3;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof) {
    e0 = take_event(c);
    e1 = take_event(c);
    cudaEventRecord(e0, st);
  }
  cudaError_t err;
  if (c->large)
    err = c->large->moments(alpha, I, n * p.P, c->lpack, st);
  else if (c->mv2 && !c->force_generic)
    err = c->mv2->launch(alpha, I, n, p.P, p.mom_per_elem, c->mv2_packed, st);
  else
    err = launch_moments(c->kmax, p, c->mom_smem, st);
  if (err != cudaSuccess) return cuda_fail(err, "moments_kernel launch");
  if (c->prof) {
    cudaEventRecord(e1, st);
    c->ev_mom.emplace_back(e0, e1);
    ++c->n_mom;
  }
  return P2S_OK;
}

p2s_status run_contract(p2s_ctx* c, const double* I, double* M, int64_t ldM, int64_t n,
                        cudaStream_t st) {
  ContractArgs a;
  std::memset(&a, 0, sizeof(a));
  a.I = I;
  a.M = M;
  a.ldM = ldM;
  a.n_tot = c->sz.n_tot;
  a.n_elem = n;
  a.nc = c->pb.n_comp;
  a.P = c->sz.n_pairs;
  a.Nv = c->pb.order[1];
  a.Nw = c->pb.order[2];
  a.Nt = c->pb.order[0] * c->pb.order[1] * c->pb.order[2];
  a.S = c->pb.n_terms;
  for (int s = 0; s < a.S; ++s) {
    a.Kv[s] = c->sz.K[s][1];
    a.Kw[s] = c->sz.K[s][2];
    a.kind_v[s] = c->pb.kind[s][1];
    a.kind_w[s] = c->pb.kind[s][2];
    a.mom_off[s] = c->sz.moment_offset[s];
    a.Cv[s] = c->d_coef[s][1];
    a.Cw[s] = c->d_coef[s][2];
  }
  a.mom_per_elem = c->sz.moments_per_elem;
  a.mom_per_pair = c->sz.moments_per_pair;
  a.cu_packed = c->cu_packed.data();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof) {
    e0 = take_event(c);
    e1 = take_event(c);
    cudaEventRecord(e0, st);
  }
  cudaError_t err;
  if (c->large) {
    err = c->large->contract(I, c->d_X, M, n * c->sz.n_pairs, c->xchunk, ldM, c->pb.n_comp,
                             c->sz.n_pairs, a.Nt, c->lpack, st);
  } else if (c->v2 && !c->force_generic) {
    V2Args v;
    v.I = I;
    v.M = M;
    v.ldM = ldM;
    v.n_tot = c->sz.n_tot;
    v.n_elem = n;
    v.mom_per_elem = c->sz.moments_per_elem;
    v.nc = c->pb.n_comp;
    v.P = c->sz.n_pairs;
    v.Nt = a.Nt;
    v.amma = c->d_amma_v2;
    err = c->v2->launch(v, c->v2_packed, st, c->num_sms);
  } else {
    err = c->entry->launch(a, c->plan, st);
  }
  if (err != cudaSuccess) return cuda_fail(err, "contract_kernel launch");
  if (c->prof) {
    cudaEventRecord(e1, st);
    c->ev_con.emplace_back(e0, e1);
    ++c->n_con;
  }
  return P2S_OK;
}

p2s_status run_fill(p2s_ctx* c, const double* alpha, double* M, int64_t ldM, int64_t n,
                    cudaStream_t st) {
  if (c->fused) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->prof) {
      e0 = take_event(c);
      e1 = take_event(c);
      cudaEventRecord(e0, st);
    }
    cudaError_t err = c->fused->launch(alpha, M, ldM, c->sz.n_tot, n, c->pb.n_comp, c->sz.n_pairs,
                                       c->pb.order[0] * c->pb.order[1] * c->pb.order[2],
                                       c->fused_cpack, c->fused_mpack, c->d_amma_fused, st,
                                       c->num_sms, nullptr);
    if (err != cudaSuccess) return cuda_fail(err, "fill_fused_kernel launch");
    if (c->prof) {
      cudaEventRecord(e1, st);
      c->ev_con.emplace_back(e0, e1);
      ++c->n_con;
      ++c->n_fused;
    }
    return P2S_OK;
  }
  const int64_t ape = c->sz.alpha_per_elem;
  const int64_t mstride = static_cast<int64_t>(c->sz.n_tot) * ldM;
  if (c->large || !c->s_mom) {  // serial (the large path overlaps inside its contraction)
    for (int64_t e0 = 0; e0 < n; e0 += c->chunk) {
      const int64_t cnt = std::min(c->chunk, n - e0);
      p2s_status s1 = run_moments(c, alpha + e0 * ape, c->d_scratch, cnt, st);
      if (s1 != P2S_OK) return s1;
      p2s_status s2 = run_contract(c, c->d_scratch, M + e0 * mstride, ldM, cnt, st);
      if (s2 != P2S_OK) return s2;
    }
    return P2S_OK;
  }
  // two-stage path, double-buffered moment scratch: the moments of chunk i+1 run
  // on s_mom while the (store-bound) contraction of chunk i runs on the caller's
  // stream; chunk i+2's moments wait for chunk i's contraction (buffer reuse)
  P2S_CUDA(cudaEventRecord(c->ev_fill_start, st));
  P2S_CUDA(cudaStreamWaitEvent(c->s_mom, c->ev_fill_start, 0));
  int64_t i = 0;
  for (int64_t e0 = 0; e0 < n; e0 += c->chunk, ++i) {
    const int64_t cnt = std::min(c->chunk, n - e0);
    const int b = static_cast<int>(i & 1);
    double* I = c->d_scratch + b * c->sz.moments_per_elem * c->chunk;
    if (i >= 2) P2S_CUDA(cudaStreamWaitEvent(c->s_mom, c->ev_con_done[b], 0));
    p2s_status s1 = run_moments(c, alpha + e0 * ape, I, cnt, c->s_mom);
    if (s1 != P2S_OK) return s1;
    P2S_CUDA(cudaEventRecord(c->ev_mom_done[b], c->s_mom));
    P2S_CUDA(cudaStreamWaitEvent(st, c->ev_mom_done[b], 0));
    p2s_status s2 = run_contract(c, I, M + e0 * mstride, ldM, cnt, st);
    if (s2 != P2S_OK) return s2;
    P2S_CUDA(cudaEventRecord(c->ev_con_done[b], st));
  }
  return P2S_OK;
}

// Large path: run_fill through a cached CUDA graph.  First call with a key
// (alpha, M, ld_M, n): direct launches (this also performs every per-kernel
// attribute / occupancy call, which must not happen while capturing); second
// call: the same launch code runs on the capture stream s_cap, the graph is
// instantiated and launched into the caller's stream; later calls: one
// cudaGraphLaunch.  At most 4 graphs per context (least recently used out).
p2s_status run_fill_graphed(p2s_ctx* c, const double* alpha, double* M, int64_t ldM, int64_t n,
                            cudaStream_t st) {
  constexpr size_t kMaxGraphs = 4;
  constexpr int64_t kMaxChunks = 1500;  // ~3 kernel nodes each; beyond that graphs cost too much memory
  const int64_t chunks = c->xchunk > 0 ? (n * c->sz.n_pairs + c->xchunk - 1) / c->xchunk : 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!c->use_graphs || n == 0 || chunks < 2 || chunks > kMaxChunks ||
      cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return run_fill(c, alpha, M, ldM, n, st);
  }
  p2s_ctx::FillGraph* g = nullptr;
  for (auto& e : c->graphs)
    if (e.alpha == alpha && e.M == M && e.ldM == ldM && e.n == n) g = &e;
  if (!g) {  // first sight: remember the key, launch directly
    if (c->graphs.size() >= kMaxGraphs) {
      size_t old = 0;
      for (size_t i = 1; i < c->graphs.size(); ++i)
        if (c->graphs[i].stamp < c->graphs[old].stamp) old = i;
      if (c->graphs[old].exec) cudaGraphExecDestroy(c->graphs[old].exec);
      c->graphs.erase(c->graphs.begin() + static_cast<std::ptrdiff_t>(old));
    }
    c->graphs.push_back({alpha, M, ldM, n, nullptr, false, ++c->graph_clock});
    return run_fill(c, alpha, M, ldM, n, st);
  }
  g->stamp = ++c->graph_clock;
  if (g->failed) return run_fill(c, alpha, M, ldM, n, st);
  if (!g->exec) {
    if (!c->s_cap && cudaStreamCreateWithFlags(&c->s_cap, cudaStreamNonBlocking) != cudaSuccess) {
      g->failed = true;
      cudaGetLastError();
      return run_fill(c, alpha, M, ldM, n, st);
    }
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(c->s_cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      const std::string saved = g_last_error;
      const bool prof = c->prof;
      c->prof = false;  // no timing events inside the graph
      ok = run_fill(c, alpha, M, ldM, n, c->s_cap) == P2S_OK;
      c->prof = prof;
      ok = (cudaStreamEndCapture(c->s_cap, &graph) == cudaSuccess) && ok && graph != nullptr;
      if (!ok) g_last_error = saved;
    }
    if (ok) ok = cudaGraphInstantiate(&g->exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
      g->exec = nullptr;
      g->failed = true;
      cudaGetLastError();  // a failed capture is not an error of this call
      return run_fill(c, alpha, M, ldM, n, st);
    }
  }
  // profiling: one event pair around the whole replayed fill (moments included),
  // reported as the contraction stage
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof) {
    e0 = take_event(c);
    e1 = take_event(c);
    cudaEventRecord(e0, st);
  }
  P2S_CUDA(cudaGraphLaunch(g->exec, st));
  if (c->prof) {
    cudaEventRecord(e1, st);
    c->ev_con.emplace_back(e0, e1);
    ++c->n_con;
  }
  return P2S_OK;
}

// buffer sizes and moment layout of a problem (basis-independent)
void problem_sizes(const p2s_problem& pb, p2s_sizes* sz) {
  *sz = p2s_sizes{};
  const int S = pb.n_terms, nc = pb.n_comp;
  sz->n_pairs = nc * nc;
  sz->n_tot = nc * pb.order[0] * pb.order[1] * pb.order[2];
  sz->alpha_per_elem = static_cast<int64_t>(sz->n_pairs) * S * pb.nq[0] * pb.nq[1] * pb.nq[2];
  int64_t off = 0;
  for (int s = 0; s < S; ++s) {
    sz->moment_offset[s] = off;
    int64_t kk = 1;
    for (int d = 0; d < 3; ++d) {
      const int K = kernel_count(pb.kind[s][d], pb.order[d]);
      sz->K[s][d] = K;
      kk *= K;
    }
    off += kk;
  }
  sz->moments_per_pair = (off + 3) & ~int64_t(3);
  sz->moments_per_elem = sz->moments_per_pair * sz->n_pairs;
}

// Held for a call that uses context scratch: the call's stream first waits
// for the previous such call (any stream), and the release records the event
// on it, so concurrent callers never share the buffers.
class ScratchUse {
 public:
  ScratchUse(p2s_ctx* c, cudaStream_t st) : c_(c), st_(st), lock_(c->scratch_mu) {
    ok_ = cudaStreamWaitEvent(st_, c_->ev_scratch, 0) == cudaSuccess;
  }
  ~ScratchUse() { cudaEventRecord(c_->ev_scratch, st_); }
  bool ok() const { return ok_; }

 private:
  p2s_ctx* c_;
  cudaStream_t st_;
  std::lock_guard<std::mutex> lock_;
  bool ok_ = false;
};

// Alpha rows are read with 32-B loads (ld.global.nc.v4.f64) when nq_u % 4 == 0,
// else with 16-B loads / 16-B bulk prefetches
int alpha_align(const p2s_ctx* c) { return c->pb.nq[0] % 4 == 0 ? 32 : 16; }

p2s_status check_ctx(const p2s_ctx* c) {
  if (!c) return fail(P2S_INVALID_ARG, "null context");
  return P2S_OK;
}

}  // namespace

p2s_status p2s_internal_fail(p2s_status st, const std::string& msg) { return fail(st, msg); }

extern "C" {

const char* p2s_last_error(void) { return g_last_error.c_str(); }

const char* p2s_version(void) { return "p2s_b200 0.2 (sm_100a)"; }

const char* p2s_jit_cache_dir(void) {
  static thread_local std::string d;
  d = jit::cache_dir();
  return d.c_str();
}

const char* p2s_kernel_path(const p2s_ctx* c) {
  if (!c) return "";
  static thread_local std::string path;
  if (c->large) {
    path = std::string("large-order: ") +
           (c->lpack.mom_wfirst ? "large_moments_w_kernel" : "large_moments_kernel") +
           " + large_w_kernel + large_v_kernel + large_u_kernel";
  } else if (c->fused) {
    path = std::string("fused: fill_fused_kernel (moments + contraction; ") + c->fused->desc + ")";
  } else if (c->v2 && !c->force_generic) {
    path = std::string(c->mv2 ? "two-stage: moments_v2_kernel + contract_v2_kernel ("
                              : "two-stage: moments_kernel + contract_v2_kernel (") +
           c->v2->desc + ")";
  } else {
    path = c->mv2 && !c->force_generic ? "two-stage: moments_v2_kernel + contract_kernel"
                                       : "two-stage: moments_kernel + contract_kernel (generic)";
  }
  if (c->jit) path += " [generated module: " + c->jit_desc + "]";
  return path.c_str();
}

int p2s_shape_supported(const p2s_problem* spec_in) {
  if (!spec_in || validate(spec_in) != P2S_OK) return 0;
  const p2s_problem eff = effective(*spec_in);
  if (find_v2(eff, Options{}) != nullptr || find_large(eff) != nullptr) return 1;
  jit::Plan pl;
  std::string why;
  if (jit::plan(eff, &pl, &why) && (jit::cached(pl) || jit::compiler_available())) return 1;
  return find_entry(eff) != nullptr;
}

p2s_status p2s_create(const p2s_problem* spec_in, int device, p2s_ctx** out) {
  return p2s_create_ex(spec_in, device, nullptr, out);
}

p2s_status p2s_shape_prepare(const p2s_problem* spec_in, const char* options, char* desc, int desc_len) {
  p2s_status st = validate(spec_in);
  if (st != P2S_OK) return st;
  Options opt;
  {
    std::string err;
    if (!parse_options(options, &opt, &err)) return fail(P2S_INVALID_ARG, "p2s_shape_prepare: " + err);
  }
  const bool force_jit = opt.get("P2S_FORCE_JIT") && opt.get("P2S_FORCE_JIT")[0] == '1';
  const p2s_problem eff = effective(*spec_in);
  std::string d;
  if (!force_jit && (find_v2(eff, opt) || find_large(eff))) {
    d = "registered (ahead of time)";
  } else {
    jit::Plan pl;
    std::string why;
    if (!jit::plan(eff, &pl, &why, overrides_of(opt)))
      return fail(P2S_UNSUPPORTED_SHAPE, "p2s_shape_prepare: " + why);
    if (!jit::module(pl, &why)) return fail(P2S_UNSUPPORTED_SHAPE, "p2s_shape_prepare: " + why);
    d = pl.desc + " | " + jit::module_path(pl);
  }
  if (desc && desc_len > 0) {
    std::strncpy(desc, d.c_str(), static_cast<size_t>(desc_len) - 1);
    desc[desc_len - 1] = '\0';
  }
  return P2S_OK;
}

p2s_status p2s_create_ex(const p2s_problem* spec_in, int device, const char* options, p2s_ctx** out) {
  if (!out) return fail(P2S_INVALID_ARG, "p2s_create: null out");
  *out = nullptr;
  p2s_status st = validate(spec_in);
  if (st != P2S_OK) return st;
  Options opt;
  {
    std::string err;
    if (!parse_options(options, &opt, &err)) return fail(P2S_INVALID_ARG, "p2s_create_ex: " + err);
  }
  const p2s_problem eff = effective(*spec_in);
  const p2s_problem* spec = &eff;
  auto flag = [&](const char* k) {
    const char* v = opt.get(k);
    return v && v[0] == '1';
  };
  const bool force_jit = flag("P2S_FORCE_JIT");
  const bool no_jit = [&] {
    const char* v = opt.get("P2S_JIT");
    return v && v[0] == '0';
  }();
  const RegEntry* entry = find_entry(*spec);
  const V2Entry* v2e = force_jit ? nullptr : find_v2(*spec, opt);
  const LargeEntry* lge = force_jit ? nullptr : find_large(*spec);
  const FusedEntry* fe = force_jit ? nullptr : find_fused(*spec, opt);
  const MV2Entry* mv2e = force_jit ? nullptr : find_mv2(*spec, opt);
  const bool want_generic = flag("P2S_FORCE_GENERIC") && entry;
  // a registered contraction whose moment kernel is registered for other nq
  // would pair with the runtime-shaped moments_kernel (0.18-0.69 of HBM on the
  // coverage grid): a generated module instantiates both for this shape instead
  if (v2e && !mv2e && !fe && !no_jit && !want_generic && !opt.get("P2S_NO_FUSED") && !opt.get("P2S_V2_VARIANT"))
    v2e = nullptr;
  // shapes without a shape-specialised kernel: a generated module (p2s_jit.cu)
  const reg::JitEntries* je = nullptr;
  std::string jit_desc;
  if (!v2e && !lge && !want_generic && !no_jit) {
    jit::Plan pl;
    std::string why;
    if (!jit::plan(*spec, &pl, &why, overrides_of(opt))) {
      if (!entry) return fail(P2S_UNSUPPORTED_SHAPE, "p2s_create: " + why);
    } else {
      je = jit::module(pl, &why);
      if (!je && !entry) return fail(P2S_UNSUPPORTED_SHAPE, "p2s_create: generated module: " + why);
      if (je && static_cast<int64_t>(je->smem) != pl.smem)
        return fail(P2S_CUDA_ERROR, "p2s_create: generated module layout differs from the plan (" +
                                        std::to_string(je->smem) + " vs " + std::to_string(pl.smem) + " B)");
      jit_desc = pl.desc;
    }
  }
  if (je) {
    if (je->family == jit::kFamilyFused) {
      v2e = &je->v2;
      mv2e = &je->mv2;
      fe = opt.get("P2S_NO_FUSED") && opt.get("P2S_NO_FUSED")[0] == '1' ? nullptr : &je->fused;
    } else {
      lge = &je->large;
      fe = nullptr;
      mv2e = nullptr;
    }
  }
  if (!entry && !v2e && !lge)
    return fail(P2S_UNSUPPORTED_SHAPE, "p2s_create: no kernel for N_u=" + std::to_string(spec->order[0]) +
                                           " with these u-kinds");
  int ndev = 0;
  cudaError_t err = cudaGetDeviceCount(&ndev);
  if (err != cudaSuccess || ndev == 0)
    return fail(P2S_CUDA_ERROR, "p2s_create: no CUDA device (the fill has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(P2S_INVALID_ARG, "p2s_create: bad device");
  P2S_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  P2S_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(P2S_CUDA_ERROR, std::string("p2s_create: built for sm_100a, device is ") + prop.name);

  // every early return below releases what was allocated so far
  std::unique_ptr<p2s_ctx, void (*)(p2s_ctx*)> c(new p2s_ctx, &p2s_destroy);
  P2S_CUDA(cudaEventCreateWithFlags(&c->ev_scratch, cudaEventDisableTiming));
  c->pb = *spec;
  c->device = device;
  c->opt = opt;
  c->jit = je;
  c->jit_desc = jit_desc;
  c->entry = entry;
  c->v2 = v2e;
  c->num_sms = prop.multiProcessorCount;
  c->force_generic = want_generic;
  const int S = spec->n_terms;
  problem_sizes(*spec, &c->sz);
  int kmax = 1;
  for (int s = 0; s < S; ++s)
    for (int d = 0; d < 3; ++d) kmax = std::max(kmax, c->sz.K[s][d]);
  c->kmax = kmax <= 8 ? 8 : kmax <= 12 ? 12 : kmax <= 16 ? 16 : kmax <= 20 ? 20 : kmax <= 24 ? 24 : 32;
  if (kmax > 32 && !lge && !mv2e)  // the runtime-shaped moments_kernel holds <= 32 per direction
    return fail(P2S_UNSUPPORTED_SHAPE, "kernel count above 32");

  // tables
  for (int d = 0; d < 3; ++d) {
    gauss_legendre_ld(spec->nq[d], c->x[d], c->w[d]);
    P2S_CUDA(cudaMalloc(&c->d_x[d], sizeof(double) * spec->nq[d]));
    P2S_CUDA(cudaMemcpy(c->d_x[d], c->x[d].data(), sizeof(double) * spec->nq[d],
                        cudaMemcpyHostToDevice));
  }
  for (int s = 0; s < S; ++s)
    for (int d = 0; d < 3; ++d) {
      const int K = c->sz.K[s][d], nq = spec->nq[d];
      c->phi[s][d] = weighted_kernel_table(K, c->x[d], c->w[d]);
      c->coef[s][d] = product_to_sum_table(spec->kind[s][d], spec->order[d]);
      const int Kp = (K + 1) & ~1;
      c->Kpad[s][d] = Kp;
      std::vector<double> T(static_cast<size_t>(nq) * Kp, 0.0);
      for (int k = 0; k < K; ++k)
        for (int q = 0; q < nq; ++q) T[static_cast<size_t>(q) * Kp + k] = c->phi[s][d][static_cast<size_t>(k) * nq + q];
      P2S_CUDA(cudaMalloc(&c->d_phiT[s][d], sizeof(double) * T.size()));
      P2S_CUDA(cudaMemcpy(c->d_phiT[s][d], T.data(), sizeof(double) * T.size(), cudaMemcpyHostToDevice));
      P2S_CUDA(cudaMalloc(&c->d_coef[s][d], sizeof(double) * c->coef[s][d].size()));
      P2S_CUDA(cudaMemcpy(c->d_coef[s][d], c->coef[s][d].data(), sizeof(double) * c->coef[s][d].size(),
                          cudaMemcpyHostToDevice));
    }
  std::vector<const std::vector<double>*> dense;
  for (int s = 0; s < S; ++s) dense.push_back(&c->coef[s][0]);
  if (entry) c->cu_packed = entry->pack(dense);
  c->fused = fe;
  if (c->fused) {
    V2Args v{};
    for (int s = 0; s < S; ++s)
      for (int d = 0; d < 3; ++d) v.dense[s][d] = &c->coef[s][d];
    c->fused_cpack = c->fused->cpack(v);
    c->fused_mpack = c->fused->mpack(c->phi);
    const std::vector<double> A = c->fused->mma_pack(v);
    if (!A.empty()) {
      P2S_CUDA(cudaMalloc(&c->d_amma_fused, sizeof(double) * A.size()));
      P2S_CUDA(cudaMemcpy(c->d_amma_fused, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice));
    }
  }
  if (const char* v = opt.get("P2S_GEO_MODE")) c->geo_mode = std::atoi(v);
  c->mv2 = mv2e;
  if (c->mv2) c->mv2_packed = c->mv2->pack(c->phi);
  if (v2e) {
    V2Args v{};
    for (int s = 0; s < S; ++s)
      for (int d = 0; d < 3; ++d) v.dense[s][d] = &c->coef[s][d];
    c->v2_packed = v2e->pack(v);
    const std::vector<double> A = v2e->mma_pack(v);
    if (!A.empty()) {
      P2S_CUDA(cudaMalloc(&c->d_amma_v2, sizeof(double) * A.size()));
      P2S_CUDA(cudaMemcpy(c->d_amma_v2, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice));
    }
  }

  // moment-kernel shared memory
  c->S2 = spec->nq[1] | 1;
  c->S3 = spec->nq[2] | 1;
  size_t msm = 0;
  for (int s = 0; s < S; ++s) {
    size_t t = 0;
    for (int d = 0; d < 3; ++d) t += static_cast<size_t>(spec->nq[d]) * c->Kpad[s][d];
    t += static_cast<size_t>(c->sz.K[s][0]) * spec->nq[2] * c->S2;
    t += static_cast<size_t>(c->sz.K[s][0]) * c->sz.K[s][1] * c->S3;
    msm = std::max(msm, t);
  }
  c->mom_smem = msm * sizeof(double);
  if (!lge && !c->mv2 && c->mom_smem > 227 * 1024)
    return fail(P2S_UNSUPPORTED_SHAPE, "moment stage needs more than 227 KB of shared memory");

  // contraction plan: G n1-values per CTA, ~256 fibers per CTA
  const int Nv = spec->order[1], Nw = spec->order[2];
  const int per_n1 = Nw * Nv * Nw;
  int G = std::max(1, std::min(Nv, 256 / std::max(1, per_n1)));
  auto contract_smem = [&](int g) {
    size_t dbl = static_cast<size_t>(c->sz.moments_per_pair);
    for (int s = 0; s < S; ++s) {
      dbl += static_cast<size_t>(g) * c->sz.K[s][0] * Nv * c->sz.K[s][2] + 1;
      dbl += static_cast<size_t>(Nv) * Nv * c->sz.K[s][1] + static_cast<size_t>(Nw) * Nw * c->sz.K[s][2] + 1;
    }
    return dbl * sizeof(double) + 64;
  };
  while (G > 1 && contract_smem(G) > 227 * 1024) --G;
  c->plan.G = G;
  c->plan.NG = (Nv + G - 1) / G;
  c->plan.threads = std::min(256, ((G * per_n1 + 31) / 32) * 32);
  c->plan.smem = contract_smem(G);
  if (!v2e && !lge && c->plan.smem > 227 * 1024)
    return fail(P2S_UNSUPPORTED_SHAPE, "contraction stage needs more than 227 KB of shared memory");
  if (!lge && c->sz.moments_per_pair * 8 >= (1 << 20))
    return fail(P2S_UNSUPPORTED_SHAPE, "moment block above the bulk-copy transaction limit");
  if (lge) {
    c->large = lge;
    LargeArgs la{};
    la.phi = c->phi;
    for (int s = 0; s < S; ++s)
      for (int d = 0; d < 3; ++d) la.dense[s][d] = &c->coef[s][d];
    if (!lge->pack(la, c->lpack)) return fail(P2S_CUDA_ERROR, "p2s_create: large-path table upload");
    // X chunk: ~96 MB of v/w-contracted intermediates per buffer (two buffers: the
    // v/w stage of the next chunk overlaps the u stage of this one)
    // X chunk (units per v/u round): L2-resident (<= 32 MB, the double buffer
    // within the 126 MB L2) when that still gives the u stage >= 2.5 waves of
    // (n1, p1) tiles over 2 CTAs per SM, else >= 6 waves (amortised tails) up to
    // 96 MB.  Measured (r2j): c12 (3.95 MB / unit) 24 MB 0.60 vs 96 MB 0.53 of
    // HBM; C5 (16.7 MB / unit) 96 MB 0.65 vs 48 MB 0.59.
    // Work items per unit of the three kernels (host mirrors of LUXs / LUPlain::TPC,
    // LVRows::VR and the w step's 8-row CTAs): shapes with small N_v N_w pack several
    // (n1, p1) tiles / k1 rows into one CTA, so a chunk must hold enough units to
    // fill the GPU with CTAs of EVERY step, not only with u-stage tiles
    const int64_t tile_threads = static_cast<int64_t>(spec->order[1]) * spec->order[2];
    const int64_t tpc = tile_threads >= 128 ? 1 : (128 + tile_threads - 1) / tile_threads;
    const int64_t vthreads = static_cast<int64_t>(spec->order[2]) * spec->order[2];
    const int64_t vr = vthreads >= 128 ? 1 : (128 + vthreads - 1) / vthreads;
    int64_t kutot = 0;
    for (int s = 0; s < S; ++s) kutot += c->sz.K[s][0];
    const double u_items = static_cast<double>(tile_threads) / static_cast<double>(tpc);
    const double v_items = static_cast<double>(kutot) / static_cast<double>(vr);
    const double w_items = static_cast<double>(kutot) / 8.0 * ((spec->order[2] + 1) / 2);
    const int64_t ctas = 2 * static_cast<int64_t>(c->num_sms);
    const int64_t xbytes = lge->xpu * 8;
    auto units_for_waves = [&](double w) {  // w waves of u-stage CTAs, >= one CTA per SM in the v / w steps
      const double need = std::max(w * static_cast<double>(ctas) / u_items,
                                   0.5 * static_cast<double>(ctas) / std::min(v_items, w_items));
      return static_cast<int64_t>(std::ceil(need));
    };
    int64_t units = units_for_waves(2.5);
    if (units * xbytes > (int64_t(32) << 20))
      units = std::max<int64_t>(1, std::min(units_for_waves(6), (int64_t(96) << 20) / xbytes));
    if (const char* v = opt.get("P2S_XCHUNK_MB")) units = ((int64_t(std::max(1, std::atoi(v)))) << 20) / xbytes;
    if (const char* v = opt.get("P2S_LARGE_PS")) c->lpack.ps = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_OVERLAP")) c->lpack.overlap = v[0] != '0';
    c->xchunk = std::max<int64_t>(1, units);
    P2S_CUDA(cudaMalloc(&c->d_X, sizeof(double) * lge->xpu * c->xchunk * 2));
    P2S_CUDA(cudaMalloc(&c->lpack.d_Z, sizeof(double) * lge->zpu * c->xchunk));
    // P2S_LARGE_PRIO=1 puts the v/w steps on a high-priority stream (the block
    // scheduler then hands retiring u-stage CTA slots to v/w CTAs first); measured
    // no gain, so off by default
    int prio_lo = 0, prio_hi = 0;
    P2S_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    bool hi = false;
    if (const char* v = opt.get("P2S_LARGE_PRIO")) hi = v[0] != '0';
    P2S_CUDA(cudaStreamCreateWithPriority(&c->lpack.aux, cudaStreamNonBlocking, hi ? prio_hi : prio_lo));
    P2S_CUDA(cudaStreamCreateWithFlags(&c->lpack.aux_u, cudaStreamNonBlocking));
    P2S_CUDA(cudaEventCreateWithFlags(&c->lpack.ev_start, cudaEventDisableTiming));
    P2S_CUDA(cudaEventCreateWithFlags(&c->lpack.ev_join, cudaEventDisableTiming));
    if (const char* v = opt.get("P2S_LARGE_USTREAMS")) c->lpack.two_u = v[0] != '1';
    c->lpack.u_ctas = -1;  // persistent u stage, every resident CTA slot (occupancy x SMs)
    c->lpack.num_sms = c->num_sms;
    if (const char* v = opt.get("P2S_LARGE_UPERSIST")) {  // k CTAs per SM; 0: one per tile; < 0: occupancy
      const int k = std::atoi(v);
      c->lpack.u_ctas = k < 0 ? -1 : static_cast<int64_t>(k) * c->num_sms;
    }
    // CTA slots of the persistent u grid left free for the next chunk's w / v steps:
    // the u stage fills every SM's registers, so those steps otherwise run only in
    // its tail.  Worth it where they are a large share of the work -- (X + Z) bytes
    // per unit against the unit's block of M: N = 9 (0.37) +21 % with one slot per
    // SM, N = 10 (0.31) +5 % and N = 11 (0.27) +3 % with one per two SMs; c12 (0.23)
    // and C5 (0.15) lose 0-4 % (tools/gpu_sweep_ures.sh, gpu_sweep_r2w.sh)
    {
      const double nt = static_cast<double>(spec->order[0]) * spec->order[1] * spec->order[2];
      const double rho = static_cast<double>(lge->xpu + lge->zpu) / (nt * nt);
      if (c->lpack.u_ctas < 0 && rho >= 0.25) c->lpack.u_ctas = -1 - (rho >= 0.34 ? c->num_sms : c->num_sms / 2);
    }
    if (const char* v = opt.get("P2S_LARGE_URESERVE"))
      if (c->lpack.u_ctas < 0) c->lpack.u_ctas = -1 - std::max(0, std::atoi(v));
    if (const char* v = opt.get("P2S_GRAPH")) c->use_graphs = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_VSPLIT")) c->lpack.v_split = std::max(0, std::atoi(v));
    if (const char* v = opt.get("P2S_LARGE_XS")) c->lpack.u_xs = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_UBULK")) c->lpack.u_bulk = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_UROLL")) c->lpack.u_roll = v[0] == '1' ? 1 : 0;
    if (const char* v = opt.get("P2S_LARGE_UPAIR")) c->lpack.u_pair = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_MSPLIT")) c->lpack.mom_split = v[0] != '0';
    if (c->lpack.mom_split) {  // ~24 MB of u-pass scratch: stays in L2 for the v/w passes
      c->lpack.t1_units = std::max<int64_t>(1, (int64_t(24) << 20) / (lge->t1u * 8));
      P2S_CUDA(cudaMalloc(&c->lpack.d_T1, sizeof(double) * lge->t1u * c->lpack.t1_units));
    }
    // moment kernel: the w-first tiled kernel where its first pass has at least two warps
    // of (q2, q1 pair) columns per CTA; rules with few points along u / v keep the u-first
    // kernel (grid shapes with Q_v (Q_u + 1) / 2 = 32-48 ran 5-18 % slower w-first)
    c->lpack.mom_wfirst = spec->nq[1] * ((spec->nq[0] + 1) / 2) >= 64;
    if (const char* v = opt.get("P2S_LARGE_MOMW")) c->lpack.mom_wfirst = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_MOMT")) c->lpack.mom_tiled = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_MOMG")) c->lpack.mom_grouped = v[0] != '0';
    if (const char* v = opt.get("P2S_LARGE_MOMCL")) c->lpack.mom_cluster = v[0] == '1';
    if (const char* v = opt.get("P2S_LARGE_USMEM")) c->lpack.u_smemc = v[0] == '1';
    if (const char* v = opt.get("P2S_LARGE_FIB")) c->lpack.ufib = std::atoi(v) == 2 ? 2 : 1;
    for (int b = 0; b < 2; ++b) {
      P2S_CUDA(cudaEventCreateWithFlags(&c->lpack.ev_vw[b], cudaEventDisableTiming));
      P2S_CUDA(cudaEventCreateWithFlags(&c->lpack.ev_u[b], cudaEventDisableTiming));
    }
  }

  // scheduler chunk: ~256 MB of moment scratch per buffer, double-buffered in the
  // two-stage path (P2S_TWO_STAGE_OVERLAP=0: serial).  Measured on C3 (elem/s):
  // 32 MB (L2-resident I, short launches with tails) 2.07 M, 128 MB 2.26 M,
  // 256 MB 2.29 M, 1 GB 2.31 M -- the I round trip through HBM (2 % of the bytes)
  // costs less than the launch tails of small chunks
  const int64_t per = c->sz.moments_per_elem * 8;
  int64_t cmb = 256;
  if (const char* v = opt.get("P2S_CHUNK_MB")) cmb = std::max(1, std::atoi(v));
  c->chunk = std::max<int64_t>(1, (cmb << 20) / per);
  bool overlap = !c->large && !c->fused;
  if (const char* v = opt.get("P2S_TWO_STAGE_OVERLAP")) overlap = overlap && v[0] != '0';
  P2S_CUDA(cudaMalloc(&c->d_scratch, sizeof(double) * c->sz.moments_per_elem * c->chunk * (overlap ? 2 : 1)));
  if (overlap) {
    // P2S_MOM_PRIO=1: the moments stream at the highest priority (its CTAs are
    // dispatched first whenever a contraction CTA retires); C3: 2.30 M either way
    int plo = 0, phi = 0;
    P2S_CUDA(cudaDeviceGetStreamPriorityRange(&plo, &phi));
    bool mhi = false;
    if (const char* v = opt.get("P2S_MOM_PRIO")) mhi = v[0] == '1';
    P2S_CUDA(cudaStreamCreateWithPriority(&c->s_mom, cudaStreamNonBlocking, mhi ? phi : plo));
    P2S_CUDA(cudaEventCreateWithFlags(&c->ev_fill_start, cudaEventDisableTiming));
    for (int b = 0; b < 2; ++b) {
      P2S_CUDA(cudaEventCreateWithFlags(&c->ev_mom_done[b], cudaEventDisableTiming));
      P2S_CUDA(cudaEventCreateWithFlags(&c->ev_con_done[b], cudaEventDisableTiming));
    }
  }
  *out = c.release();
  return P2S_OK;
}

void p2s_destroy(p2s_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int s = 0; s < kMaxTerms; ++s)
    for (int d = 0; d < 3; ++d) {
      if (c->d_phiT[s][d]) cudaFree(c->d_phiT[s][d]);
      if (c->d_coef[s][d]) cudaFree(c->d_coef[s][d]);
    }
  for (int d = 0; d < 3; ++d)
    if (c->d_x[d]) cudaFree(c->d_x[d]);
  if (c->d_scratch) cudaFree(c->d_scratch);
  if (c->s_mom) cudaStreamDestroy(c->s_mom);
  if (c->ev_fill_start) cudaEventDestroy(c->ev_fill_start);
  for (int b = 0; b < 2; ++b) {
    if (c->ev_mom_done[b]) cudaEventDestroy(c->ev_mom_done[b]);
    if (c->ev_con_done[b]) cudaEventDestroy(c->ev_con_done[b]);
  }
  if (c->d_X) cudaFree(c->d_X);
  if (c->lpack.d_Z) cudaFree(c->lpack.d_Z);
  if (c->lpack.d_cu) cudaFree(c->lpack.d_cu);
  if (c->lpack.d_cvw) cudaFree(c->lpack.d_cvw);
  if (c->lpack.d_T1) cudaFree(c->lpack.d_T1);
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->s_cap) cudaStreamDestroy(c->s_cap);
  if (c->lpack.aux) cudaStreamDestroy(c->lpack.aux);
  if (c->lpack.aux_u) cudaStreamDestroy(c->lpack.aux_u);
  if (c->lpack.ev_start) cudaEventDestroy(c->lpack.ev_start);
  if (c->lpack.ev_join) cudaEventDestroy(c->lpack.ev_join);
  for (int b = 0; b < 2; ++b) {
    if (c->lpack.ev_vw[b]) cudaEventDestroy(c->lpack.ev_vw[b]);
    if (c->lpack.ev_u[b]) cudaEventDestroy(c->lpack.ev_u[b]);
  }
  if (c->d_amma_fused) cudaFree(c->d_amma_fused);
  for (int b = 0; b < 2; ++b) {
    if (c->d_geo_alpha[b]) cudaFree(c->d_geo_alpha[b]);
    if (c->ev_ga[b]) cudaEventDestroy(c->ev_ga[b]);
    if (c->ev_gf[b]) cudaEventDestroy(c->ev_gf[b]);
  }
  if (c->ev_geo_start) cudaEventDestroy(c->ev_geo_start);
  if (c->ev_scratch) cudaEventDestroy(c->ev_scratch);
  if (c->d_bad) cudaFree(c->d_bad);
  if (c->h_bad) cudaFreeHost(c->h_bad);
  if (c->s_geo) cudaStreamDestroy(c->s_geo);
  if (c->d_amma_v2) cudaFree(c->d_amma_v2);
  for (int i = 0; i < 2; ++i) {
    if (c->d_ring_alpha[i]) cudaFree(c->d_ring_alpha[i]);
    if (c->d_ring_M[i]) cudaFree(c->d_ring_M[i]);
    if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
    if (c->ev_comp[i]) cudaEventDestroy(c->ev_comp[i]);
    if (c->ev_d2h[i]) cudaEventDestroy(c->ev_d2h[i]);
  }
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_comp) cudaStreamDestroy(c->s_comp);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  harvest(c);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  delete c;
}

p2s_status p2s_problem_sizes(const p2s_problem* spec, p2s_sizes* out) {
  if (!out) return fail(P2S_INVALID_ARG, "p2s_problem_sizes: null out");
  p2s_status st = validate(spec);
  if (st != P2S_OK) return st;
  problem_sizes(*spec, out);
  return P2S_OK;
}

p2s_status p2s_get_sizes(const p2s_ctx* c, p2s_sizes* out) {
  if (check_ctx(c) != P2S_OK || !out) return fail(P2S_INVALID_ARG, "p2s_get_sizes: null argument");
  *out = c->sz;
  return P2S_OK;
}

p2s_status p2s_moments(p2s_ctx* c, const double* d_alpha, double* d_I, int64_t n, void* stream) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && (!d_alpha || !d_I))) return fail(P2S_INVALID_ARG, "p2s_moments: bad buffers");
  if (reinterpret_cast<uintptr_t>(d_alpha) % alpha_align(c))
    return fail(P2S_INVALID_ARG, "p2s_moments: alpha must be " + std::to_string(alpha_align(c)) + "-byte aligned");
  P2S_CUDA(cudaSetDevice(c->device));
  return run_moments(c, d_alpha, d_I, n, static_cast<cudaStream_t>(stream));
}

p2s_status p2s_contract(p2s_ctx* c, const double* d_I, double* d_M, int64_t ldM, int64_t n,
                        void* stream) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && (!d_I || !d_M))) return fail(P2S_INVALID_ARG, "p2s_contract: bad buffers");
  if (ldM < c->sz.n_tot) return fail(P2S_INVALID_ARG, "p2s_contract: ld_M < n_tot");
  if (reinterpret_cast<uintptr_t>(d_I) % 16) return fail(P2S_INVALID_ARG, "I must be 16-byte aligned");
  P2S_CUDA(cudaSetDevice(c->device));
  if (c->large) {  // the w / v / u steps run through context scratch
    ScratchUse use(c, static_cast<cudaStream_t>(stream));
    if (!use.ok()) return fail(P2S_CUDA_ERROR, "p2s_contract: stream ordering");
    return run_contract(c, d_I, d_M, ldM, n, static_cast<cudaStream_t>(stream));
  }
  return run_contract(c, d_I, d_M, ldM, n, static_cast<cudaStream_t>(stream));
}

p2s_status p2s_fill(p2s_ctx* c, const double* d_alpha, double* d_M, int64_t ldM, int64_t n,
                    void* stream) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && (!d_alpha || !d_M))) return fail(P2S_INVALID_ARG, "p2s_fill: bad buffers");
  if (ldM < c->sz.n_tot) return fail(P2S_INVALID_ARG, "p2s_fill: ld_M < n_tot");
  if (reinterpret_cast<uintptr_t>(d_alpha) % alpha_align(c))
    return fail(P2S_INVALID_ARG, "p2s_fill: alpha must be " + std::to_string(alpha_align(c)) + "-byte aligned");
  P2S_CUDA(cudaSetDevice(c->device));
  if (!c->fused) {  // two-stage / large paths: moment and intermediate scratch
    ScratchUse use(c, static_cast<cudaStream_t>(stream));
    if (!use.ok()) return fail(P2S_CUDA_ERROR, "p2s_fill: stream ordering");
    if (c->large) return run_fill_graphed(c, d_alpha, d_M, ldM, n, static_cast<cudaStream_t>(stream));
    return run_fill(c, d_alpha, d_M, ldM, n, static_cast<cudaStream_t>(stream));
  }
  return run_fill(c, d_alpha, d_M, ldM, n, static_cast<cudaStream_t>(stream));
}

p2s_status p2s_fill_host(p2s_ctx* c, const double* h_alpha, double* h_M, int64_t ldM, int64_t n) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && (!h_alpha || !h_M))) return fail(P2S_INVALID_ARG, "p2s_fill_host: bad buffers");
  if (ldM < c->sz.n_tot) return fail(P2S_INVALID_ARG, "p2s_fill_host: ld_M < n_tot");
  P2S_CUDA(cudaSetDevice(c->device));
  const int64_t nt = c->sz.n_tot;
  const int64_t ape = c->sz.alpha_per_elem;
  const int64_t mel = nt * nt;  // device ring keeps ld = n_tot
  std::lock_guard<std::mutex> ring_lock(c->scratch_mu);  // synchronous: host-side order suffices
  if (!c->s_h2d) {
    P2S_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    P2S_CUDA(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
    P2S_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      P2S_CUDA(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming));
      P2S_CUDA(cudaEventCreateWithFlags(&c->ev_comp[i], cudaEventDisableTiming));
      P2S_CUDA(cudaEventCreateWithFlags(&c->ev_d2h[i], cudaEventDisableTiming));
    }
    // ~64 MB of matrices per slot (P2S_HOST_CHUNK_MB); C2 e2e measured 32 MB 15.31 k,
    // 64 MB 15.38 k, 256 MB 15.26 k, 1 GB 15.02 k elem/s: the D2H copy (51.7 GB/s of a
    // 56.4 GB/s PCIe peak) is the bound
    int64_t hmb = 64;
    if (const char* v = c->opt.get("P2S_HOST_CHUNK_MB")) hmb = std::max(1, std::atoi(v));
    c->host_chunk = std::max<int64_t>(1, (hmb << 20) / (mel * 8));
    for (int i = 0; i < 2; ++i) {
      P2S_CUDA(cudaMalloc(&c->d_ring_alpha[i], sizeof(double) * ape * c->host_chunk));
      P2S_CUDA(cudaMalloc(&c->d_ring_M[i], sizeof(double) * mel * c->host_chunk));
    }
  }
  int64_t slot_iter[2] = {0, 0};
  int it = 0;
  for (int64_t e0 = 0; e0 < n; e0 += c->host_chunk, ++it) {
    const int sl = it & 1;
    const int64_t cnt = std::min(c->host_chunk, n - e0);
    if (slot_iter[sl] > 0) P2S_CUDA(cudaStreamWaitEvent(c->s_h2d, c->ev_d2h[sl], 0));
    P2S_CUDA(cudaMemcpyAsync(c->d_ring_alpha[sl], h_alpha + e0 * ape, sizeof(double) * ape * cnt,
                             cudaMemcpyHostToDevice, c->s_h2d));
    P2S_CUDA(cudaEventRecord(c->ev_h2d[sl], c->s_h2d));
    P2S_CUDA(cudaStreamWaitEvent(c->s_comp, c->ev_h2d[sl], 0));
    p2s_status st = run_fill(c, c->d_ring_alpha[sl], c->d_ring_M[sl], nt, cnt, c->s_comp);
    if (st != P2S_OK) return st;
    P2S_CUDA(cudaEventRecord(c->ev_comp[sl], c->s_comp));
    P2S_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_comp[sl], 0));
    if (ldM == nt) {
      P2S_CUDA(cudaMemcpyAsync(h_M + e0 * mel, c->d_ring_M[sl], sizeof(double) * mel * cnt,
                               cudaMemcpyDeviceToHost, c->s_d2h));
    } else {
      P2S_CUDA(cudaMemcpy2DAsync(h_M + e0 * nt * ldM, sizeof(double) * ldM, c->d_ring_M[sl],
                                 sizeof(double) * nt, sizeof(double) * nt, nt * cnt,
                                 cudaMemcpyDeviceToHost, c->s_d2h));
    }
    P2S_CUDA(cudaEventRecord(c->ev_d2h[sl], c->s_d2h));
    ++slot_iter[sl];
  }
  P2S_CUDA(cudaStreamSynchronize(c->s_d2h));
  P2S_CUDA(cudaStreamSynchronize(c->s_comp));
  return P2S_OK;
}

p2s_status p2s_moments_host(p2s_ctx* c, const double* h_alpha, double* h_I, int64_t n) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && (!h_alpha || !h_I))) return fail(P2S_INVALID_ARG, "p2s_moments_host: bad buffers");
  if (n == 0) return P2S_OK;
  P2S_CUDA(cudaSetDevice(c->device));
  double *da = nullptr, *dI = nullptr;
  const size_t na = sizeof(double) * c->sz.alpha_per_elem * n, ni = sizeof(double) * c->sz.moments_per_elem * n;
  P2S_CUDA(cudaMalloc(&da, na));
  cudaError_t e = cudaMalloc(&dI, ni);
  p2s_status st = P2S_OK;
  if (e == cudaSuccess) e = cudaMemcpy(da, h_alpha, na, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) st = run_moments(c, da, dI, n, 0);
  if (e == cudaSuccess && st == P2S_OK) e = cudaMemcpy(h_I, dI, ni, cudaMemcpyDeviceToHost);
  cudaFree(da);
  if (dI) cudaFree(dI);
  if (e != cudaSuccess) return cuda_fail(e, "p2s_moments_host");
  return st;
}

p2s_status p2s_contract_host(p2s_ctx* c, const double* h_I, double* h_M, int64_t ldM, int64_t n) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && (!h_I || !h_M))) return fail(P2S_INVALID_ARG, "p2s_contract_host: bad buffers");
  if (ldM < c->sz.n_tot) return fail(P2S_INVALID_ARG, "p2s_contract_host: ld_M < n_tot");
  if (n == 0) return P2S_OK;
  P2S_CUDA(cudaSetDevice(c->device));
  double *dI = nullptr, *dM = nullptr;
  const int64_t nt = c->sz.n_tot;
  const size_t ni = sizeof(double) * c->sz.moments_per_elem * n, nm = sizeof(double) * nt * nt * n;
  P2S_CUDA(cudaMalloc(&dI, ni));
  cudaError_t e = cudaMalloc(&dM, nm);
  p2s_status st = P2S_OK;
  if (e == cudaSuccess) e = cudaMemcpy(dI, h_I, ni, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    if (c->large) {
      ScratchUse use(c, 0);
      st = run_contract(c, dI, dM, nt, n, 0);
    } else {
      st = run_contract(c, dI, dM, nt, n, 0);
    }
  }
  if (e == cudaSuccess && st == P2S_OK)
    e = cudaMemcpy2D(h_M, sizeof(double) * ldM, dM, sizeof(double) * nt, sizeof(double) * nt, nt * n,
                     cudaMemcpyDeviceToHost);
  cudaFree(dI);
  if (dM) cudaFree(dM);
  if (e != cudaSuccess) return cuda_fail(e, "p2s_contract_host");
  return st;
}

p2s_status p2s_alpha_generate(p2s_ctx* c, int kind, double lo, double hi, uint64_t seed,
                              int64_t e0, int64_t n, double* d_alpha, void* stream) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (kind < 0 || kind > 2) return fail(P2S_INVALID_ARG, "p2s_alpha_generate: bad kind");
  if (n < 0 || (n > 0 && !d_alpha)) return fail(P2S_INVALID_ARG, "p2s_alpha_generate: bad buffer");
  P2S_CUDA(cudaSetDevice(c->device));
  const double* xs[3] = {c->d_x[0], c->d_x[1], c->d_x[2]};
  cudaError_t err = launch_alpha(d_alpha, xs, c->pb.nq, c->pb.n_comp, c->pb.n_terms, kind, lo, hi,
                                 seed, e0, n, c->sz.alpha_per_elem, static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "alpha_kernel launch");
  return P2S_OK;
}

p2s_status p2s_geometry_generate(p2s_ctx* c, double lo, double hi, uint64_t seed, int64_t e0, int64_t n,
                                 double* d_geom, void* stream) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && !d_geom)) return fail(P2S_INVALID_ARG, "p2s_geometry_generate: bad buffer");
  P2S_CUDA(cudaSetDevice(c->device));
  cudaError_t err = launch_geometry(d_geom, lo, hi, seed, e0, n, static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "geometry_kernel launch");
  return P2S_OK;
}

namespace {
// GeometryError of the reference (assembly.cpp:95-99): the geometry entry points
// clear a device flag, their kernels set it at any quadrature point with
// det J <= 0, and the call waits for the stream and reports it
p2s_status geo_flag_begin(p2s_ctx* c, cudaStream_t st) {
  if (!c->d_bad) {
    P2S_CUDA(cudaMalloc(&c->d_bad, sizeof(int)));
    P2S_CUDA(cudaMallocHost(&c->h_bad, sizeof(int)));
  }
  P2S_CUDA(cudaMemsetAsync(c->d_bad, 0, sizeof(int), st));
  return P2S_OK;
}

p2s_status geo_flag_end(p2s_ctx* c, cudaStream_t st, const char* where) {
  P2S_CUDA(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  P2S_CUDA(cudaStreamSynchronize(st));
  if (*c->h_bad)
    return fail(P2S_GEOMETRY_ERROR, std::string(where) + ": non-positive Jacobian at a quadrature point");
  return P2S_OK;
}
}  // namespace

p2s_status p2s_alpha_from_geometry(p2s_ctx* c, const double* d_geom, int64_t n, double* d_alpha,
                                   void* stream) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || (n > 0 && (!d_geom || !d_alpha)))
    return fail(P2S_INVALID_ARG, "p2s_alpha_from_geometry: bad buffer");
  if (n == 0) return P2S_OK;
  P2S_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ScratchUse use(c, st);  // the Jacobian flag
  if (!use.ok()) return fail(P2S_CUDA_ERROR, "p2s_alpha_from_geometry: stream ordering");
  p2s_status s0 = geo_flag_begin(c, st);
  if (s0 != P2S_OK) return s0;
  const double* xs[3] = {c->d_x[0], c->d_x[1], c->d_x[2]};
  cudaError_t err = launch_alpha_geometry_fast(d_alpha, d_geom, xs, c->pb.nq, c->pb.n_comp, c->pb.n_terms,
                                               n, c->sz.alpha_per_elem, c->d_bad, st);
  if (err != cudaSuccess) return cuda_fail(err, "alpha_geometry_kernel launch");
  return geo_flag_end(c, st, "p2s_alpha_from_geometry");
}

p2s_status p2s_fill_geometry(p2s_ctx* c, const double* d_geom, double* d_M, int64_t ld_M, int64_t n,
                             void* stream) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (n < 0 || ld_M < c->sz.n_tot) return fail(P2S_INVALID_ARG, "p2s_fill_geometry: bad sizes");
  if (n == 0) return P2S_OK;
  if (!d_geom || !d_M) return fail(P2S_INVALID_ARG, "p2s_fill_geometry: null buffer");
  P2S_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ScratchUse use(c, st);  // geometry buffers, flag, fill scratch
  if (!use.ok()) return fail(P2S_CUDA_ERROR, "p2s_fill_geometry: stream ordering");
  p2s_status s0 = geo_flag_begin(c, st);
  if (s0 != P2S_OK) return s0;
  const fused_fn geo_launch = !c->fused              ? nullptr
                             : c->geo_mode == 2     ? c->fused->launch_geo_cluster
                             : c->geo_mode == 1     ? c->fused->launch_geo
                                                    : nullptr;
  if (geo_launch) {
    // one kernel: the moment phase gets the coupling factors from the records
    std::vector<double> mp = c->fused_mpack;
    for (int d = 0; d < 3; ++d) mp.insert(mp.end(), c->x[d].begin(), c->x[d].end());
    cudaError_t err = geo_launch(d_geom, d_M, ld_M, c->sz.n_tot, n, c->pb.n_comp, c->sz.n_pairs,
                                 c->pb.order[0] * c->pb.order[1] * c->pb.order[2], c->fused_cpack, mp,
                                 c->d_amma_fused, st, c->num_sms, c->d_bad);
    if (err != cudaSuccess) return cuda_fail(err, "fill_fused_kernel (geometry) launch");
    return geo_flag_end(c, st, "p2s_fill_geometry");
  }
  if (!c->s_geo) {  // lazily: two alpha buffers of ~48 MB (L2), a stream, events
    const int64_t per = c->sz.alpha_per_elem * 8;
    int64_t mb = 48;
    if (const char* v = c->opt.get("P2S_GEO_CHUNK_MB")) mb = std::max(1, std::atoi(v));
    c->geo_chunk = std::max<int64_t>(1, (mb << 20) / per);
    for (int b = 0; b < 2; ++b) {
      P2S_CUDA(cudaMalloc(&c->d_geo_alpha[b], static_cast<size_t>(per * c->geo_chunk)));
      P2S_CUDA(cudaEventCreateWithFlags(&c->ev_ga[b], cudaEventDisableTiming));
      P2S_CUDA(cudaEventCreateWithFlags(&c->ev_gf[b], cudaEventDisableTiming));
    }
    P2S_CUDA(cudaEventCreateWithFlags(&c->ev_geo_start, cudaEventDisableTiming));
    P2S_CUDA(cudaStreamCreateWithFlags(&c->s_geo, cudaStreamNonBlocking));
  }
  const double* xs[3] = {c->d_x[0], c->d_x[1], c->d_x[2]};
  const int64_t mstride = static_cast<int64_t>(c->sz.n_tot) * ld_M;
  P2S_CUDA(cudaEventRecord(c->ev_geo_start, st));
  P2S_CUDA(cudaStreamWaitEvent(c->s_geo, c->ev_geo_start, 0));
  int64_t i = 0;
  for (int64_t e0 = 0; e0 < n; e0 += c->geo_chunk, ++i) {
    const int64_t cnt = std::min(c->geo_chunk, n - e0);
    const int b = static_cast<int>(i % 2);
    if (i >= 2) P2S_CUDA(cudaStreamWaitEvent(c->s_geo, c->ev_gf[b], 0));  // buffer b free
    cudaError_t err = launch_alpha_geometry_fast(c->d_geo_alpha[b], d_geom + e0 * 28, xs, c->pb.nq,
                                                 c->pb.n_comp, c->pb.n_terms, cnt, c->sz.alpha_per_elem,
                                                 c->d_bad, c->s_geo);
    if (err != cudaSuccess) return cuda_fail(err, "alpha_geometry_kernel launch");
    P2S_CUDA(cudaEventRecord(c->ev_ga[b], c->s_geo));
    P2S_CUDA(cudaStreamWaitEvent(st, c->ev_ga[b], 0));
    const p2s_status s2 = run_fill(c, c->d_geo_alpha[b], d_M + e0 * mstride, ld_M, cnt, st);
    if (s2 != P2S_OK) return s2;
    P2S_CUDA(cudaEventRecord(c->ev_gf[b], st));
  }
  return geo_flag_end(c, st, "p2s_fill_geometry");
}

p2s_status p2s_get_tables(const p2s_ctx* c, int term, int dir, double* phi, double* coef,
                          double* nodes, double* weights) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  if (term < 0 || term >= c->pb.n_terms || dir < 0 || dir > 2)
    return fail(P2S_INVALID_ARG, "p2s_get_tables: bad term/dir");
  if (phi) std::memcpy(phi, c->phi[term][dir].data(), sizeof(double) * c->phi[term][dir].size());
  if (coef) std::memcpy(coef, c->coef[term][dir].data(), sizeof(double) * c->coef[term][dir].size());
  if (nodes) std::memcpy(nodes, c->x[dir].data(), sizeof(double) * c->x[dir].size());
  if (weights) std::memcpy(weights, c->w[dir].data(), sizeof(double) * c->w[dir].size());
  return P2S_OK;
}

p2s_status p2s_set_profiling(p2s_ctx* c, int enable) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  P2S_CUDA(cudaSetDevice(c->device));
  P2S_CUDA(cudaDeviceSynchronize());
  harvest(c);
  c->prof = enable != 0;
  c->ms_mom = c->ms_con = 0.0;
  c->n_mom = c->n_con = c->n_fused = 0;
  return P2S_OK;
}

p2s_status p2s_get_stage_times(p2s_ctx* c, double* ms_mom, double* ms_con, int64_t* n_mom,
                               int64_t* n_con) {
  if (check_ctx(c) != P2S_OK) return P2S_INVALID_ARG;
  P2S_CUDA(cudaSetDevice(c->device));
  P2S_CUDA(cudaDeviceSynchronize());
  harvest(c);
  if (ms_mom) *ms_mom = c->ms_mom;
  if (ms_con) *ms_con = c->ms_con;
  if (n_mom) *n_mom = c->n_mom;
  if (n_con) *n_con = c->n_con;
  return P2S_OK;
}

}  // extern "C"
