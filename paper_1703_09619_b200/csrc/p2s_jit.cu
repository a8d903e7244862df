// p2s_jit.cu -- shape planner and generated per-shape modules.
//
// The reference accepts any Orders / kinds / nq (assembly.hpp:52-56, 82-83;
// fill_elements assembly.cpp:654-700; Table I sweeps M = N = 3..18).
// The fast kernels of this library unroll every product-to-sum band at compile
// time (p2s_contract_v2.cuh, p2s_fused.cuh, p2s_large.cuh), so a problem that
// no ahead-of-time registry entry covers gets its own instantiation:
//
//   plan()      picks the kernel family and its template parameters from the
//               problem (shared-memory and kernel-parameter budgets computed
//               with the same formulas as the templates' constexpr layouts):
//                 fused   fill_fused_kernel (+ contract_v2 / moments_v2 of the
//                         same shape for p2s_moments / p2s_contract) when one
//                         (element, pair) unit's moments and intermediates fit
//                         a CTA's shared memory;
//                 large   moments -> w step -> v step -> u stage through an
//                         L2-resident intermediate otherwise.
//   module()    writes a one-line translation unit instantiating that plan,
//               compiles it with nvcc for sm_100a into a shared object in the
//               module cache (default: <dir of libp2s_b200.so>/jit, override
//               P2S_JIT_CACHE), loads it and returns its registry entries.  A
//               cached module is reused by every later context and process;
//               the cache key covers the generated source, the compiler flags
//               and a hash of every kernel header (P2S_SRC_HASH, Makefile).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "p2s_jit.hpp"
#include "p2s_registry.hpp"
#include "p2s_tables.hpp"

#ifndef P2S_SRC_HASH
#define P2S_SRC_HASH "unknown"
#endif

namespace p2s {
namespace jit {

namespace {

// ---------------------------------------------------------------- layout mirrors
// Host mirrors of the constexpr layouts of Shape (p2s_contract_v2.cuh), MShape
// (p2s_moments_v2.cuh), FusedLayout (p2s_fused.cuh) and LShape (p2s_large.cuh).
// The generated module reports the compiled sizes back (JitEntries) and p2s_create
// checks them against these.

struct Desc {
  int N[3], Q[3], S;
  int kind[kMaxTerms][3];
  int K(int s, int d) const { return kernel_count(kind[s][d], N[d]); }
  int KMAX(int d) const {
    int m = 0;
    for (int s = 0; s < S; ++s) m = std::max(m, K(s, d));
    return m;
  }
  int ctot(int d) const {
    int o = 0;
    for (int s = 0; s < S; ++s)
      for (int a = 0; a < N[d]; ++a)
        for (int b = 0; b < N[d]; ++b) o += band_count(kind[s][d], a, b);
    return o > 0 ? o : 1;
  }
  bool sym(int d) const {
    for (int s = 0; s < S; ++s)
      if (base_kind(kind[s][d]) != PP && base_kind(kind[s][d]) != DD) return false;
    return true;
  }
  bool any_conforming() const {
    for (int s = 0; s < S; ++s)
      for (int d = 0; d < 3; ++d)
        if (conforming(kind[s][d])) return true;
    return false;
  }
  int64_t mpp() const {
    int64_t o = 0;
    for (int s = 0; s < S; ++s) o += static_cast<int64_t>(K(s, 0)) * K(s, 1) * K(s, 2);
    return (o + 3) & ~int64_t(3);
  }
  int H(int d) const { return (Q[d] + 1) / 2; }
  int ktot_u() const {
    int o = 0;
    for (int s = 0; s < S; ++s) o += K(s, 0);
    return o;
  }
};

struct FusedCand {
  int T, threads, minb, flags, fpt;
  bool pf;
  int64_t smem_fused, smem_v2, smem_mv2, param_bytes;
};

// Shape<..>::SMEM pieces (doubles)
void shape_layout(const Desc& d, int T, int flags, int64_t* A, int64_t* B) {
  const int NV = d.N[1], NW = d.N[2];
  const bool SYM = (flags >> 2) & 1;
  const bool AALL = (flags & 1) || SYM;
  const int AT = AALL ? NV : T;
  const int NQV = NV * (NV + 1) / 2, NQW = NW * (NW + 1) / 2;
  int64_t a = 0, b = 0;
  const int64_t BSTR = SYM ? ((NV * NQW) | 1) : ((NW * NV * NW) | 1);
  for (int s = 0; s < d.S; ++s) {
    const int64_t aks = SYM ? ((static_cast<int64_t>(NQV) * d.K(s, 2)) | 1) : ((static_cast<int64_t>(NV) * d.K(s, 2)) | 1);
    a += (SYM ? 1 : AT) * static_cast<int64_t>(d.K(s, 0)) * aks;
    b += static_cast<int64_t>(T) * d.K(s, 0) * BSTR;
  }
  *A = (a + 1) & ~int64_t(1);
  *B = (b + 1) & ~int64_t(1);
}

// MShape::scratch_all_dbl (fused moment phase, all terms at once)
int64_t ms_scratch_all(const Desc& d) {
  const int QU = d.Q[0], QV = d.Q[1], QW = d.Q[2];
  const bool WFIRST = d.KMAX(2) < d.KMAX(0);
  int64_t o = 0;
  if (WFIRST) {
    for (int s = 0; s < d.S; ++s) o += static_cast<int64_t>(d.K(s, 2)) * QV * (QU | 1);
    for (int s = 0; s < d.S; ++s) o += static_cast<int64_t>(d.K(s, 2)) * d.K(s, 1) * (QU | 1);
  } else {
    for (int s = 0; s < d.S; ++s) o += static_cast<int64_t>(d.K(s, 0)) * QW * (QV | 1);
    for (int s = 0; s < d.S; ++s) o += static_cast<int64_t>(d.K(s, 0)) * d.K(s, 1) * (QW | 1);
  }
  return (o + 1) & ~int64_t(1);
}

// MShape::scratch_dbl (two-stage moments, one term per CTA)
int64_t ms_scratch_one(const Desc& d) {
  int64_t m = 0;
  for (int s = 0; s < d.S; ++s)
    m = std::max(m, static_cast<int64_t>(d.K(s, 0)) * d.Q[2] * (d.Q[1] | 1) +
                        static_cast<int64_t>(d.K(s, 0)) * d.K(s, 1) * (d.Q[2] | 1));
  return (m + 1) & ~int64_t(1);
}

int64_t ms_tall(const Desc& d) {
  int64_t o = 0;
  for (int s = 0; s < d.S; ++s)
    for (int e = 0; e < 3; ++e) o += static_cast<int64_t>(d.K(s, e)) * d.H(e);
  for (int e = 0; e < 3; ++e) o += static_cast<int64_t>(d.KMAX(e)) * d.H(e);
  return o;
}

constexpr int64_t kSmemMax = 227 * 1024;
constexpr int64_t kSmemTwo = 113 * 1024;        // two CTAs per SM
constexpr int64_t kParamMax = 32 * 1024 - 256;  // kernel parameter space (CUDA 12.1+), with headroom

FusedCand fused_candidate(const Desc& d, int T, int flags, int threads, int fpt) {
  FusedCand c{};
  c.T = T;
  c.flags = flags;
  c.threads = threads;
  c.fpt = fpt;
  c.pf = true;
  int64_t A = 0, B = 0;
  shape_layout(d, T, flags, &A, &B);
  const int64_t mpp = d.mpp();
  c.smem_fused = 8 * (mpp + std::max(A + B, ms_scratch_all(d)));
  c.smem_v2 = 8 * (mpp + A + B) + 16;
  c.smem_mv2 = 8 * ms_scratch_one(d);
  c.minb = c.smem_fused <= kSmemTwo ? 2 : 1;
  c.param_bytes = 8 * (d.ctot(0) + d.ctot(1) + d.ctot(2) + ms_tall(d) + d.Q[0] + d.Q[1] + d.Q[2]) + 128;
  return c;
}

bool fused_ok(const FusedCand& c) {
  return c.smem_fused <= kSmemMax && c.smem_v2 <= kSmemMax && c.smem_mv2 <= kSmemMax &&
         c.param_bytes <= kParamMax;
}

std::string kinds_list(const Desc& d) {
  std::ostringstream o;
  for (int s = 0; s < d.S; ++s) o << ", " << (d.kind[s][0] | (d.kind[s][1] << 3) | (d.kind[s][2] << 6));
  return o.str();
}

// Fused family: the first candidate that fits, in order of preference.
bool plan_fused(const Desc& d, Plan* pl, const Overrides& ov) {
  const int NU = d.N[0], NV = d.N[1];
  const bool sym = d.sym(1) && d.sym(2);
  const bool modal = !d.any_conforming();
  // stage-C fiber: FPT fibers of KTOT_U doubles (halved by the parity split)
  const int ktot = d.ktot_u();
  const bool psplit = modal && ktot > 24;
  const int fpt = (psplit ? (ktot + 1) / 2 : ktot) <= 24 ? 2 : 1;
  int base = (psplit ? 64 : 0) | (NU >= 8 ? 2 : 0);
  std::vector<int> tiles;
  for (int t = NV; t >= 1; --t)
    if (NV % t == 0 && (ov.T < 0 || t == ov.T)) tiles.push_back(t);
  const int threads = ov.threads > 0 ? ov.threads : 256;
  FusedCand best{};
  bool found = false;
  // two CTAs per SM with the widest n1 tile, else one CTA per SM
  // non-symmetric v/w kinds: stage A once per unit for all n1 (AALL, flag 1);
  // the per-tile stage A (T < N_v without AALL) gave wrong matrices for a
  // generated (7, 7, 7) shape at T = 1 (fused and contract_v2 alike,
  // tools/jit_variants.py; profiles/r2_jit_variants.txt), so the planner never
  // emits it (the registered C2 / C4 variants with T = 2 pass their parity tests)
  for (int pass = 0; pass < 2 && !found; ++pass)
    for (int symf : {sym ? 4 : 1, 1}) {
      for (int t : tiles) {
        FusedCand c = fused_candidate(d, t, ov.flags >= 0 ? ov.flags : (base | symf), threads,
                                      ov.fpt > 0 ? ov.fpt : fpt);
        if (ov.minb > 0) c.minb = ov.minb;
        if (!fused_ok(c)) continue;
        if (((c.flags >> 2) & 1) && !sym) continue;
        if (!(c.flags & 5) && c.T < NV) continue;  // see above
        if (pass == 0 && c.smem_fused > kSmemTwo && ov.minb < 0) continue;
        // a two-CTA tile must still give stage C a CTA's worth of work items (a
        // (12, 9, 3) shape at T = 1 has 41: 2.5 M elem/s vs 4.9 M for one CTA with
        // all nine n1, profiles/r2z_sweep_fused.jsonl)
        if (pass == 0 && ov.T < 0 && c.T < NV &&
            static_cast<int64_t>(c.T) * d.N[2] * NV * d.N[2] / c.fpt < 128)
          continue;
        best = c;
        found = true;
        break;
      }
      if (found) break;
    }
  if (!found) return false;
  // small units (little shared memory per CTA): more, smaller CTAs per SM -- such
  // shapes are latency-bound (a CTA is a chain of short phases between barriers),
  // so occupancy by independent CTAs is what pays: ~600 threads per SM over up to 8
  // CTAs.  Measured (r2z): (1, 1, 12) 64 threads x 8: 31 M elem/s vs 9.6 M at 256 x 2;
  // (1, 3, 7) 96 x 6: 129 M vs 76 M; (13, 12, 1) 128 x 4: 18.5 M vs 13.9 M;
  // (5, 5, 5) 192 x 3: 28.4 M vs 24.5 M.
  if (ov.threads <= 0 && ov.minb <= 0) {
    const int ctas = static_cast<int>(std::min<int64_t>(8, kSmemMax / (best.smem_fused + 1024)));
    if (ctas >= 3) {
      best.minb = ctas;
      best.threads = std::max(64, std::min(256, (608 / ctas) / 32 * 32));
    }
  }
  std::ostringstream sh, ms, desc;
  sh << "p2s::Shape<" << d.N[0] << ", " << d.N[1] << ", " << d.N[2] << ", " << best.T << ", " << d.N[2]
     << ", " << d.N[2] << ", " << best.threads << ", " << best.minb << ", " << best.flags << ", " << best.fpt
     << kinds_list(d) << ">";
  ms << "p2s::MShape<" << d.N[0] << ", " << d.N[1] << ", " << d.N[2] << ", " << d.Q[0] << ", " << d.Q[1]
     << ", " << d.Q[2] << ", " << best.threads << kinds_list(d) << ">";
  pl->family = kFamilyFused;
  pl->source = "using JitShape = " + sh.str() + ";\nusing JitMShape = " + ms.str() +
               ";\nP2S_JIT_FUSED(JitShape, JitMShape, " + (best.pf ? "true" : "false") + ")\n";
  desc << "fused fill, n1 tile " << best.T << ", " << best.threads << " threads, " << best.minb
       << " CTA/SM, flags " << best.flags << ", " << best.fpt << " fiber(s)/thread, "
       << best.smem_fused / 1024 << " KB";
  pl->desc = desc.str();
  pl->smem = best.smem_fused;
  return true;
}

bool plan_large(const Desc& d, Plan* pl, std::string* why, const Overrides& ov) {
  // k1 chunks of the moment kernel: 4 (C5); the moment scratch must fit
  int kc = ov.kc > 0 ? ov.kc : 4;
  auto mom_smem = [&](int k) {
    return 8 * (static_cast<int64_t>(k) * d.Q[2] * (d.Q[1] | 1) + static_cast<int64_t>(k) * d.KMAX(1) * (d.Q[2] | 1));
  };
  if (ov.kc <= 0) {
    // every k1 chunk re-reads and re-folds the alpha slab: take the largest (even)
    // chunk whose scratch still lets two CTAs share an SM (80 KB; C5: 4), balanced
    // over the chunks -- small rules (few quadrature points) get all k1 in one CTA
    const int kmax0 = d.KMAX(0);
    int kcmax = 4;
    for (int k = 4; k <= ((kmax0 + 1) & ~1); k += 2)
      if (mom_smem(k) <= 80 * 1024) kcmax = k;
    const int nch = (kmax0 + kcmax - 1) / kcmax;
    kc = std::max(2, ((kmax0 + nch - 1) / nch + 1) & ~1);
  }
  while (kc > 2 && mom_smem(kc) > kSmemMax) kc -= 2;
  if (mom_smem(kc) > kSmemMax) {
    *why = "large path: moment scratch above 227 KB";
    return false;
  }
  if (d.KMAX(1) > 64) {
    *why = "large path: more than 64 kernel polynomials along v";
    return false;
  }
  const int64_t tall = static_cast<int64_t>(d.KMAX(0)) * d.H(0) + static_cast<int64_t>(d.KMAX(1)) * d.H(1) +
                       static_cast<int64_t>(d.KMAX(2)) * d.H(2);
  if (8 * tall + 64 > kParamMax) {
    *why = "large path: weighted kernel tables exceed the kernel parameter space";
    return false;
  }
  std::ostringstream ls, desc;
  ls << "p2s::LShape<" << d.N[0] << ", " << d.N[1] << ", " << d.N[2] << ", " << d.Q[0] << ", " << d.Q[1] << ", "
     << d.Q[2] << ", " << kc << kinds_list(d) << ">";
  pl->family = kFamilyLarge;
  pl->source = "using JitLShape = " + ls.str() + ";\nP2S_JIT_LARGE(JitLShape)\n";
  desc << "large-order: moments (k1 chunks of " << kc << ") + w step + v step + u stage";
  for (int dd = 0; dd < 3; ++dd)
    if (8 * d.ctot(dd) > 30 * 1024)
      desc << ", dir " << dd
           << (8 * d.ctot(dd) <= 128 * 1024 ? " coefficients staged in shared memory" : " coefficients in global memory");
  pl->desc = desc.str();
  pl->smem = mom_smem(kc);
  return true;
}

// ---------------------------------------------------------------- module cache

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char ch : s) {
    h ^= ch;
    h *= 1099511628211ull;
  }
  return h;
}

std::string lib_dir() {
  Dl_info info{};
  if (dladdr(reinterpret_cast<void*>(&fnv1a), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const size_t k = p.find_last_of('/');
    if (k != std::string::npos) return p.substr(0, k);
  }
  return ".";
}

bool is_dir(const std::string& p) {
  struct stat st{};
  return stat(p.c_str(), &st) == 0 && S_ISDIR(st.st_mode);
}

bool is_file(const std::string& p) {
  struct stat st{};
  return stat(p.c_str(), &st) == 0 && S_ISREG(st.st_mode);
}

// <cache root>/<hash of the kernel headers>/: modules of other header versions
// sit in sibling directories (never loaded; build scripts prune them)
}  // namespace

std::string cache_dir() {
  const char* v = std::getenv("P2S_JIT_CACHE");
  const std::string root = v ? v : lib_dir() + "/jit";
  if (!is_dir(root)) mkdir(root.c_str(), 0755);
  return root + "/" + P2S_SRC_HASH;
}

namespace {

std::string src_dir() {
  if (const char* v = std::getenv("P2S_JIT_SRC")) return v;
  return lib_dir() + "/csrc";
}

std::string nvcc_path() {
  if (const char* v = std::getenv("P2S_NVCC")) return v;
  if (const char* h = std::getenv("CUDA_HOME")) {
    const std::string p = std::string(h) + "/bin/nvcc";
    if (is_file(p)) return p;
  }
  if (is_file("/usr/local/cuda/bin/nvcc")) return "/usr/local/cuda/bin/nvcc";
  return "nvcc";
}

const char* kFlags =
    "-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr "
    "-Xcompiler -fPIC -shared -cudart shared -Xptxas -v -DP2S_LEAN";

struct Loaded {
  std::mutex mu;  // held while this shape's module is compiled / loaded
  void* handle = nullptr;
  reg::JitEntries entries{};
};

std::mutex g_mu;                                          // guards the map only
std::map<std::string, std::unique_ptr<Loaded>> g_loaded;  // key -> module (process lifetime)

std::string full_source(const Plan& pl) {
  return std::string("// generated by p2s_jit (libp2s_b200): ") + pl.desc + "\n#include \"p2s_jit_module.cuh\"\n" +
         pl.source;
}

std::string key_of(const Plan& pl) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%016llx",
                static_cast<unsigned long long>(fnv1a(std::string(P2S_SRC_HASH) + "\n" + kFlags + "\n" + full_source(pl))));
  return buf;
}

bool compile(const Plan& pl, const std::string& dir, const std::string& key, std::string* err) {
  if (!is_dir(dir) && mkdir(dir.c_str(), 0755) != 0 && !is_dir(dir)) {
    *err = "cannot create the kernel module cache " + dir;
    return false;
  }
  const std::string inc = src_dir();
  if (!is_file(inc + "/p2s_jit_module.cuh")) {
    *err = "kernel headers not found in " + inc + " (set P2S_JIT_SRC)";
    return false;
  }
  std::ostringstream tag;
  tag << getpid() << "_" << std::hash<std::thread::id>()(std::this_thread::get_id());
  const std::string base = dir + "/p2s_jit_" + key;
  const std::string cu = base + "." + tag.str() + ".cu", tmp = base + "." + tag.str() + ".so";
  {
    FILE* f = std::fopen(cu.c_str(), "w");
    if (!f) {
      *err = "cannot write " + cu;
      return false;
    }
    const std::string src = full_source(pl);
    std::fwrite(src.data(), 1, src.size(), f);
    std::fclose(f);
  }
  const std::string cmd = nvcc_path() + " " + kFlags + " -I'" + inc + "' '" + cu + "' -o '" + tmp + "' > '" +
                          base + ".log' 2>&1";
  const int rc = std::system(cmd.c_str());
  if (rc != 0 || !is_file(tmp)) {
    std::string log;
    if (FILE* f = std::fopen((base + ".log").c_str(), "r")) {
      char b[4096];
      size_t n = 0;
      while ((n = std::fread(b, 1, sizeof(b), f)) > 0 && log.size() < 2000) log.append(b, n);
      std::fclose(f);
    }
    *err = "nvcc failed (" + cmd + "): " + log.substr(0, 1500);
    std::remove(tmp.c_str());
    return false;
  }
  std::rename(cu.c_str(), (base + ".cu").c_str());
  if (std::rename(tmp.c_str(), (base + ".so").c_str()) != 0) {  // atomic publish
    *err = "cannot publish " + base + ".so";
    return false;
  }
  return true;
}

}  // namespace

bool plan(const p2s_problem& eff, Plan* pl, std::string* why, const Overrides& ov) {
  Desc d{};
  for (int k = 0; k < 3; ++k) {
    d.N[k] = eff.order[k];
    d.Q[k] = eff.nq[k];
  }
  d.S = eff.n_terms;
  for (int s = 0; s < d.S; ++s)
    for (int k = 0; k < 3; ++k) d.kind[s][k] = eff.kind[s][k];
  if (ov.family != kFamilyLarge && plan_fused(d, pl, ov)) return true;
  if (ov.family == kFamilyFused) {
    *why = "no fused-family instantiation fits this shape (with these overrides)";
    return false;
  }
  return plan_large(d, pl, why, ov);
}

const reg::JitEntries* module(const Plan& pl, std::string* err) {
  const std::string key = key_of(pl);
  Loaded* L = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto& slot = g_loaded[key];
    if (!slot) slot = std::make_unique<Loaded>();
    L = slot.get();
  }
  std::lock_guard<std::mutex> lock(L->mu);  // one compile per shape per process; shapes in parallel
  if (L->handle) return &L->entries;
  const std::string dir = cache_dir();
  const std::string so = dir + "/p2s_jit_" + key + ".so";
  if (!is_file(so) && !compile(pl, dir, key, err)) return nullptr;
  void* h = dlopen(so.c_str(), RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    *err = std::string("dlopen ") + so + ": " + dlerror();
    return nullptr;
  }
  using entry_fn = int (*)(reg::JitEntries*);
  auto fn = reinterpret_cast<entry_fn>(dlsym(h, "p2s_jit_entry"));
  reg::JitEntries e{};
  if (!fn || fn(&e) != 0 || e.abi != reg::kJitAbi) {
    *err = "module " + so + " has no compatible p2s_jit_entry";
    dlclose(h);
    return nullptr;
  }
  L->entries = e;
  L->handle = h;
  return &L->entries;
}

bool cached(const Plan& pl) { return is_file(cache_dir() + "/p2s_jit_" + key_of(pl) + ".so"); }

bool compiler_available() {
  const std::string n = nvcc_path();
  if (n.find('/') != std::string::npos) return is_file(n);
  return std::system("command -v nvcc > /dev/null 2>&1") == 0;
}

std::string module_path(const Plan& pl) { return cache_dir() + "/p2s_jit_" + key_of(pl) + ".so"; }

}  // namespace jit
}  // namespace p2s
