// p2s_registry.hpp -- the shape registries shared by the C-ABI (p2s_capi.cu)
// and the translation units that instantiate the kernels (p2s_reg_*.cu, built
// in parallel): entry structs, launch / pack function types and accessors.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/p2s_b200.h"
#include "p2s_kernels.cuh"
#include "p2s_tables.hpp"

namespace p2s {
namespace reg {

struct ContractArgs {
  const double* I;
  double* M;
  int64_t ldM, n_tot, n_elem;
  int nc, P, Nv, Nw, Nt;
  int S;
  int Kv[kMaxTerms], Kw[kMaxTerms], kind_v[kMaxTerms], kind_w[kMaxTerms];
  int64_t mom_per_elem, mom_per_pair, mom_off[kMaxTerms];
  const double* Cv[kMaxTerms];
  const double* Cw[kMaxTerms];
  const double* cu_packed;  // host, Cfg-packed
};

struct Plan {  // per-context launch geometry of the contraction
  int G, NG, threads;
  size_t smem;
};

using contract_fn = cudaError_t (*)(const ContractArgs&, const Plan&, cudaStream_t);

struct RegEntry {
  int NU, S;
  int kinds[kMaxTerms];
  contract_fn launch;
  std::vector<double> (*pack)(const std::vector<const std::vector<double>*>&);
  int ktot;
};

struct V2Args {
  const double* I;
  double* M;
  int64_t ldM, n_tot, n_elem, mom_per_elem;
  int nc, P, Nt;
  const std::vector<double>* dense[kMaxTerms][3];  // [N][N][K] per term, direction
  const double* amma;                              // device stage-C A (MMA shapes)
};

using v2_fn = cudaError_t (*)(const V2Args&, const std::vector<double>&, cudaStream_t, int);

using v2_pack_fn = std::vector<double> (*)(const V2Args&);

struct V2Entry {
  int order[3];
  int S;
  int kinds[kMaxTerms][3];
  v2_fn launch;
  v2_pack_fn pack;
  v2_pack_fn mma_pack;
  size_t smem;
  const char* desc;
};

using mv2_fn = cudaError_t (*)(const double*, double*, int64_t, int, int64_t,
                               const std::vector<double>&, cudaStream_t);

using mv2_pack_fn = std::vector<double> (*)(const std::vector<double> (*)[3]);

struct MV2Entry {
  int order[3], nq[3], S;
  int kinds[kMaxTerms][3];
  mv2_fn launch;
  mv2_pack_fn pack;
};

// (alpha or geometry records, M, ld_M, n_tot, n_elem, n_comp, P, Nt, band-packed
//  coefficients, weighted tables, DMMA operands, stream, SM count, Jacobian flag)
using fused_fn = cudaError_t (*)(const double*, double*, int64_t, int64_t, int64_t, int, int, int,
                                 const std::vector<double>&, const std::vector<double>&,
                                 const double*, cudaStream_t, int, int*);

struct FusedEntry {
  int order[3], nq[3], S;
  int kinds[kMaxTerms][3];
  fused_fn launch;
  fused_fn launch_geo;          // coupling factors from geometry records, per unit
  fused_fn launch_geo_cluster;  // ... shared per element through a cluster (DSMEM)
  v2_pack_fn cpack;
  mv2_pack_fn mpack;
  v2_pack_fn mma_pack;
  const char* desc;
  // p2s_fill runs the two-stage path (moments_v2 + contract_v2) for this shape
  // unless P2S_FUSED_VARIANT asks for a fused kernel: measured faster (C3)
  bool prefer_two_stage;
};

struct LargeArgs {
  const std::vector<double> (*phi)[3];            // [s][d] full tables
  const std::vector<double>* dense[kMaxTerms][3];  // [s][d] [N][N][K]
};

struct LargePack {
  std::vector<double> tab, cu, cvw;  // cvw: band-packed Cv then Cw (kernel parameters)
  double* d_Z = nullptr;             // w-step output of one chunk (ZPU x xchunk doubles)
  double* d_cu = nullptr;            // device copy of cu (shared-memory / global-memory coefficients)
  double* d_cvw = nullptr;           // device copy of cvw (global-memory coefficients)
  double* d_T1 = nullptr;            // split moments: u-pass output of a sub-batch (L2-resident)
  int64_t t1_units = 0;              // (unit, term)s per sub-batch
  bool mom_split = false;            // P2S_LARGE_MSPLIT: split moment stage (u pass / v-w passes;
                                     // measured C5 1.33 vs 1.27 us/elem: the v/w passes dominate)
  bool u_xs = true;                  // P2S_LARGE_XS: next class staged by cp.async (C5 29.4 k vs 28.4 k)
  bool u_bulk = false;               // P2S_LARGE_UBULK: u-stage rows written with TMA bulk stores
                                     // (measured slower: c12 0.56 vs 0.59, C5 0.55 vs 0.65 of HBM)
  bool u_pair = false;               // P2S_LARGE_UPAIR: two adjacent fibers per u-stage thread
                                     // (measured slower: c12 0.53 vs 0.58, C5 0.59 vs 0.65 of HBM)
  int u_roll = 1;                    // P2S_LARGE_UROLL: runtime row loop (1) or unrolled rows (0, slower)
  bool mom_wfirst = true;            // P2S_LARGE_MOMW: w-first register-tiled moment kernel (coalesced alpha reads;
                                     // C5 1.00 vs 1.24 us per element); 0: the u-first kernel, one row per thread
  bool mom_tiled = false;            // P2S_LARGE_MOMT: register-tiled passes (two rows x KG polynomials per thread)
  bool mom_grouped = false;          // P2S_LARGE_MOMG: (row, k group) items in the v / w passes, staged tables
  bool mom_cluster = false;          // P2S_LARGE_MOMCL: one cluster per (unit, term), alpha read once (0.77 vs 0.71 ms: slower)
  bool u_smemc = false;              // P2S_LARGE_USMEM (measured 28.1 k vs 28.4 k elem/s constant-bank)
  // runtime: parity-split u stage; v/w of chunk i+1 on `aux` overlapping u of
  // chunk i (X double-buffered), ordered by events; two_u: the u stages of
  // consecutive chunks alternate between the caller's stream and `aux_u`, so the
  // tail wave of one overlaps the start of the next
  bool ps = true, overlap = true, two_u = true;
  int64_t u_ctas = -1;  // u-stage grid: persistent, resident CTAs (-1), k CTAs (> 0), one per tile (0)
  int num_sms = 148;
  int ufib = 1;  // u-stage fibers per thread (P2S_LARGE_FIB; 2 measured 18 % slower)
  int v_split = 0;  // P2S_LARGE_VSPLIT: the n1 rows of a v-step item are dealt to up to N_v CTAs until
                    // the step has this many waves of 2 CTAs per SM (0: one CTA per item; measured
                    // slower: C5 0.65 -> 0.64 / 0.62 at 4 / 8 waves, c12 0.605 -> 0.573 / 0.53)
  cudaStream_t aux = nullptr, aux_u = nullptr;
  cudaEvent_t ev_start = nullptr, ev_join = nullptr, ev_vw[2]{}, ev_u[2]{};
};

using large_pack_fn = bool (*)(const LargeArgs&, LargePack&);

using large_mom_fn = cudaError_t (*)(const double*, double*, int64_t, const LargePack&, cudaStream_t);

using large_con_fn = cudaError_t (*)(const double*, double*, double*, int64_t, int64_t, int64_t, int,
                                     int, int, const LargePack&, cudaStream_t);

struct LargeEntry {
  int order[3], nq[3], S;
  int kinds[kMaxTerms][3];
  large_pack_fn pack;
  large_mom_fn moments;
  large_con_fn contract;
  int64_t mpp, xpu, zpu;
  int64_t t1u;  // split moments: T1 scratch per (unit, term), doubles
};

// Registry entries of one generated per-shape module (p2s_jit.cu,
// p2s_jit_module.cuh); kJitAbi changes whenever these structs change.
constexpr int kJitAbi = 5;
struct JitEntries {
  int abi, family;   // family: 1 fused (+ two-stage entries of the shape), 2 large
  FusedEntry fused;
  V2Entry v2;
  MV2Entry mv2;
  LargeEntry large;
  size_t smem;       // shared memory of the dominant kernel as compiled (bytes)
  int64_t mpp;       // moment block of one pair as compiled (doubles)
};

// accessors (one translation unit each)
const std::vector<RegEntry>& registry();         // p2s_reg_generic.cu
const std::vector<V2Entry>& v2_registry();       // p2s_reg_v2.cu
const std::vector<MV2Entry>& mv2_registry();     // p2s_reg_v2.cu
const std::vector<FusedEntry>& fused_registry(); // p2s_reg_fused.cu
const std::vector<LargeEntry>& large_registry(); // p2s_reg_large.cu
// runtime-shaped moment kernel (p2s_reg_generic.cu)
cudaError_t launch_moments(int kmax, const MomentParams& p, size_t smem, cudaStream_t st);

}  // namespace reg
}  // namespace p2s
