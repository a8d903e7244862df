// p2s_reg_fused.cu -- fused fill registry (fill_fused_kernel: moments + contraction in one kernel; geometry modes).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "p2s_fused.cuh"
#include "p2s_reg_common.cuh"

namespace p2s {
namespace reg {

// ------------------------------------------------------------ fused fill registry


// GEO > 0: `alpha` is the geometry records and the kernel computes the coupling
// factors itself (xq = the GL nodes u, v, w appended to mpack); GEO == 2 launches
// one thread-block cluster of P CTAs per element (non-portable size for P = 9)
template <class Sh, class Ms, int GEO = 0, bool PF = true>
cudaError_t launch_fused(const double* alpha, double* M, int64_t ldM, int64_t n_tot, int64_t n_elem,
                         int nc, int P, int Nt, const std::vector<double>& cpack,
                         const std::vector<double>& mpack, const double* amma, cudaStream_t st,
                         int num_sms) {
  FusedParams<Sh, Ms> p;
  p.geom = GEO ? alpha : nullptr;
  if constexpr (GEO != 0)
    std::memcpy(p.xq, mpack.data() + Ms::TALL, sizeof(double) * (Ms::Q(0) + Ms::Q(1) + Ms::Q(2)));
  p.c.I = nullptr;
  p.c.M = M;
  p.c.ldM = ldM;
  p.c.mat_stride = n_tot * ldM;
  p.c.n_units = n_elem * P;
  p.c.nc = nc;
  p.c.P = P;
  p.c.Nt = Nt;
  p.c.mom_per_elem = 0;
  p.c.amma = amma;
  p.c.vec2 = vec2_ok(M, ldM);
  p.c.prefetch_stride = 0;  // (contract_v2 only)
  std::memcpy(p.c.cu, cpack.data(), sizeof(double) * Sh::ctot(0));
  std::memcpy(p.c.cv, cpack.data() + Sh::ctot(0), sizeof(double) * Sh::ctot(1));
  std::memcpy(p.c.cw, cpack.data() + Sh::ctot(0) + Sh::ctot(1), sizeof(double) * Sh::ctot(2));
  p.alpha = alpha;
  p.prefetch_stride = 0;
  std::memcpy(p.tab, mpack.data(), sizeof(double) * Ms::TALL);
  if (p.c.n_units == 0) return cudaSuccess;
  constexpr size_t smem = FusedLayout<Sh, Ms, GEO>::SMEM;
  static int blocks_per_sm = -1;
  if (blocks_per_sm < 0) {
    cudaError_t e = cudaFuncSetAttribute(fill_fused_kernel<Sh, Ms, GEO>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if constexpr (GEO == 2) {
      e = cudaFuncSetAttribute(fill_fused_kernel<Sh, Ms, GEO>,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fill_fused_kernel<Sh, Ms, GEO>, Sh::THREADS,
                                                      smem);
    if (e != cudaSuccess) return e;
    if (b < 1) return cudaErrorInvalidConfiguration;
    blocks_per_sm = b;
  }
  const int64_t resident = static_cast<int64_t>(blocks_per_sm) * num_sms;
  const int64_t grid = Sh::PERSIST ? std::min<int64_t>(p.c.n_units, resident) : p.c.n_units;
  // L2 prefetch of the alpha of the unit that takes this SM slot next (PF, per
  // shape; P2S_PREFETCH_AHEAD=k overrides): C2 +0.6 %, C4 -1.5 % (L2 pressure)
  p.prefetch_stride = PF ? resident : 0;
  if (const char* v = std::getenv("P2S_PREFETCH_AHEAD")) p.prefetch_stride = resident * std::max(0, std::atoi(v));
  if constexpr (GEO == 2) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(p.c.n_units));
    cfg.blockDim = dim3(Sh::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(P);  // one element per cluster
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fill_fused_kernel<Sh, Ms, GEO>, p);
  }
  fill_fused_kernel<Sh, Ms, GEO><<<static_cast<unsigned>(grid), Sh::THREADS, smem, st>>>(p);
  return cudaGetLastError();
}


template <class Sh, class Ms, bool WITH_GEO = false, bool PREFER_TWO_STAGE = false, bool PF = true>
FusedEntry make_fused() {
  FusedEntry r{};
  for (int d = 0; d < 3; ++d) {
    r.order[d] = Sh::N(d);
    r.nq[d] = Ms::Q(d);
  }
  r.S = Sh::S;
  for (int s = 0; s < Sh::S; ++s)
    for (int d = 0; d < 3; ++d) r.kinds[s][d] = Sh::kind(s, d);
  r.launch = &launch_fused<Sh, Ms, 0, PF>;
  r.launch_geo = r.launch_geo_cluster = nullptr;
  if constexpr (WITH_GEO) {
    r.launch_geo = &launch_fused<Sh, Ms, 1>;
    r.launch_geo_cluster = &launch_fused<Sh, Ms, 2>;
  }
  r.cpack = &pack_v2<Sh>;
  r.mpack = &pack_mv2<Ms>;
  r.mma_pack = &pack_mma<Sh>;
  r.desc = stage_c_desc<Sh>();
  r.prefer_two_stage = PREFER_TWO_STAGE;
  return r;
}

// <Shape: N_u, N_v, N_w, n1 tile, p1 tile, p1 group, threads, min CTAs/SM, flags, FPT, kinds>
// flags: 1 AALL, 2 ROWLOOP, 4 SYM, 8 PERSIST, 16 MMA (stage C on DMMA), 32 PAIR (16-B
// stores), 64 PSPLIT (parity-split stage C), 128 NOUSYM, 256 QUAD (32-B stores),
// 512 NSYM ((n1, n2)-symmetric stage C).  The first match of a problem is the
// default; P2S_FUSED_VARIANT=k selects the k-th (tuning / A-B measurements, see
// profiles/README.md for the numbers behind each default).
const std::vector<FusedEntry>& fused_registry() {
  static const std::vector<FusedEntry> reg = {
      make_fused<Shape<4, 4, 4, 4, 4, 4, 256, 2, 4, 1, kPPP>,
                 MShape<4, 4, 4, 8, 8, 8, 256, kPPP>>(),                              // C1
      // C2: 0 banded (default, also compiled in geometry mode), 1 paired stores,
      // 2 parity split, 3 DMMA
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 4, 2, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>, true>(),
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 36, 2, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 68, 2, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 20, 1, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      // C2: 4 parity split + paired (FPT 2), 5 same FPT 4
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 100, 2, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 100, 4, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      // C3: p2s_fill runs the two-stage path by default (moments_v2 + contract_v2 over
      // 256 MB chunks, the next chunk's moments overlapping this chunk's contraction:
      // 2.29-2.31 M elem/s vs 2.26 M fused -- the fused kernel fits one 223 KB CTA per
      // SM, so its moment phase never overlaps another CTA's stores); fused variants (via
      // P2S_FUSED_VARIANT): 0 paired stores, 1 banded, 2 parity split + paired, 3 DMMA
      make_fused<Shape<8, 8, 8, 1, 8, 8, 256, 1, 38, 2, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>, false, true>(),
      make_fused<Shape<8, 8, 8, 1, 8, 8, 256, 1, 6, 2, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>>(),
      make_fused<Shape<8, 8, 8, 1, 8, 8, 256, 1, 102, 2, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>>(),
      make_fused<Shape<8, 8, 8, 1, 8, 8, 256, 1, 22, 1, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>>(),
      // C4: 0 parity split with n1 tiles of 2, 2 CTAs of 256 threads per SM (default:
      // 1.174 M elem/s; 192 threads 1.133 M, n1 tiles of 3 1.009 M, 2 fibers/thread
      // 1.105 M), 1 the same at 192 threads, then parity split with all six n1 per tile
      // and 2 fibers / thread (1 CTA of 288 threads per SM, 1.104 M), banded, paired
      // stores, DMMA
      make_fused<Shape<10, 6, 4, 2, 4, 4, 256, 2, 70, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 256, kPPP, kDDD>, false, false, false>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 70, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 6, 4, 4, 288, 1, 70, 2, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 288, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 6, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 38, 2, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 22, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      // C2 in the conforming basis
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 4, 2, kCPPP, kCDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      // C4 w-last contraction (p2s_contract_wl.cuh): 5 (TM 11), 6 (TM 19)
      make_fused<WShape<10, 6, 4, 11, 192, 2, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_fused<WShape<10, 6, 4, 19, 256, 2, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 256, kPPP, kDDD>>(),
      // 32-B stores (QUAD, flag 256: st.global.v4.f64): C2 variant 6 (FPT 4, spills),
      // C3 variants 4 (FPT 4; 1.75 M vs 2.21 M default) and 5 (+ parity split; 2.01 M),
      // C4 variant 7 (parity split, FPT 4; 0.97 M vs 1.11 M): the 4 fibers per thread
      // cost more (registers) than the halved store count gains
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 260, 4, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      make_fused<Shape<8, 8, 8, 1, 8, 8, 256, 1, 262, 4, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>>(),
      make_fused<Shape<8, 8, 8, 1, 8, 8, 256, 1, 326, 4, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 6, 4, 4, 288, 1, 326, 4, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 288, kPPP, kDDD>>(),
      // (n1, n2)-symmetric stage C (NSYM, flag 512): C2 variant 7 (1.26 M vs 1.69 M),
      // C3 variant 6 (1.87 M vs 2.19 M), C4 variant 8 (1.04 M vs 1.11 M): 42 % fewer
      // stage-C DFMAs, but the mirrored stores (row n2, N_w-double runs) are poorly
      // coalesced and the later n1 tiles leave threads idle
      make_fused<Shape<6, 6, 6, 2, 6, 6, 256, 2, 516, 2, kPPP, kDDD>,
                 MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),
      make_fused<Shape<8, 8, 8, 1, 8, 8, 256, 1, 550, 2, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 6, 4, 4, 288, 1, 582, 2, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 288, kPPP, kDDD>>(),
      // (C2 at 288 / 320 threads, 96 registers: 1.694 M / 1.698 M burst, 1.486 M / 1.488 M
      // at 1000 steps vs 1.705 M / 1.504 M for the 256-thread default)
      // test shapes
      make_fused<Shape<3, 3, 3, 3, 3, 3, 96, 4, 0, 1, kPPP, kDDD>,
                 MShape<3, 3, 3, 6, 6, 6, 96, kPPP, kDDD>>(),
      make_fused<Shape<4, 3, 3, 3, 3, 3, 96, 4, 0, 1, enc_kind(DP, PD, PP), enc_kind(PD, DP, DD)>,
                 MShape<4, 3, 3, 9, 5, 7, 96, enc_kind(DP, PD, PP), enc_kind(PD, DP, DD)>>(),
  };
  return reg;
}

}  // namespace reg
}  // namespace p2s
