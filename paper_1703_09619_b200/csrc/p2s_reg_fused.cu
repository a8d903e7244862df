// p2s_reg_fused.cu -- fused fill registry (fill_fused_kernel: moments + contraction in one kernel; geometry modes).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "p2s_reg_fused.cuh"

namespace p2s {
namespace reg {

// <Shape: N_u, N_v, N_w, n1 tile, p1 tile, p1 group, threads, min CTAs/SM, flags, FPT, kinds>
// flags: 1 AALL, 2 ROWLOOP, 4 SYM, 8 PERSIST, 16 MMA (stage C on DMMA), 32 PAIR (16-B
// stores), 64 PSPLIT (parity-split stage C), 128 NOUSYM, 256 QUAD (32-B stores),
// 512 NSYM ((n1, n2)-symmetric stage C), 1024 AL1 (alpha loads allocate in L1).  The first match of a problem is the
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
      // (round 2: alpha loads without L1 allocation +2 %; with them the L2 prefetch of
      // the next unit's alpha, 1.5 % slower in round 1, gains 1.6 %: 1.166 M vs 1.148 M,
      // tools/gpu_ab_c4pf.sh; variant 7 = prefetch off)
      make_fused<Shape<10, 6, 4, 2, 4, 4, 256, 2, 70, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 256, kPPP, kDDD>, false, false, true>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 70, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 256, 2, 1094, 1, kPPP, kDDD>,   // 2: default with L1-allocating alpha loads
                 MShape<10, 6, 4, 16, 16, 16, 256, kPPP, kDDD>, false, false, false>(),
      make_fused<Shape<10, 6, 4, 6, 4, 4, 288, 1, 70, 2, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 288, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 6, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 38, 2, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_fused<Shape<10, 6, 4, 2, 4, 4, 192, 2, 22, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      // C4 default without the L2 prefetch of the next unit's alpha (variant 7)
      make_fused<Shape<10, 6, 4, 2, 4, 4, 256, 2, 70, 1, kPPP, kDDD>,
                 MShape<10, 6, 4, 16, 16, 16, 256, kPPP, kDDD>, false, false, false>(),
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
      // C3 variant 7: parity split, 512 threads, row loop (as the two-stage default)
      make_fused<Shape<8, 8, 8, 1, 8, 8, 512, 1, 70, 1, kPPP, kDDD>,
                 MShape<8, 8, 8, 20, 20, 20, 512, kPPP, kDDD>>(),
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
