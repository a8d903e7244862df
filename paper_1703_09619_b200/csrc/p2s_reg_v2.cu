// p2s_reg_v2.cu -- shape-specialised contraction (contract_v2_kernel) and moment (moments_v2_kernel) registries.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "p2s_reg_v2.cuh"

namespace p2s {
namespace reg {

// ------------------------------------------------------------ shape-specialised registry


// <N_u, N_v, N_w, n1 tile, p1 tile, threads, min CTAs/SM, A once per unit, fibers per
//  thread, term kinds...>.  Several variants per shape: the first is the default,
//  P2S_V2_VARIANT=k selects the k-th match (tuning).
const std::vector<V2Entry>& v2_registry() {
  static const std::vector<V2Entry> reg = {
      // <NU, NV, NW, T, P1T (= NW), PG (= NW), threads, minB,
      //  flags (1 AALL, 2 ROWLOOP, 4 SYM, 8 PERSIST), FPT, kinds...>
      make_v2<Shape<4, 4, 4, 4, 4, 4, 256, 2, 4, 1, kPPP>>(),                 // C1
      make_v2<Shape<6, 6, 6, 2, 6, 6, 256, 2, 4, 2, kPPP, kDDD>>(),           // C2
      make_v2<Shape<6, 6, 6, 1, 6, 6, 224, 2, 4, 1, kPPP, kDDD>>(),
      make_v2<Shape<6, 6, 6, 2, 6, 6, 256, 2, 0, 2, kPPP, kDDD>>(),
      // C3 (persistent SYM variants <..., 256, 1, 12, 1|2> were dropped: both fault with an
      // illegal address at 255 registers + 100-140 B of stack even for one element,
      // where they execute the non-persistent code path; unused, never a default)
      // C3 default: parity-split stage C (half the register-resident fiber: 90 registers)
      // with 512 threads and a runtime row loop: 2.45 M elem/s (0.873) vs 2.37 M (0.84) for
      // the 256-thread banded kernels below (254 registers, 8 warps per SM);
      // profiles/r2_c3_v2_variants.txt.  1, 2 = 256 threads banded (FPT 1 / 2), 3 = 512
      // threads with unrolled rows (126 registers, 2.32 M), 4 = 384 threads (2.28 M)
      make_v2<Shape<8, 8, 8, 1, 8, 8, 512, 1, 70, 1, kPPP, kDDD>>(),          // C3
      make_v2<Shape<8, 8, 8, 1, 8, 8, 256, 1, 4, 1, kPPP, kDDD>>(),
      make_v2<Shape<8, 8, 8, 1, 8, 8, 256, 1, 4, 2, kPPP, kDDD>>(),
      make_v2<Shape<8, 8, 8, 1, 8, 8, 512, 1, 68, 1, kPPP, kDDD>>(),
      make_v2<Shape<8, 8, 8, 1, 8, 8, 384, 1, 70, 1, kPPP, kDDD>>(),
      // (C3 banded, not parity split, at 384 / 512 threads: 168 / 128 registers with
      // 284 / 256 B of spills, 1.96 M / 2.07 M elem/s)
      make_v2<Shape<10, 6, 4, 2, 4, 4, 192, 2, 6, 1, kPPP, kDDD>>(),          // C4
      make_v2<Shape<10, 6, 4, 2, 4, 4, 192, 2, 4, 1, kPPP, kDDD>>(),
      make_v2<Shape<10, 6, 4, 2, 4, 4, 192, 2, 2, 1, kPPP, kDDD>>(),
      make_v2<Shape<3, 3, 3, 3, 3, 3, 96, 4, 0, 1, kPPP, kDDD>>(),            // test shapes
      make_v2<Shape<3, 3, 3, 1, 3, 3, 64, 4, 12, 2, kPPP, kDDD>>(),
      make_v2<Shape<4, 3, 3, 3, 3, 3, 96, 4, 2, 1, enc_kind(DP, PD, PP), enc_kind(PD, DP, DD)>>(),
      make_v2<Shape<4, 3, 3, 3, 3, 3, 96, 4, 18, 1, enc_kind(DP, PD, PP), enc_kind(PD, DP, DD)>>(),
      make_v2<Shape<3, 3, 3, 3, 3, 3, 96, 4, 20, 1, kPPP, kDDD>>(),
      make_v2<Shape<3, 3, 3, 3, 3, 3, 96, 4, 64, 2, kPPP, kDDD>>(),
      make_v2<Shape<4, 3, 3, 3, 3, 3, 96, 4, 66, 2, enc_kind(DP, PD, PP), enc_kind(PD, DP, DD)>>(),
      // conforming basis
      make_v2<Shape<6, 6, 6, 2, 6, 6, 256, 2, 4, 2, kCPPP, kCDDD>>(),
      make_v2<Shape<3, 3, 3, 3, 3, 3, 96, 4, 0, 1, kCPPP, kCDDD>>(),
  };
  return reg;
}


// ------------------------------------------------------------ shape-specialised moments


// <N_u, N_v, N_w, nq_u, nq_v, nq_w, threads, term kinds...>
const std::vector<MV2Entry>& mv2_registry() {
  static const std::vector<MV2Entry> reg = {
      make_mv2<MShape<4, 4, 4, 8, 8, 8, 128, kPPP>>(),                    // C1
      make_mv2<MShape<6, 6, 6, 14, 14, 14, 256, kPPP, kDDD>>(),           // C2
      make_mv2<MShape<8, 8, 8, 20, 20, 20, 512, kPPP, kDDD>>(),           // C3 (512 threads)
      make_mv2<MShape<10, 6, 4, 16, 16, 16, 256, kPPP, kDDD>>(),          // C4
      make_mv2<MShape<3, 3, 3, 6, 6, 6, 128, kPPP, kDDD>>(),              // test shapes
      make_mv2<MShape<4, 3, 3, 9, 5, 7, 128, enc_kind(DP, PD, PP), enc_kind(PD, DP, DD)>>(),
      make_mv2<MShape<5, 5, 5, 9, 9, 9, 128, kPPP, kDDD>>(),
      // thread-count variants (P2S_MV2_VARIANT), FP64 TF/s of the C3 moments kernel:
      // C3 0 = 512 (25.8, default), 1 = 200 (18.9), 2 = 320 (21.2), 3 = 400 (25.6),
      // 4 = 256 (19.8); C4 1 = 192, 2 = 384 and C2 1 = 128, 2 = 196 (all within 2 % of
      // their 256-thread defaults)
      make_mv2<MShape<8, 8, 8, 20, 20, 20, 200, kPPP, kDDD>>(),
      make_mv2<MShape<8, 8, 8, 20, 20, 20, 320, kPPP, kDDD>>(),
      make_mv2<MShape<8, 8, 8, 20, 20, 20, 400, kPPP, kDDD>>(),
      make_mv2<MShape<8, 8, 8, 20, 20, 20, 256, kPPP, kDDD>>(),
      make_mv2<MShape<10, 6, 4, 16, 16, 16, 192, kPPP, kDDD>>(),
      make_mv2<MShape<10, 6, 4, 16, 16, 16, 384, kPPP, kDDD>>(),
      make_mv2<MShape<6, 6, 6, 14, 14, 14, 128, kPPP, kDDD>>(),
      make_mv2<MShape<6, 6, 6, 14, 14, 14, 196, kPPP, kDDD>>(),
  };
  return reg;
}

}  // namespace reg
}  // namespace p2s
