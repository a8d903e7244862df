// p2s_reg_large.cu -- large-order registry (C5: large_moments_w_kernel, large_w_kernel, large_v_kernel,
// large_u_xs_kernel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cstdint>

#include "p2s_reg_large.cuh"

namespace p2s {
namespace reg {

// ------------------------------------------------------------ large-order registry


const std::vector<LargeEntry>& large_registry() {
  static const std::vector<LargeEntry> reg = {
      // C5; moment chunks of 8 (w-first tiled kernel: 169 KB, one CTA of 352 threads per SM,
      // 0.94 us per element vs 1.05 with chunks of 4; the round-1 u-first kernel preferred 4)
      make_large<LShape<16, 16, 16, 36, 36, 36, 8, kPPP, kDDD>>(),
      make_large<LShape<5, 4, 3, 8, 8, 6, 4, kPPP, kDDD>>(),         // test shape
      make_large<LShape<5, 4, 3, 8, 8, 6, 4, kCPPP, kCDDD>>(),       // test shape, conforming
  };
  return reg;
}

}  // namespace reg
}  // namespace p2s
