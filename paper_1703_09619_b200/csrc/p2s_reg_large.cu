// p2s_reg_large.cu -- large-order registry (C5: large_moments_kernel, large_w_kernel, large_v_kernel,
// large_u_kernel).
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
      // C5; k1 chunks of 4 (79 KB, 2 CTAs/SM): moments 0.71 ms vs 0.97 ms with chunks of 8
      make_large<LShape<16, 16, 16, 36, 36, 36, 4, kPPP, kDDD>>(),
      make_large<LShape<5, 4, 3, 8, 8, 6, 4, kPPP, kDDD>>(),         // test shape
      make_large<LShape<5, 4, 3, 8, 8, 6, 4, kCPPP, kCDDD>>(),       // test shape, conforming
  };
  return reg;
}

}  // namespace reg
}  // namespace p2s
