// p2s_reg_common.cuh -- template helpers shared by the v2 and fused registry
// translation units: coefficient packing, stage-C descriptions, term-kind codes.
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

#include "p2s_contract_v2.cuh"
#include "p2s_moments_v2.cuh"
#include "p2s_registry.hpp"

namespace p2s {
namespace reg {

constexpr int kPPP = enc_kind(PP, PP, PP);
constexpr int kDDD = enc_kind(DD, DD, DD);
constexpr int kCPPP = enc_kind(PP | kConforming, PP | kConforming, PP | kConforming);
constexpr int kCDDD = enc_kind(DD | kConforming, DD | kConforming, DD | kConforming);

template <class Sh>
std::vector<double> pack_v2(const V2Args& a) {
  std::vector<double> out(static_cast<size_t>(Sh::ctot(0) + Sh::ctot(1) + Sh::ctot(2)), 0.0);
  const int base[3] = {0, Sh::ctot(0), Sh::ctot(0) + Sh::ctot(1)};
  for (int d = 0; d < 3; ++d)
    for (int s = 0; s < Sh::S; ++s) {
      const int K = Sh::K(s, d), kd = Sh::kind(s, d), N = Sh::N(d);
      const std::vector<double>& C = *a.dense[s][d];
      for (int x = 0; x < N; ++x)
        for (int y = 0; y < N; ++y) {
          const int lo = band_lo(kd, x, y), cnt = band_count(kd, x, y);
          const int co = Sh::coff(d, s, x, y);
          for (int j = 0; j < cnt; ++j)
            out[static_cast<size_t>(base[d] + co + j)] =
                C[(static_cast<size_t>(x) * N + y) * K + lo + band_step(kd, x, y) * j];
        }
    }
  return out;
}

// fragment-ordered stage-C A of an MMA shape (empty otherwise)
template <class Sh>
std::vector<double> pack_mma(const V2Args& a) {
  if constexpr (Sh::MMA) {
    const std::vector<double>* d[kMaxTerms];
    for (int s = 0; s < Sh::S; ++s) d[s] = a.dense[s][0];
    return build_mma_a<Sh>(d);
  } else {
    return {};
  }
}

// widest vector store the M rows allow: 4 (32-B aligned rows), 2 (16-B), else 0
inline int vec2_ok(const double* M, int64_t ldM) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(M);
  if (ldM % 4 == 0 && a % 32 == 0) return 4;
  return (ldM % 2 == 0 && a % 16 == 0) ? 2 : 0;
}

template <class Sh>
constexpr const char* stage_c_desc() {
  if constexpr (!Sh::WLAST && Sh::NSYM)
    return Sh::PSPLIT ? "banded stage C, parity split, (n1, n2)-symmetric"
           : Sh::PAIR ? "banded stage C, paired 16-B stores, (n1, n2)-symmetric"
                      : "banded stage C, (n1, n2)-symmetric";
  return Sh::WLAST   ? "w-last contraction"
         : Sh::MMA  ? "stage C on DMMA"
         : Sh::QUAD   ? (Sh::PSPLIT ? "banded stage C, parity split, 32-B stores"
                                    : "banded stage C, 32-B stores")
         : Sh::PSPLIT ? (Sh::PAIR ? "banded stage C, parity split, paired 16-B stores"
                                  : "banded stage C, parity split")
         : Sh::PAIR   ? "banded stage C, paired 16-B stores"
                      : "banded stage C";
}

template <class Ms>
std::vector<double> pack_mv2(const std::vector<double> (*phi)[3]) {
  // phi[s][d] = [K][nq] full weighted table -> half tables [K][H]
  std::vector<double> out(static_cast<size_t>(Ms::TALL), 0.0);
  for (int s = 0; s < Ms::S; ++s)
    for (int d = 0; d < 3; ++d) {
      const int K = Ms::K(s, d), Q = Ms::Q(d), H = Ms::H(d);
      for (int k = 0; k < K; ++k)
        for (int h = 0; h < H; ++h) {
          const double v = phi[s][d][static_cast<size_t>(k) * Q + h];
          out[static_cast<size_t>(Ms::toff(s, d) + k * H + h)] = v;
          out[static_cast<size_t>(Ms::ttoff(d) + k * H + h)] = v;  // shared (identical rows)
        }
    }
  return out;
}

}  // namespace reg
}  // namespace p2s
