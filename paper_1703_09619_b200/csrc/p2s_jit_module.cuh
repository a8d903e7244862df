// p2s_jit_module.cuh -- included by the translation units p2s_jit.cu generates
// for one problem shape: instantiates the planned kernel family and exports its
// registry entries through p2s_jit_entry (loaded with dlopen by libp2s_b200).
#pragma once

#include "p2s_reg_fused.cuh"
#include "p2s_reg_large.cuh"
#include "p2s_reg_v2.cuh"

namespace p2s {
namespace reg {

template <class Sh, class Ms, bool PF>
int jit_fused(JitEntries* out) {
  *out = JitEntries{};
  out->abi = kJitAbi;
  out->family = 1;
  out->fused = make_fused<Sh, Ms, false, false, PF>();
  out->v2 = make_v2<Sh>();
  out->mv2 = make_mv2<Ms>();
  out->smem = FusedLayout<Sh, Ms, 0>::SMEM;
  out->mpp = Sh::MPP;
  return 0;
}

template <class Ls>
int jit_large(JitEntries* out) {
  *out = JitEntries{};
  out->abi = kJitAbi;
  out->family = 2;
  out->large = make_large<Ls>();
  out->smem = Ls::MOM_SMEM;
  out->mpp = Ls::MPP;
  return 0;
}

}  // namespace reg
}  // namespace p2s

#define P2S_JIT_FUSED(SH, MS, PF) \
  extern "C" int p2s_jit_entry(p2s::reg::JitEntries* out) { return p2s::reg::jit_fused<SH, MS, PF>(out); }
#define P2S_JIT_LARGE(LS) \
  extern "C" int p2s_jit_entry(p2s::reg::JitEntries* out) { return p2s::reg::jit_large<LS>(out); }
