// p2s_jit.hpp -- shape planner and generated per-shape kernel modules
// (p2s_jit.cu): every problem the ahead-of-time registries do not cover gets
// its own compile-time-banded instantiation, built once and cached.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/p2s_b200.h"
#include "p2s_registry.hpp"

namespace p2s {
namespace jit {

constexpr int kFamilyFused = 1;  // fill_fused_kernel + contract_v2 / moments_v2 of the shape
constexpr int kFamilyLarge = 2;  // large-order path (p2s_large.cuh)

struct Plan {
  int family = 0;
  std::string source;  // body of the generated translation unit
  std::string desc;    // human-readable summary (p2s_kernel_path)
  int64_t smem = 0;    // planned shared memory of the dominant kernel (bytes)
};

// Planner overrides (p2s_create_ex options P2S_JIT_*; -1 = planner's choice):
// family (1 fused, 2 large), n1 tile, Shape flags, fibers per thread, CTAs per
// SM, threads, large-path k1 chunk.
struct Overrides {
  int family = -1, T = -1, flags = -1, fpt = -1, minb = -1, threads = -1, kc = -1;
};

// Kernel family and template parameters for a problem (basis folded into the
// kinds); false with *why when no family can hold it.
bool plan(const p2s_problem& eff, Plan* pl, std::string* why, const Overrides& ov = Overrides{});

// The plan's compiled module (cached on disk, loaded once per process).
const reg::JitEntries* module(const Plan& pl, std::string* err);

bool cached(const Plan& pl);
bool compiler_available();
std::string module_path(const Plan& pl);
std::string cache_dir();

}  // namespace jit
}  // namespace p2s
