// p2s_alpha.cu -- seeded synthetic coupling factor on the device (benchmark
// harness input; not part of the timed fill).  Plays the role of
// build_element_quad (assembly.cpp:51-119) for BASELINE.json's configs:
//   SINE      alpha = 1 + 0.3 sin(a u + b v + c w + phi), a,b,c ~ U[lo,hi],
//             phi ~ U[0,2pi), independent per (element, pair, term)
//   EXPSIN    alpha = exp(0.5 sin(f (u+v+w))) (1 + 0.2 u v w), f ~ U[lo,hi]
//   JACOBIAN  trilinear map of the reference cube with corners offset by
//             U[-0.1,0.1]^3; alpha_mat (SINE form) times detJ (J^T J)^-1 for
//             even terms (mass) and (J^T J)/detJ for odd terms (curl type)
// Parameters come from a counter-based splitmix64 keyed by (seed, element,
// slot, j), identical bit for bit to the host generator; this file is
// compiled with -fmad=false so the arithmetic rounds like the host's.
#include <cuda_runtime.h>

#include <cstdint>

namespace p2s {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform(uint64_t seed, int64_t elem, int slot, int j) {
  uint64_t h = splitmix64(seed ^ 0x7032735F62323030ULL);
  h = splitmix64(h + static_cast<uint64_t>(elem));
  h = splitmix64(h + static_cast<uint64_t>(slot));
  return static_cast<double>(splitmix64(h + static_cast<uint64_t>(j)) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double lerp(double lo, double hi, double u) { return lo + (hi - lo) * u; }

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxTerms = 4;

// Geometry record of a hexahedral element (the 3-D analogue of the reference's
// element nodes + material, build_element_quad assembly.cpp:51-119): the 8
// corners X[c][d] of its trilinear map (corner c at reference (+-1,+-1,+-1),
// bit d of c = sign of coordinate d) and the material parameters (a, b, c, phi)
// of alpha_mat = 1 + 0.3 sin(a u + b v + c w + phi).
constexpr int kGeomDoubles = 28;

__device__ __forceinline__ void geometry_record(uint64_t seed, int64_t e, double lo, double hi, double* g) {
  for (int cn = 0; cn < 8; ++cn)
    for (int dd = 0; dd < 3; ++dd) {
      const double sgn = ((cn >> dd) & 1) ? 1.0 : -1.0;
      g[cn * 3 + dd] = sgn + lerp(-0.1, 0.1, uniform(seed, e, 200 + cn, dd));
    }
  g[24] = lerp(lo, hi, uniform(seed, e, 0, 0));
  g[25] = lerp(lo, hi, uniform(seed, e, 0, 1));
  g[26] = lerp(lo, hi, uniform(seed, e, 0, 2));
  g[27] = 2.0 * kPi * uniform(seed, e, 0, 3);
}

// coupling factors at reference point (u, v, w): alpha_mat detJ (J^T J)^-1 for
// even terms (mass), alpha_mat (J^T J) / detJ for odd terms (curl type), per
// component pair; written to ae[(pair * S + s) * npts + q]
__device__ __forceinline__ void jacobian_alpha(const double* g, double u, double v, double w, int nc, int S,
                                               double* ae, int64_t npts, int q) {
  const double r[3] = {u, v, w};
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int cn = 0; cn < 8; ++cn) {
    double f[3], df[3];
    for (int dd = 0; dd < 3; ++dd) {
      const double sgn = ((cn >> dd) & 1) ? 1.0 : -1.0;
      f[dd] = 0.5 * (1.0 + sgn * r[dd]);
      df[dd] = 0.5 * sgn;
    }
    const double g0 = df[0] * f[1] * f[2];
    const double g1 = f[0] * df[1] * f[2];
    const double g2 = f[0] * f[1] * df[2];
    for (int xi = 0; xi < 3; ++xi) {
      const double X = g[cn * 3 + xi];
      J[xi][0] += g0 * X;
      J[xi][1] += g1 * X;
      J[xi][2] += g2 * X;
    }
  }
  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                     J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  double G[3][3];
  for (int a1 = 0; a1 < 3; ++a1)
    for (int a2 = 0; a2 < 3; ++a2)
      G[a1][a2] = J[0][a1] * J[0][a2] + J[1][a1] * J[1][a2] + J[2][a1] * J[2][a2];
  const double dg = det * det;
  double Gi[3][3];
  Gi[0][0] = (G[1][1] * G[2][2] - G[1][2] * G[2][1]) / dg;
  Gi[0][1] = (G[0][2] * G[2][1] - G[0][1] * G[2][2]) / dg;
  Gi[0][2] = (G[0][1] * G[1][2] - G[0][2] * G[1][1]) / dg;
  Gi[1][0] = (G[1][2] * G[2][0] - G[1][0] * G[2][2]) / dg;
  Gi[1][1] = (G[0][0] * G[2][2] - G[0][2] * G[2][0]) / dg;
  Gi[1][2] = (G[0][2] * G[1][0] - G[0][0] * G[1][2]) / dg;
  Gi[2][0] = (G[1][0] * G[2][1] - G[1][1] * G[2][0]) / dg;
  Gi[2][1] = (G[0][1] * G[2][0] - G[0][0] * G[2][1]) / dg;
  Gi[2][2] = (G[0][0] * G[1][1] - G[0][1] * G[1][0]) / dg;
  const double am = 1.0 + 0.3 * sin(g[24] * r[0] + g[25] * r[1] + g[26] * r[2] + g[27]);
  for (int gi = 0; gi < nc; ++gi)
    for (int gj = 0; gj < nc; ++gj)
      for (int s = 0; s < S; ++s) {
        const double val = (s % 2 == 0) ? am * det * Gi[gi][gj] : am * G[gi][gj] / det;
        ae[(static_cast<int64_t>(gi * nc + gj) * S + s) * npts + q] = val;
      }
}

struct AlphaParams {
  double* alpha;
  const double* x[3];
  int nq[3];
  int nc, S;
  int kind;
  double lo, hi;
  uint64_t seed;
  int64_t e0, n;
  int64_t per_elem;
};

// one thread per (element, quadrature point)
__global__ void alpha_kernel(const __grid_constant__ AlphaParams p) {
  const int64_t npts = static_cast<int64_t>(p.nq[0]) * p.nq[1] * p.nq[2];
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= npts * p.n) return;
  const int64_t ie = gid / npts;
  const int q = static_cast<int>(gid - ie * npts);
  const int i = q % p.nq[0];
  const int j = (q / p.nq[0]) % p.nq[1];
  const int k = q / (p.nq[0] * p.nq[1]);
  const double u = p.x[0][i], v = p.x[1][j], w = p.x[2][k];
  const int64_t e = p.e0 + ie;
  double* ae = p.alpha + ie * p.per_elem;
  const int P = p.nc * p.nc;
  if (p.kind == 0) {  // SINE
    for (int pr = 0; pr < P; ++pr)
      for (int s = 0; s < p.S; ++s) {
        const int slot = 1 + pr * kMaxTerms + s;
        const double a = lerp(p.lo, p.hi, uniform(p.seed, e, slot, 0));
        const double b = lerp(p.lo, p.hi, uniform(p.seed, e, slot, 1));
        const double c = lerp(p.lo, p.hi, uniform(p.seed, e, slot, 2));
        const double ph = 2.0 * kPi * uniform(p.seed, e, slot, 3);
        ae[(static_cast<int64_t>(pr) * p.S + s) * npts + q] = 1.0 + 0.3 * sin(a * u + b * v + c * w + ph);
      }
  } else if (p.kind == 2) {  // EXPSIN
    const double f = lerp(p.lo, p.hi, uniform(p.seed, e, 0, 0));
    const double val = exp(0.5 * sin(f * (u + v + w))) * (1.0 + 0.2 * u * v * w);
    for (int pr = 0; pr < P; ++pr)
      for (int s = 0; s < p.S; ++s) ae[(static_cast<int64_t>(pr) * p.S + s) * npts + q] = val;
  } else {  // JACOBIAN: the element's geometry record, then the coupling at the point
    double g[kGeomDoubles];
    geometry_record(p.seed, e, p.lo, p.hi, g);
    jacobian_alpha(g, u, v, w, p.nc, p.S, ae, npts, q);
  }
}

// seeded geometry records (harness): [E][kGeomDoubles]
__global__ void geometry_kernel(double* geom, double lo, double hi, uint64_t seed, int64_t e0, int64_t n) {
  const int64_t ie = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ie >= n) return;
  double g[kGeomDoubles];
  geometry_record(seed, e0 + ie, lo, hi, g);
  for (int i = 0; i < kGeomDoubles; ++i) geom[ie * kGeomDoubles + i] = g[i];
}

}  // namespace

cudaError_t launch_alpha(double* alpha, const double* const x[3], const int nq[3], int nc, int S,
                         int kind, double lo, double hi, uint64_t seed, int64_t e0, int64_t n,
                         int64_t per_elem, cudaStream_t stream) {
  AlphaParams p;
  p.alpha = alpha;
  for (int d = 0; d < 3; ++d) {
    p.x[d] = x[d];
    p.nq[d] = nq[d];
  }
  p.nc = nc;
  p.S = S;
  p.kind = kind;
  p.lo = lo;
  p.hi = hi;
  p.seed = seed;
  p.e0 = e0;
  p.n = n;
  p.per_elem = per_elem;
  const int64_t total = static_cast<int64_t>(nq[0]) * nq[1] * nq[2] * n;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  alpha_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_geometry(double* geom, double lo, double hi, uint64_t seed, int64_t e0, int64_t n,
                            cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  geometry_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, stream>>>(geom, lo, hi, seed, e0, n);
  return cudaGetLastError();
}

}  // namespace p2s
