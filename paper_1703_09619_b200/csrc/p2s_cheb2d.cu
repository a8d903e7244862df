// p2s_cheb2d.cu -- the reference's own 2-D Chebyshev specialisation on the GPU
// (SURVEY.md 8(f) rank 1): the same two stages as the reference,
//   p2s_cheb2d_kernel_tables  ~ compute_kernel_tables (assembly.cpp:276-314):
//       Ks, Kuu, Kuv, Kvv = 2-D moments of the weighted coupling grids of
//       build_element_quad (assembly.cpp:102-106) against T / U / T^ns tables
//   p2s_cheb2d_assemble       ~ assemble_p2s_element (assembly.cpp:375-474):
//       the eight blocks S_uu .. M_vv (Eqs. (8)-(15)), every entry a
//       signed <= 4-term sum of kernel-table entries (flat_combine, :363-371)
// so the GPU can be checked against the reference's own numbers
// (tests/golden/ref2d_elements.npz).  Elements are independent: one CTA per
// (element, table) and per (element, block).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/p2s_b200.h"
#include "p2s_tables.hpp"

p2s_status p2s_internal_fail(p2s_status st, const std::string& msg);

namespace {

using namespace p2s;

constexpr int kTables = 4, kBlocks = 8;

struct TableSpec {
  int Ku, Kv;             // rows (u degrees) x cols (v degrees)
  const double* phiu;     // [Ku][nq]
  const double* phiv;     // [Kv][nq]
  int grid;               // which coupling grid (0 ws, 1 wuu, 2 wuv, 3 wvv)
  int64_t out_off;        // offset in the per-element table block
};

struct BlockSpec {
  int rows, cols;         // nt_u*nt_v x nr_u*nr_v
  int ntv, nrv;           // v-basis counts (row = mu*ntv + nv, col = mu'*nrv + nv')
  int table;              // kernel table used
  const int* su;          // CSR over (a, b) of the u expansions: [nt_u*nr_u + 1]
  const int* ku;
  const double* cu;
  const int* sv;          // CSR over (a, b) of the v expansions
  const int* kv;
  const double* cv;
  int nru;                // trial u count (CSR row length)
  int64_t out_off;
};

struct Cheb2dParams {
  TableSpec t[kTables];
  BlockSpec b[kBlocks];
  int nq;
  int64_t grids_per_elem, tables_per_elem, blocks_per_elem;
  int table_cols[kTables];
};

// T[m][n] = sum_i phiu[m][i] sum_j phiv[n][j] W[i][j]; two passes in smem
__global__ void cheb2d_tables_kernel(const __grid_constant__ Cheb2dParams p, const double* grids,
                                     double* tables) {
  extern __shared__ double sm[];
  const int64_t e = blockIdx.x / kTables;
  const int ti = blockIdx.x % kTables;
  const TableSpec& t = p.t[ti];
  const int nq = p.nq;
  const double* W = grids + e * p.grids_per_elem + static_cast<int64_t>(t.grid) * nq * nq;
  double* R = sm;  // [Ku][nq]: R[m][j] = sum_i phiu[m][i] W[i][j]
  for (int idx = threadIdx.x; idx < t.Ku * nq; idx += blockDim.x) {
    const int m = idx / nq, j = idx - (idx / nq) * nq;
    double s = 0.0;
    for (int i = 0; i < nq; ++i) s = fma(t.phiu[m * nq + i], W[i * nq + j], s);
    R[idx] = s;
  }
  __syncthreads();
  double* out = tables + e * p.tables_per_elem + t.out_off;
  for (int idx = threadIdx.x; idx < t.Ku * t.Kv; idx += blockDim.x) {
    const int m = idx / t.Kv, n = idx - (idx / t.Kv) * t.Kv;
    double s = 0.0;
    for (int j = 0; j < nq; ++j) s = fma(R[m * nq + j], t.phiv[n * nq + j], s);
    out[idx] = s;
  }
}

// one thread per block entry: sum over the u- and v-expansion terms
__global__ void cheb2d_assemble_kernel(const __grid_constant__ Cheb2dParams p, const double* tables,
                                       double* blocks) {
  const int64_t e = blockIdx.x / kBlocks;
  const int bi = blockIdx.x % kBlocks;
  const BlockSpec& b = p.b[bi];
  const double* T = tables + e * p.tables_per_elem + p.t[b.table].out_off;
  const int tcols = p.table_cols[b.table];
  double* out = blocks + e * p.blocks_per_elem + b.out_off;
  for (int idx = threadIdx.x; idx < b.rows * b.cols; idx += blockDim.x) {
    const int row = idx / b.cols, col = idx - (idx / b.cols) * b.cols;
    const int m1 = row / b.ntv, n1 = row - m1 * b.ntv;
    const int m2 = col / b.nrv, n2 = col - m2 * b.nrv;
    const int au = m1 * b.nru + m2, av = n1 * b.nrv + n2;
    double s = 0.0;
    for (int iu = b.su[au]; iu < b.su[au + 1]; ++iu) {
      const double* trow = T + b.ku[iu] * tcols;
      double r = 0.0;
      for (int iv = b.sv[av]; iv < b.sv[av + 1]; ++iv) r = fma(b.cv[iv], trow[b.kv[iv]], r);
      s = fma(b.cu[iu], r, s);
    }
    out[idx] = s;
  }
}

// 1-D basis of a block direction: index a -> (family, degree, prefactor)
enum Basis { B_U, B_T, B_DU, B_NDU, B_NT };
bool basis(int kind, int a, int& fam, int& deg, double& pref) {
  switch (kind) {
    case B_U: fam = CHEB_U; deg = a; pref = 1.0; return true;
    case B_T: fam = CHEB_T; deg = a; pref = 1.0; return true;
    case B_NT: fam = CHEB_T; deg = a; pref = -1.0; return true;
    case B_DU: if (a < 1) return false; fam = CHEB_U; deg = a - 1; pref = a; return true;
    default: if (a < 1) return false; fam = CHEB_U; deg = a - 1; pref = -a; return true;
  }
}

struct Csr {
  std::vector<int> start, k;
  std::vector<double> c;
};

// expansions of test(a) x trial(b) in family kfam (<= 2 terms each, prefactors folded)
bool build_csr(int bt, int nt, int br, int nr, int kfam, int K, Csr& out, std::string& err) {
  out.start.assign(static_cast<size_t>(nt * nr + 1), 0);
  for (int a = 0; a < nt; ++a)
    for (int b = 0; b < nr; ++b) {
      out.start[static_cast<size_t>(a * nr + b)] = static_cast<int>(out.k.size());
      int fa, da, fb, db;
      double pa, pb;
      if (!basis(bt, a, fa, da, pa) || !basis(br, b, fb, db, pb)) continue;
      ChebTerm t[2];
      const int n = cheb_product(fa, da, fb, db, t);
      for (int i = 0; i < n; ++i) {
        if (t[i].fam != kfam || t[i].deg >= K) {
          err = "kernel table family mismatch";  // assembly.cpp:344
          return false;
        }
        out.k.push_back(t[i].deg);
        out.c.push_back(pa * pb * t[i].coeff);
      }
    }
  out.start[static_cast<size_t>(nt * nr)] = static_cast<int>(out.k.size());
  return true;
}

// The reference's conforming change of basis on one side of a CSR (apply_conforming_
// transform, assembly.cpp:491-574; R = conforming_matrix, :476-489): entry (a', b')
// becomes sum_{a, b} R[a][a'] R[b][b'] entry(a, b) over the <= 2 x 2 supports, with
// the expansion terms merged by kernel index.  ta / tb: transform the test / trial side.
Csr conform_csr(const Csr& in, int nt, int nr, bool ta, bool tb) {
  Csr out;
  out.start.assign(static_cast<size_t>(nt * nr + 1), 0);
  auto sup = [](bool on, int m, int i, int& idx, double& r) {
    if (!on) {
      idx = m;
      r = 1.0;
      return i == 0;
    }
    idx = conf_sup(m, i);
    r = conf_r(m, i);
    return true;
  };
  for (int a2 = 0; a2 < nt; ++a2)
    for (int b2 = 0; b2 < nr; ++b2) {
      out.start[static_cast<size_t>(a2 * nr + b2)] = static_cast<int>(out.k.size());
      std::vector<std::pair<int, double>> acc;
      for (int i = 0; i < 2; ++i) {
        int a;
        double ra;
        if (!sup(ta, a2, i, a, ra)) continue;
        for (int j = 0; j < 2; ++j) {
          int b;
          double rb;
          if (!sup(tb, b2, j, b, rb)) continue;
          const size_t ab = static_cast<size_t>(a * nr + b);
          for (int t = in.start[ab]; t < in.start[ab + 1]; ++t) {
            const double v = ra * rb * in.c[static_cast<size_t>(t)];
            bool found = false;
            for (auto& kv : acc)
              if (kv.first == in.k[static_cast<size_t>(t)]) {
                kv.second += v;
                found = true;
              }
            if (!found) acc.emplace_back(in.k[static_cast<size_t>(t)], v);
          }
        }
      }
      for (const auto& kv : acc)
        if (kv.second != 0.0) {
          out.k.push_back(kv.first);
          out.c.push_back(kv.second);
        }
    }
  out.start[static_cast<size_t>(nt * nr)] = static_cast<int>(out.k.size());
  return out;
}

}  // namespace

struct p2s_cheb2d_ctx {
  p2s_cheb2d_problem pb{};
  int device = 0;
  p2s_cheb2d_sizes sz{};
  Cheb2dParams params{};
  std::vector<void*> allocs;
  size_t tables_smem = 0;
};

namespace {

template <class T>
bool upload(p2s_cheb2d_ctx* c, const std::vector<T>& v, const T** out) {
  void* d = nullptr;
  const size_t bytes = sizeof(T) * (v.empty() ? 1 : v.size());
  if (cudaMalloc(&d, bytes) != cudaSuccess) return false;
  c->allocs.push_back(d);
  if (!v.empty() && cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return false;
  *out = static_cast<const T*>(d);
  return true;
}

}  // namespace

bool p2s_cheb2d_block_layout(const p2s_cheb2d_ctx* c, int64_t off[8], int rows[8], int cols[8],
                             int* n_eu, int* n_ev) {
  if (!c) return false;
  for (int q = 0; q < 8; ++q) {
    off[q] = c->sz.block_offset[q];
    rows[q] = c->sz.block_rows[q];
    cols[q] = c->sz.block_cols[q];
  }
  *n_eu = c->sz.n_eu;
  *n_ev = c->sz.n_ev;
  return true;
}

extern "C" {

p2s_status p2s_cheb2d_create(const p2s_cheb2d_problem* spec, int device, p2s_cheb2d_ctx** out) {
  if (!spec || !out) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_create: null argument");
  *out = nullptr;
  const int M = spec->M, N = spec->N, nq = spec->nq;
  if (M < 1 || N < 1 || M > 64 || N > 64) return p2s_internal_fail(P2S_INVALID_ARG, "orders must be 1..64");
  if (nq < 1 || nq > 128) return p2s_internal_fail(P2S_INVALID_ARG, "nq must be 1..128");
  if (spec->conforming != 0 && spec->conforming != 1)
    return p2s_internal_fail(P2S_INVALID_ARG, "conforming must be 0 or 1");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return p2s_internal_fail(P2S_CUDA_ERROR, "p2s_cheb2d_create: no CUDA device (no CPU fallback)");
  if (device < 0 || device >= ndev) return p2s_internal_fail(P2S_INVALID_ARG, "bad device");
  if (cudaSetDevice(device) != cudaSuccess) return p2s_internal_fail(P2S_CUDA_ERROR, "cudaSetDevice");
  // early returns below free the device tables uploaded so far
  std::unique_ptr<p2s_cheb2d_ctx, void (*)(p2s_cheb2d_ctx*)> c(new p2s_cheb2d_ctx, &p2s_cheb2d_destroy);
  c->pb = *spec;
  c->device = device;
  std::vector<double> x, w;
  gauss_legendre_ld(nq, x, w);
  // kernel tables: Ks (Tns, Tns) ws, Kuu (Tns, T) wuu, Kuv (U, U) wuv, Kvv (T, Tns) wvv
  const int fu[kTables] = {CHEB_TNS, CHEB_TNS, CHEB_U, CHEB_T};
  const int fv[kTables] = {CHEB_TNS, CHEB_T, CHEB_U, CHEB_TNS};
  int64_t off = 0;
  size_t smem = 0;
  for (int t = 0; t < kTables; ++t) {
    const int Ku = fu[t] == CHEB_U ? 2 * M : 2 * M + 1;
    const int Kv = fv[t] == CHEB_U ? 2 * N : 2 * N + 1;
    std::vector<double> pu(static_cast<size_t>(Ku) * nq), pv(static_cast<size_t>(Kv) * nq);
    for (int k = 0; k < Ku; ++k)
      for (int q = 0; q < nq; ++q) pu[static_cast<size_t>(k) * nq + q] = static_cast<double>(cheb_eval(fu[t], k, x[q]));
    for (int k = 0; k < Kv; ++k)
      for (int q = 0; q < nq; ++q) pv[static_cast<size_t>(k) * nq + q] = static_cast<double>(cheb_eval(fv[t], k, x[q]));
    TableSpec& ts = c->params.t[t];
    ts.Ku = Ku;
    ts.Kv = Kv;
    ts.grid = t;
    ts.out_off = off;
    if (!upload(c.get(), pu, &ts.phiu) || !upload(c.get(), pv, &ts.phiv))
      return p2s_internal_fail(P2S_CUDA_ERROR, "p2s_cheb2d_create: upload");
    c->params.table_cols[t] = Kv;
    c->sz.table_offset[t] = off;
    c->sz.table_rows[t] = Ku;
    c->sz.table_cols[t] = Kv;
    off += static_cast<int64_t>(Ku) * Kv;
    smem = std::max(smem, sizeof(double) * static_cast<size_t>(Ku) * nq);
  }
  c->sz.tables_per_elem = off;
  c->tables_smem = smem;
  // blocks (Eqs. (8)-(15); assembly.cpp:162-269): {u test, u trial, v test, v trial, table}
  struct { int ut, ur, vt, vr, table; } spec8[kBlocks] = {
      {B_U, B_U, B_DU, B_DU, 0},   {B_U, B_NDU, B_DU, B_U, 0}, {B_NDU, B_U, B_U, B_DU, 0},
      {B_DU, B_DU, B_U, B_U, 0},   {B_U, B_U, B_T, B_T, 1},    {B_U, B_NT, B_T, B_U, 2},
      {B_NT, B_U, B_U, B_T, 2},    {B_T, B_T, B_U, B_U, 3}};
  off = 0;
  const int neu = M * (N + 1), nev = (M + 1) * N;
  c->sz.n_eu = neu;
  c->sz.n_ev = nev;
  for (int bi = 0; bi < kBlocks; ++bi) {
    const int q = bi % 4;
    const int ti = (q == 0 || q == 1) ? 0 : 1, tj = (q == 0 || q == 2) ? 0 : 1;
    const int ntu = ti == 0 ? M : M + 1, ntv = ti == 0 ? N + 1 : N;
    const int nru = tj == 0 ? M : M + 1, nrv = tj == 0 ? N + 1 : N;
    const int tab = spec8[bi].table;
    Csr cu, cv;
    std::string err;
    if (!build_csr(spec8[bi].ut, ntu, spec8[bi].ur, nru, fu[tab], c->params.t[tab].Ku, cu, err) ||
        !build_csr(spec8[bi].vt, ntv, spec8[bi].vr, nrv, fv[tab], c->params.t[tab].Kv, cv, err))
      return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_create: " + err);
    if (spec->conforming) {
      // E_u = m (N+1) + n: the v index n is transformed; E_v = m N + n: the u index m
      cv = conform_csr(cv, ntv, nrv, ti == 0, tj == 0);
      cu = conform_csr(cu, ntu, nru, ti == 1, tj == 1);
    }
    BlockSpec& b = c->params.b[bi];
    b.rows = ntu * ntv;
    b.cols = nru * nrv;
    b.ntv = ntv;
    b.nrv = nrv;
    b.nru = nru;
    b.table = tab;
    b.out_off = off;
    if (!upload(c.get(), cu.start, &b.su) || !upload(c.get(), cu.k, &b.ku) ||
        !upload(c.get(), cu.c, &b.cu) || !upload(c.get(), cv.start, &b.sv) ||
        !upload(c.get(), cv.k, &b.kv) || !upload(c.get(), cv.c, &b.cv))
      return p2s_internal_fail(P2S_CUDA_ERROR, "p2s_cheb2d_create: upload");
    c->sz.block_offset[bi] = off;
    c->sz.block_rows[bi] = b.rows;
    c->sz.block_cols[bi] = b.cols;
    off += static_cast<int64_t>(b.rows) * b.cols;
  }
  c->sz.blocks_per_elem = off;
  c->sz.grids_per_elem = static_cast<int64_t>(kTables) * nq * nq;
  c->params.nq = nq;
  c->params.grids_per_elem = c->sz.grids_per_elem;
  c->params.tables_per_elem = c->sz.tables_per_elem;
  c->params.blocks_per_elem = c->sz.blocks_per_elem;
  *out = c.release();
  return P2S_OK;
}

void p2s_cheb2d_destroy(p2s_cheb2d_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (void* p : c->allocs) cudaFree(p);
  delete c;
}

p2s_status p2s_cheb2d_get_sizes(const p2s_cheb2d_ctx* c, p2s_cheb2d_sizes* out) {
  if (!c || !out) return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_get_sizes: null argument");
  *out = c->sz;
  return P2S_OK;
}

p2s_status p2s_cheb2d_kernel_tables(p2s_cheb2d_ctx* c, const double* d_grids, double* d_tables,
                                    int64_t n, void* stream) {
  if (!c) return p2s_internal_fail(P2S_INVALID_ARG, "null context");
  if (n < 0 || (n > 0 && (!d_grids || !d_tables)))
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_kernel_tables: bad buffers");
  if (n == 0) return P2S_OK;
  cudaSetDevice(c->device);
  cheb2d_tables_kernel<<<static_cast<unsigned>(n * kTables), 256, c->tables_smem,
                         static_cast<cudaStream_t>(stream)>>>(c->params, d_grids, d_tables);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return p2s_internal_fail(P2S_CUDA_ERROR, std::string("cheb2d_tables_kernel: ") + cudaGetErrorString(e));
  return P2S_OK;
}

p2s_status p2s_cheb2d_assemble(p2s_cheb2d_ctx* c, const double* d_tables, double* d_blocks, int64_t n,
                               void* stream) {
  if (!c) return p2s_internal_fail(P2S_INVALID_ARG, "null context");
  if (n < 0 || (n > 0 && (!d_tables || !d_blocks)))
    return p2s_internal_fail(P2S_INVALID_ARG, "p2s_cheb2d_assemble: bad buffers");
  if (n == 0) return P2S_OK;
  cudaSetDevice(c->device);
  cheb2d_assemble_kernel<<<static_cast<unsigned>(n * kBlocks), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(c->params, d_tables, d_blocks);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return p2s_internal_fail(P2S_CUDA_ERROR, std::string("cheb2d_assemble_kernel: ") + cudaGetErrorString(e));
  return P2S_OK;
}

}  // extern "C"
