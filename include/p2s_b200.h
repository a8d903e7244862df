/*
 * p2s_b200.h -- C-ABI of the B200-native product-to-sum element fill.
 *
 * Drop-in boundary for the reference's fill path (/root/reference/proj):
 *
 *   reference (C++, include/chebfem/assembly.hpp)        this ABI
 *   ---------------------------------------------------  ------------------------
 *   poly_table / FlatTable / product_to_sum tables,       p2s_create
 *     rebuilt per element (assembly.cpp:41-49,110-117,
 *     332-352; chebyshev.cpp:156-178)
 *   compute_kernel_tables(mesh, e, orders, nq)            p2s_moments
 *     (assembly.hpp:52; assembly.cpp:276-314)
 *   assemble_p2s_element(kernels, orders)                 p2s_contract
 *     (assembly.hpp:56; assembly.cpp:375-474)
 *   fill_elements(mesh, orders, Backend::p2s, nq, thr)    p2s_fill (device buffers)
 *     (assembly.hpp:82-83; assembly.cpp:654-700)          p2s_fill_host (host buffers)
 *   C++ exceptions (std::invalid_argument,                p2s_status + p2s_last_error
 *     GeometryError, std::logic_error)                      (include/p2s_b200.hpp maps
 *                                                           them back to exceptions)
 *
 * Problem: the paper's general 3-D scheme (Eqs. (1)-(4)) with
 * Legendre kernel polynomials.  n_comp field components share the orders
 * N_u, N_v, N_w (basis P_0..P_{N-1} per direction); every ordered component
 * pair (gi, gj) carries n_terms coupling factors alpha_s^{gi gj}; term s uses,
 * per direction, the operator pair kind (P2S_PP: P_m1 P_m2, P2S_DD: P'_m1
 * P'_m2, P2S_DP: P'_m1 P_m2, P2S_PD: P_m1 P'_m2).
 *
 * Layouts (FP64, all row-major, u fastest in alpha, p fastest in M):
 *   alpha  [E][P][S][nq_w][nq_v][nq_u]          P = n_comp^2, pair = gi*n_comp+gj
 *          values of alpha_s at the Gauss-Legendre nodes; the quadrature
 *          weights are NOT included (they live in the kernel tables).
 *   I      [E][P] blocks of sizes.moments_per_pair doubles; term s of a pair
 *          starts at sizes.moment_offset[s] and holds [K_u][K_v][K_w].
 *   M      E matrices of n_tot x n_tot with leading dimension ld_M (>= n_tot),
 *          matrix e at M + e * n_tot * ld_M;
 *          row = gi*Nu*Nv*Nw + (m1*Nv + n1)*Nw + p1 (test),
 *          col = gj*Nu*Nv*Nw + (m2*Nv + n2)*Nw + p2 (trial).
 *
 * Ownership: the caller owns alpha / I / M buffers; the context owns the
 * uploaded tables and its scratch and is immutable after p2s_create (the
 * profiling switch aside).  One context per device; any entry point may be
 * called from several host threads and streams: calls that use context scratch
 * (p2s_fill on the two-stage and large-order paths, p2s_contract on the
 * large-order path, p2s_fill_host, the geometry entry points) are ordered on the
 * device behind each other through a context event, the others run concurrently.
 * Alignment: alpha 32-byte aligned when nq_u % 4 == 0 (32-B row loads), else
 * 16-byte; I 16-byte; M 8-byte (wider stores are used where rows allow).
 *
 * There is no CPU fallback: every compute entry point runs sm_100a kernels
 * and fails with P2S_CUDA_ERROR when no B200 is present.
 */
#ifndef P2S_B200_H
#define P2S_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2S_MAX_TERMS 4

typedef enum {
  P2S_OK = 0,
  P2S_INVALID_ARG = 1,        /* std::invalid_argument in the reference      */
  P2S_CUDA_ERROR = 2,         /* device / driver failure                      */
  P2S_UNSUPPORTED_SHAPE = 3,  /* no kernel instantiation for these orders    */
  P2S_GEOMETRY_ERROR = 4      /* GeometryError (J <= 0) in the reference      */
} p2s_status;

enum { P2S_PP = 0, P2S_DD = 1, P2S_DP = 2, P2S_PD = 3 };

/* synthetic coupling-factor families of BASELINE.json's configs */
enum { P2S_ALPHA_SINE = 0, P2S_ALPHA_JACOBIAN = 1, P2S_ALPHA_EXPSIN = 2 };

typedef struct {
  int32_t n_comp;                        /* 1 or 3                              */
  int32_t order[3];                      /* N_u, N_v, N_w (>= 1)                */
  int32_t n_terms;                       /* N_s (1 .. P2S_MAX_TERMS)            */
  int32_t kind[P2S_MAX_TERMS][3];        /* P2S_PP / DD / DP / PD               */
  int32_t nq[3];                         /* Gauss-Legendre points per direction */
  int32_t basis;                         /* P2S_BASIS_MODAL / P2S_BASIS_CONFORMING */
} p2s_problem;

/* Basis of the element matrices (both sides, every direction):
 *   MODAL       P_0 .. P_{N-1}
 *   CONFORMING  phi_0 = (P_0 - P_1)/2, phi_1 = (P_0 + P_1)/2, phi_n = P_n - P_{n mod 2}:
 *               the reference's conforming change of basis (conforming_matrix /
 *               apply_conforming_transform, assembly.cpp:476-574), folded into the
 *               product-to-sum tables -- M_conf = T^T M_modal T at no extra cost. */
enum { P2S_BASIS_MODAL = 0, P2S_BASIS_CONFORMING = 1 };

typedef struct {
  int64_t alpha_per_elem;                /* doubles                              */
  int64_t moments_per_elem;              /* doubles (= n_pairs * per_pair)       */
  int64_t moments_per_pair;              /* doubles, padded to a multiple of 4   */
  int64_t moment_offset[P2S_MAX_TERMS];  /* doubles, within a pair block         */
  int32_t n_tot;                         /* matrix dimension                     */
  int32_t n_pairs;                       /* n_comp^2                             */
  int32_t K[P2S_MAX_TERMS][3];           /* kernel polynomial counts             */
} p2s_sizes;

typedef struct p2s_ctx p2s_ctx;

/* Builds and uploads the Gauss-Legendre rules, weighted Legendre kernel tables
 * and product-to-sum coefficient tables once.  Every valid problem is accepted
 * (the reference's fill takes any Orders, kinds and nq: assembly.hpp:52-56,
 * 82-83): shapes without an ahead-of-time kernel get a generated module --
 * the planned kernel family instantiated for exactly this shape, compiled once
 * for sm_100a with nvcc into the module cache (<dir of libp2s_b200.so>/jit, or
 * $P2S_JIT_CACHE; compiler $P2S_NVCC, else $CUDA_HOME/bin/nvcc, else nvcc) and
 * reused by later contexts and processes.  P2S_UNSUPPORTED_SHAPE: no family
 * holds the shape, or its module is neither cached nor compilable here. */
p2s_status p2s_create(const p2s_problem* spec, int device, p2s_ctx** out);

/* p2s_create with test / tuning hooks: options = "KEY=VALUE" pairs separated by
 * ';' (NULL or "" = p2s_create).  Keys (unknown keys -> P2S_INVALID_ARG):
 * P2S_NO_FUSED, P2S_FORCE_GENERIC, P2S_JIT (0: no generated module),
 * P2S_FORCE_JIT, P2S_FUSED_VARIANT / P2S_V2_VARIANT / P2S_MV2_VARIANT (k-th
 * registered variant), P2S_CHUNK_MB, P2S_TWO_STAGE_OVERLAP, P2S_MOM_PRIO,
 * P2S_HOST_CHUNK_MB, P2S_GEO_MODE, P2S_GEO_CHUNK_MB, P2S_XCHUNK_MB and the
 * large-path switches P2S_LARGE_* (see p2s_capi.cu).  The library never reads
 * these from the environment. */
p2s_status p2s_create_ex(const p2s_problem* spec, int device, const char* options, p2s_ctx** out);

/* Plans the problem and builds (or finds) its generated module without touching
 * a device -- ahead-of-time warm-up of the module cache (build scripts, CI);
 * options as for p2s_create_ex (planner overrides P2S_JIT_*).  desc (may be
 * NULL) receives the plan and the module path. */
p2s_status p2s_shape_prepare(const p2s_problem* spec, const char* options, char* desc, int desc_len);

/* Directory of this library's generated modules (root/<kernel-header hash>). */
const char* p2s_jit_cache_dir(void);
void p2s_destroy(p2s_ctx* ctx);

p2s_status p2s_get_sizes(const p2s_ctx* ctx, p2s_sizes* out);
/* The same sizes from the problem alone (no context, no device). */
p2s_status p2s_problem_sizes(const p2s_problem* spec, p2s_sizes* out);

/* Moment stage:  I_s[k1][k2][k3] = sum_q w_q alpha_s(q) P_k1(u) P_k2(v) P_k3(w). */
p2s_status p2s_moments(p2s_ctx* ctx, const double* d_alpha, double* d_I, int64_t n_elem,
                       void* stream);

/* Contraction stage:  M = sum_s sum_k C_u C_v C_w I_s, every entry written once. */
p2s_status p2s_contract(p2s_ctx* ctx, const double* d_I, double* d_M, int64_t ld_M,
                        int64_t n_elem, void* stream);

/* Both stages over a batch, moments staged in context scratch (chunked so the
 * scratch stays L2-resident).  Large-order shapes (hundreds of short kernels per
 * fill): a call that repeats the (d_alpha, d_M, ld_M, n_elem) of an earlier call
 * is captured into a CUDA graph and replayed from then on -- same kernels, same
 * results, one cudaGraphLaunch on `stream` (option P2S_GRAPH=0: never; a stream
 * that is itself being captured launches directly). */
p2s_status p2s_fill(p2s_ctx* ctx, const double* d_alpha, double* d_M, int64_t ld_M,
                    int64_t n_elem, void* stream);

/* Host buffers in and out; H2D, fill and D2H pipelined over chunks on the
 * context's streams.  Returns after the last matrix is in h_M. */
p2s_status p2s_fill_host(p2s_ctx* ctx, const double* h_alpha, double* h_M, int64_t ld_M,
                         int64_t n_elem);

/* Host-buffer variants of the two stages (the reference's value-semantics
 * compute_kernel_tables / assemble_p2s_element on host memory): device
 * staging is internal; synchronous. */
p2s_status p2s_moments_host(p2s_ctx* ctx, const double* h_alpha, double* h_I, int64_t n_elem);
p2s_status p2s_contract_host(p2s_ctx* ctx, const double* h_I, double* h_M, int64_t ld_M,
                             int64_t n_elem);

/* Seeded synthetic coupling factor (benchmark harness input, not part of the
 * fill): elements e0 .. e0+n_elem-1 into d_alpha.  lo/hi: frequency range. */
p2s_status p2s_alpha_generate(p2s_ctx* ctx, int alpha_kind, double lo, double hi,
                              uint64_t seed, int64_t e0, int64_t n_elem, double* d_alpha,
                              void* stream);

/* ---- Element geometry instead of sampled alpha ----
 * A geometry record of P2S_GEOM_DOUBLES doubles per element: the 8 corners of the
 * hexahedron's trilinear map X[c][d] (corner c at reference (+-1, +-1, +-1), bit d
 * of c = sign along d) and the material (a, b, c, phi) of
 * alpha_mat = 1 + 0.3 sin(a u + b v + c w + phi).  The coupling factors are the
 * P2S_ALPHA_JACOBIAN family: alpha_mat detJ (J^T J)^-1 (even terms) and
 * alpha_mat (J^T J)/detJ (odd terms), per component pair -- the 3-D analogue of
 * build_element_quad (assembly.cpp:51-119).
 *   p2s_geometry_generate    seeded records (harness; p2s_alpha_generate(JACOBIAN)
 *                            is alpha_from_geometry of these records, bit for bit)
 *   p2s_alpha_from_geometry  alpha [E][P][S][nq_w][nq_v][nq_u] from records
 *   p2s_fill_geometry        the fill straight from records: alpha of a chunk of
 *                            elements is produced into an L2-resident double buffer
 *                            on an internal stream while the fill consumes the
 *                            other, so alpha never round-trips through HBM; equal
 *                            bit for bit to p2s_fill(p2s_alpha_from_geometry(...)).
 *                            Not re-entrant on one context (internal buffers).
 * Both geometry entry points wait for their stream and return P2S_GEOMETRY_ERROR
 * when the Jacobian determinant is <= 0 at any quadrature point of any element
 * (the reference's GeometryError, assembly.cpp:95-99); the outputs of such a call
 * are unspecified. */
#define P2S_GEOM_DOUBLES 28
p2s_status p2s_geometry_generate(p2s_ctx* ctx, double lo, double hi, uint64_t seed, int64_t e0,
                                 int64_t n_elem, double* d_geom, void* stream);
p2s_status p2s_alpha_from_geometry(p2s_ctx* ctx, const double* d_geom, int64_t n_elem, double* d_alpha,
                                   void* stream);
p2s_status p2s_fill_geometry(p2s_ctx* ctx, const double* d_geom, double* d_M, int64_t ld_M, int64_t n_elem,
                             void* stream);

/* Host copies of the uploaded tables: phi = w_q P_k(x_q) as [K][nq],
 * coef = [N][N][K]; nodes/weights [nq].  Any pointer may be NULL. */
p2s_status p2s_get_tables(const p2s_ctx* ctx, int term, int dir, double* phi, double* coef,
                          double* nodes, double* weights);

/* Stage timing on the launching stream (CUDA events around every launch);
 * accumulated until the next p2s_set_profiling call. */
p2s_status p2s_set_profiling(p2s_ctx* ctx, int enable);
p2s_status p2s_get_stage_times(p2s_ctx* ctx, double* ms_moments, double* ms_contract,
                               int64_t* n_moment_launches, int64_t* n_contract_launches);

/* ---- Direct-quadrature fill (the ablation baseline the paper's scheme replaces) ----
 * reference: assemble_direct_element (assembly.hpp:50; assembly.cpp:134-274) and
 * fill_elements(.., Backend::direct, ..) (assembly.hpp:12-15, 82-83).  Same problem
 * description, alpha and M layouts as p2s_fill; every entry is the full tensor
 * Gauss-Legendre sum (per element, pair and term one dense FP64 GEMM on the tensor
 * cores via cuBLAS).  The context holds the tensor basis tables (2 x n_terms x
 * nq_u nq_v nq_w x N_u N_v N_w doubles) and ~1 GiB of scratch; p2s_direct_fill
 * calls on one context must not overlap. */
typedef struct p2s_direct_ctx p2s_direct_ctx;
p2s_status p2s_direct_create(const p2s_problem* spec, int device, p2s_direct_ctx** out);
void p2s_direct_destroy(p2s_direct_ctx* ctx);
p2s_status p2s_direct_fill(p2s_direct_ctx* ctx, const double* d_alpha, double* d_M, int64_t ld_M,
                           int64_t n_elem, void* stream);

/* ---- Global scatter-add (the step after the fill: reference assemble_global,
 * assembly.cpp:594-652) ----
 * G[gi][gj] += s_i s_j E_e[i][j] over elements e and local DOFs i, j whose free
 * index dof_free[e][i] is >= 0 (-1 = PEC-constrained, dropped); dof_sign = +-1.
 * Element e's matrix: d_elem + e*elem_stride, row-major with leading dimension
 * ld_elem (the p2s_fill output: elem_stride = n_tot*ld_M).  The caller zeroes G
 * (n_free x n_free, leading dimension ld_G).  FP64 atomics: shared entries add up
 * in unspecified order (equal to the reference's serial sum up to rounding).
 * n_local <= 4096. */
p2s_status p2s_scatter_add(const double* d_elem, int64_t elem_stride, int64_t ld_elem, int32_t n_local,
                           const int32_t* d_dof_free, const double* d_dof_sign, int64_t n_elem,
                           double* d_G, int64_t ld_G, void* stream);

/* Deterministic scatter: the reference's summation order (elements ascending,
 * then local row; assembly.cpp:626-641) and arithmetic (G += (s_i s_j) E, no
 * FMA contraction), so G equals the reference's serial sum bit for bit.  The plan
 * (per global row, its (element, local row) contributions in that order) is
 * built once per mesh from the HOST copy of the free-index map
 * h_dof_free[n_elem][n_local]; the device copy passed to the scatter calls must
 * hold the same values.  One CTA per global row, no atomics.  Requires that no
 * element lists one free index twice. */
typedef struct p2s_scatter_plan p2s_scatter_plan;
p2s_status p2s_scatter_plan_create(const int32_t* h_dof_free, int64_t n_elem, int32_t n_local, int32_t n_free,
                                   int device, p2s_scatter_plan** out);
void p2s_scatter_plan_destroy(p2s_scatter_plan* plan);
p2s_status p2s_scatter_add_ordered(const p2s_scatter_plan* plan, const double* d_elem, int64_t elem_stride,
                                   int64_t ld_elem, const int32_t* d_dof_free, const double* d_dof_sign,
                                   double* d_G, int64_t ld_G, void* stream);

/* 1 if p2s_create accepts the problem here: an ahead-of-time kernel, or a
 * generated module that is cached or can be compiled (nvcc present). */
int p2s_shape_supported(const p2s_problem* spec);

/* Thread-local description of the last failure on this thread. */
const char* p2s_last_error(void);

const char* p2s_version(void);

/* Which kernels p2s_fill runs for this context (shape-specialised fused
 * kernel, two-stage specialised, or the runtime-shaped generic kernels). */
const char* p2s_kernel_path(const p2s_ctx* ctx);

/* ------------------------------------------------------------------------
 * 2-D Chebyshev mode: the reference's own specialisation (Sec. III;
 * chebfem, 2-component curl-curl element with E_u = U_m(u) T_n(v), m < M,
 * n <= N and E_v = T_m(u) U_n(v)), on the GPU, for drop-in parity with
 * chebfem::compute_kernel_tables / assemble_p2s_element (assembly.hpp:52-56).
 *   grids   [E][4][nq][nq]  ws, wuu, wuv, wvv of build_element_quad
 *                           (assembly.cpp:102-106), [i_u][j_v], weights folded
 *   tables  [E][...]        Ks, Kuu, Kuv, Kvv, row-major [u degree][v degree]
 *   blocks  [E][...]        Suu, Suv, Svu, Svv, Muu, Muv, Mvu, Mvv, row-major
 *                           (E_u index m*(N+1)+n, E_v index m*N+n)
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t M, N;        /* orders (chebfem::Orders) */
  int32_t nq;          /* Gauss-Legendre points per direction */
  int32_t conforming;  /* 1: blocks after apply_conforming_transform (assembly.cpp:555-574),
                          folded into the expansion lists (no extra pass) */
} p2s_cheb2d_problem;

typedef struct {
  int64_t grids_per_elem, tables_per_elem, blocks_per_elem;
  int64_t table_offset[4];
  int64_t block_offset[8];
  int32_t table_rows[4], table_cols[4];
  int32_t block_rows[8], block_cols[8];
  int32_t n_eu, n_ev;
} p2s_cheb2d_sizes;

typedef struct p2s_cheb2d_ctx p2s_cheb2d_ctx;

p2s_status p2s_cheb2d_create(const p2s_cheb2d_problem* spec, int device, p2s_cheb2d_ctx** out);
void p2s_cheb2d_destroy(p2s_cheb2d_ctx* ctx);
p2s_status p2s_cheb2d_get_sizes(const p2s_cheb2d_ctx* ctx, p2s_cheb2d_sizes* out);
/* compute_kernel_tables (assembly.cpp:276-314) for n_elem elements */
p2s_status p2s_cheb2d_kernel_tables(p2s_cheb2d_ctx* ctx, const double* d_grids, double* d_tables,
                                    int64_t n_elem, void* stream);
/* assemble_p2s_element (assembly.cpp:375-474) for n_elem elements */
/* assemble_global (assembly.cpp:594-652) from the eight blocks in place: local DOF
 * i < n_eu is E_u row i, else E_v row i - n_eu; S from Suu..Svv, M from Muu..Mvv
 * (build the blocks with conforming = 1 for the reference's assemble_system);
 * dof_free / dof_sign [E][n_eu + n_ev] from the reference's DofMap (free_index of
 * element_dofs[e][i].global, and .sign).  The caller zeroes S and M. */
p2s_status p2s_cheb2d_scatter(const p2s_cheb2d_ctx* ctx, const double* d_blocks, const int32_t* d_dof_free,
                              const double* d_dof_sign, int64_t n_elem, double* d_S, double* d_M,
                              int64_t ld_G, void* stream);
p2s_status p2s_cheb2d_assemble(p2s_cheb2d_ctx* ctx, const double* d_tables, double* d_blocks,
                               int64_t n_elem, void* stream);
/* p2s_cheb2d_scatter in the reference's summation order, bit for bit (plan from
 * p2s_scatter_plan_create with n_local = n_eu + n_ev). */
p2s_status p2s_cheb2d_scatter_ordered(const p2s_cheb2d_ctx* ctx, const p2s_scatter_plan* plan,
                                      const double* d_blocks, const int32_t* d_dof_free, const double* d_dof_sign,
                                      double* d_S, double* d_M, int64_t ld_G, void* stream);

#ifdef __cplusplus
}
#endif
#endif
