/*
 * p2s_oracle.h -- CPU ORACLE for the product-to-sum (p2s) element fill.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * algorithm (/root/reference/proj/src/assembly.cpp, chebyshev.cpp,
 * quadrature.cpp, verify.cpp), generalised from the reference's 2-D Chebyshev
 * specialisation to the paper's general 3-D scheme (Eqs. (1)-(4))
 * with Legendre kernel polynomials.  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline / reference arm may load it.  The product path
 * (paper_1703_09619_b200/, libp2s_b200.so) never links or calls it.
 *
 * Pinning:
 *   - por_gauss_legendre restates quadrature.cpp:13-53 and is checked bitwise
 *     against the compiled reference (tests/golden/ref2d_*.npz).
 *   - the generic separable engine (por_term_moments / por_term_contract /
 *     por_term_direct) is run in a 2-D Chebyshev mode (por_cheb2d_element)
 *     and checked against the compiled reference's compute_kernel_tables /
 *     assemble_p2s_element / assemble_direct_element on seeded curved
 *     elements and the reference's own known-answer tests.
 *   - the 3-D Legendre instance is pinned by p2s == direct quadrature and by
 *     pointwise identity checks of the Legendre product-to-sum tables.
 */
#ifndef P2S_ORACLE_H
#define P2S_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POR_MAX_TERMS 4

/* per-direction operator pair (test, trial): P = value, D = derivative */
enum { POR_PP = 0, POR_DD = 1, POR_DP = 2, POR_PD = 3 };

/* coupling-factor generators (BASELINE.json configs) */
enum { POR_ALPHA_SINE = 0, POR_ALPHA_JACOBIAN = 1, POR_ALPHA_EXPSIN = 2 };

typedef struct {
  int n_comp;                     /* 1 (scalar) or 3 (vector)              */
  int order[3];                   /* N_u, N_v, N_w: basis P_0..P_{N-1}     */
  int n_terms;                    /* N_s                                    */
  int kind[POR_MAX_TERMS][3];     /* POR_PP/DD/DP/PD per term, direction   */
  int nq[3];                      /* Gauss-Legendre points per direction   */
  int basis;                      /* 0 modal, 1 conforming (por_conforming) */
} por_problem;

/* ---------------- 1-D primitives ---------------- */

/* Restates gauss_legendre (quadrature.cpp:27-53): Newton on the Legendre
 * recurrence (quadrature.cpp:13-24), symmetric nodes, exact centre node. */
void por_gauss_legendre(int n, double* nodes, double* weights);

/* P_k(x) and P'_k(x), k < K, long-double three-term recurrences. */
void por_legendre_eval(int K, double x, double* P, double* dP);

/* Number of kernel polynomials for an operator pair: degree bound of the
 * product + 1 (paper Eq. (3): K1 = m1+m2, m1+m2-1, m1+m2-2). */
int por_kernel_count(int kind, int N);

/* Legendre product-to-sum table C[a][b][k] (a,b < N, k < K) such that
 * f_a(x) g_b(x) = sum_k C[a][b][k] P_k(x), f,g = P or P' per kind.
 * Role of product_to_sum (chebyshev.cpp:156-178) for the Legendre family. */
void por_legendre_coef(int kind, int N, int K, double* C);

/* The reference's conforming change of basis, conforming_matrix(n-1)
 * (assembly.cpp:476-489): R is n x n, column m holds the modal coefficients of
 * phi_m: phi_0 = (P_0 - P_1)/2, phi_1 = (P_0 + P_1)/2, phi_m = P_m - P_{m mod 2}.
 * Row-major R[a*n + m]; n >= 2. */
void por_conforming_matrix(int n, double* R);

/* ---------------- generic separable engine ---------------- */

typedef struct {
  int nt, nr;            /* test / trial basis counts                     */
  int K;                 /* kernel polynomial count                       */
  int nq;                /* quadrature points                             */
  const double* phi;     /* [K][nq] kernel polynomial values (x weights)  */
  const double* coef;    /* [nt][nr][K] product-to-sum coefficients       */
  const double* btest;   /* [nt][nq] test basis values (direct path)      */
  const double* btrial;  /* [nr][nq] trial basis values (direct path)     */
  const double* wq;      /* [nq] weights for the direct path, NULL = 1    */
  int symmetric;         /* btest == btrial, nt == nr (direct-path reuse) */
} por_dir;

typedef struct { por_dir d[3]; } por_term;

/* Moment stage (compute_kernel_tables, assembly.cpp:276-314), sum-factorised:
 * I[k0][k1][k2] = sum_q alpha[q2][q1][q0] phi0[k0][q0] phi1[k1][q1] phi2[k2][q2] */
void por_term_moments(const por_term* t, const double* alpha, double* I, double* scratch);
long por_term_moment_scratch(const por_term* t);

/* Contraction stage (assemble_p2s_element, assembly.cpp:375-474): adds
 * sum_k C0[m1][m2][k0] C1[n1][n2][k1] C2[p1][p2][k2] I[k0][k1][k2] into the
 * block M[(m1 n1 p1)][(m2 n2 p2)] (row-major, leading dimension ldM). */
void por_term_contract(const por_term* t, const double* I, double* M, long ldM, double* scratch);
long por_term_contract_scratch(const por_term* t);

/* Direct fill (assemble_direct_element, assembly.cpp:142-274): every entry
 * by one full 3-D quadrature, canonical entries mirrored when a direction is
 * symmetric.  Adds into M. */
void por_term_direct(const por_term* t, const double* alpha, double* M, long ldM);

/* ---------------- 3-D Legendre problem ---------------- */

typedef struct por_tables por_tables;

por_tables* por_create(const por_problem* pb);
void por_destroy(por_tables* t);

/* sizes in doubles */
long por_alpha_per_elem(const por_tables* t);  /* P * S * nq_w nq_v nq_u        */
long por_moments_per_elem(const por_tables* t);/* P * sum_s K_u K_v K_w         */
int por_n_tot(const por_tables* t);            /* n_comp N_u N_v N_w            */
int por_K(const por_tables* t, int term, int dir);
long por_moment_offset(const por_tables* t, int pair, int term); /* within elem */

/* read-only views of the tables (for cross-checks against the product) */
const double* por_nodes(const por_tables* t, int dir);
const double* por_weights(const por_tables* t, int dir);
const double* por_phi(const por_tables* t, int term, int dir);   /* [K][nq]      */
const double* por_coef(const por_tables* t, int term, int dir);  /* [N][N][K]    */

/* Seeded coupling factor alpha[e][pair][s][q_w][q_v][q_u] (harness input;
 * role of build_element_quad, assembly.cpp:51-119).  lo/hi: frequency range
 * of the sine family.  Elements e0 .. e0+n-1. */
void por_alpha_gen(const por_tables* t, int alpha_kind, double lo, double hi, uint64_t seed,
                   int64_t e0, int64_t n, double* alpha);

/* Per-element parameters of the generator (for device-generator checks). */
double por_uniform(uint64_t seed, int64_t elem, int slot, int j);

/* Batch entry points.  threads <= 1: serial; else a fill_elements-style pool
 * (assembly.cpp:654-700) over elements.  Results are thread-count independent. */
void por_moments(const por_tables* t, const double* alpha, int64_t n, double* I, int threads);
void por_contract(const por_tables* t, const double* I, int64_t n, double* M, int64_t ldM,
                  int threads);
void por_fill(const por_tables* t, const double* alpha, int64_t n, double* M, int64_t ldM,
              int threads);
long por_direct_sample(const por_tables* t, const double* alpha, int m1_lo, int m1_hi, double* M, int64_t ldM,
                       long* total_pairs);
void por_direct(const por_tables* t, const double* alpha, int64_t n, double* M, int64_t ldM,
                int threads);

/* ---------------- comparator (verify.cpp:81-99) ---------------- */

/* Pass if |a-b| <= rtol*max(|a|,|b|) or |a-b| <= 1e-12*max(max|A|,max|B|).
 * Returns 1 on pass; on failure writes the first offending (i, j). */
int por_block_close(const double* a, int64_t lda, const double* b, int64_t ldb, int rows,
                    int cols, double rtol, int* bad_i, int* bad_j);

/* ---------------- 2-D Chebyshev mode (reference pin) ---------------- */

enum { POR_T = 0, POR_U = 1, POR_TNS = 2 };
double por_cheb_eval(int fam, int n, double u);
/* product_to_sum (chebyshev.cpp:156-178); returns term count (<= 2). */
int por_cheb_p2s(int fam_a, int a, int fam_b, int b, double* coeff, int* fam, int* deg);

/* Reference 2-D element on the generic engine.  Inputs: orders M, N, rule
 * size nq, GL nodes, and the four weighted coupling grids of
 * build_element_quad (assembly.cpp:102-106) as [i_u][j_v] row-major nq x nq.
 * Outputs (each may be NULL):
 *   tables: Ks (2M+1)(2N+1), Kuu (2M+1)(2N+1), Kuv 2M*2N, Kvv (2M+1)(2N+1)
 *   p2s / direct: Suu Suv Svu Svv Muu Muv Mvu Mvv, sizes
 *     n_eu = M(N+1), n_ev = (M+1)N, blocks row-major (uu n_eu^2, uv n_eu n_ev,
 *     vu n_ev n_eu, vv n_ev^2) concatenated in that order, S then M. */
void por_cheb2d_element(int M, int N, int nq, const double* nodes, const double* ws,
                        const double* wuu, const double* wuv, const double* wvv,
                        double* tables, double* p2s_blocks, double* direct_blocks);

#ifdef __cplusplus
}
#endif
#endif
