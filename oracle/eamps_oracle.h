/* eamps_oracle.h -- plain, slow, obviously-correct CPU oracle of the EA-MPS/MPO gate update.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_2307_16870_b200) never
 * links, imports or calls it, and shares no code, header or constant with it.
 *
 * Arithmetic: complex128 (C99 `double complex`), plain loops, no BLAS/LAPACK, its own textbook
 * cyclic one-sided (Hestenes) Jacobi SVD. Each function cites the passage it follows:
 *   PAPER.md = /root/reference/PAPER.md (LaTeX of arXiv:2307.16870), SPEC.md likewise,
 *   SURVEY §8(c) = the reading adopted where the paper is silent or garbled.
 *
 * Layouts: site tensor B_i row-major (chi_l, d, chi_r); theta / V column-major;
 * theta row (a,s) = a*d+s, column (t,c) = t*chi_r + c. Gates U[(s*d+t),(s'*d+t')] row-major.
 */
#ifndef EAMPS_ORACLE_H
#define EAMPS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_E_INVAL = -1, ORC_E_RANGE = -2, ORC_E_NOMEM = -3,
       ORC_E_NOCONV = -6, ORC_E_STATE = -8 };
enum { ORC_STRAT_NAIVE = 0, ORC_STRAT_NEAREST = 1, ORC_STRAT_GLOBAL = 2, ORC_STRAT_FIXED = 3 };
enum { ORC_RULE_PURE = 0, ORC_RULE_WANG = 1, ORC_RULE_RATIO = 2 };

typedef struct {
  int64_t gate_index; int32_t bond, chi_before, chi_after, capped;
  double target_f, achieved_f, discarded_weight; /* discarded = T_k / P */
} orc_record;

typedef struct orc_mps orc_mps;

/* ---- building blocks (each pinned by tests/test_oracle_*.py) ---------------------------- */
/* One-sided Jacobi SVD of A (m x n, column-major, complex128, interleaved re/im doubles).
 * On return A holds A*V (= X Sigma), V (n x n col-major) the accumulated rotations,
 * sigma[j] = ||(AV)_j|| (unsorted). PAPER.md:65 (M = U Lambda V^dagger); SURVEY §8(c) item 3. */
int orc_jacobi_svd(int m, int n, double* A, double* V, double* sigma, int max_sweeps, int* sweeps);
/* pi = argsort(sigma) descending (ties by index); T[k] = sum_{j>=k} sigma_pi[j]^2 summed from the
 * smallest, T has n+1 entries, T[n] = 0. PAPER.md:114 ("in decreasing order"), SURVEY §8(c) item 4. */
void orc_sort_tails(int n, const double* sigma, int32_t* pi, double* T);
/* log of the target truncation fidelity (PAPER.md:143-148 Eq. E14, 153, 158; SPEC.md:423 in log
 * space). Returns ORC_E_STATE if j >= n_planned (not for FIXED). */
int orc_target_log(int strategy, double log_fmin, int64_t n_planned, double log_E, int64_t j,
                   double log_f_fixed, double* log_t);
/* Smallest k >= 1 with T_k <= tau*P ("as close to but not lower than f_t"),
 * tau per rule (E10/E11 readings), capped at chi_cap,
 * clamped to kmax = min(m,n). f = achieved truncation fidelity; dlogE = its log. */
void orc_select(int rule, int n, const double* sigma_sorted, const double* T, double log_t,
                int chi_cap, int kmax, int* k, double* f, double* dlogE, int* capped);

/* ---- the state --------------------------------------------------------------------------- */
typedef struct {
  double f_min; int64_t n_planned; int32_t strategy, rule, chi_cap, max_sweeps;
  double f_fixed; /* per-truncation target for ORC_STRAT_FIXED (config-2 microbench) */
} orc_config;

int  orc_create(int n_sites, int d, const orc_config* cfg, orc_mps** out);
void orc_destroy(orc_mps*);
/* dims3 = {chi_l, d, chi_r}; B interleaved complex128 row-major; lam_left (chi_l) sets the
 * lambda of the bond left of `site` (only used for site 0 / explicit boundary legs). */
int  orc_import_site(orc_mps*, int site, const double* B, const int32_t* dims3);
int  orc_set_lambda(orc_mps*, int bond, const double* lam, int len);   /* bond in [-1, N-1] */
int  orc_export_site(orc_mps*, int site, double* B, int32_t* dims3);   /* B may be NULL */
int  orc_apply_gate1(orc_mps*, int site, const double* U);               /* d x d, no truncation */
int  orc_apply_gate2(orc_mps*, int site, const double* U);               /* d^2 x d^2 */
/* all gates of one layer: disjoint sites; contraction + SVD in parallel (OpenMP), selection
 * sequential in ascending-site order, then reabsorb in parallel. */
int  orc_apply_layer(orc_mps*, int n_gates, const int32_t* sites, const double* Us);
int  orc_bond_dims(orc_mps*, int32_t* out /* N-1 */);
int  orc_schmidt_values(orc_mps*, int bond, double* out, int cap, int* len);
int  orc_estimate(orc_mps*, double* log_est, int64_t* n_done, int* guarantee_held);
int  orc_records(orc_mps*, orc_record* out, int64_t cap, int64_t* len);
int  orc_set_ledger(orc_mps*, double log_E, int64_t j, int guarantee_held);
int  orc_amplitude(orc_mps*, const uint8_t* digits, double* re_im);
int  orc_statevector(orc_mps*, double* out, int64_t n_complex);
/* ---- observables (NEXT-4) -------------------------------------------------------
 * <a|b> = sum_sigma conj(C^a_sigma) C^b_sigma by left-to-right transfer matrices
 * E_{i+1} = sum_s A_i^{s dagger} E_i B_i^s (E2): the overlap of E7;
 * for d = 4 the Hilbert-Schmidt inner product Tr(rho_a^dagger rho_b) of the vectorised density
 * operators, the numerator and purities of the Wang fidelity E9. Same N and d. */
int  orc_overlap(orc_mps* a, orc_mps* b, double* re_im);
/* Tr rho = <<vec(I)|rho>> (d = 4 only: digits s = 2 sigma + sigma' with sigma = sigma', i.e. s in
 * {0, 3}); ORC_E_STATE for d = 2. */
int  orc_trace(orc_mps* s, double* re_im);
/* <psi|O_{site,site+1}|psi> / <psi|psi> (E5: arbitrary gauge, full left and right
 * environments); O is d^2 x d^2 row-major complex128, O[(s d + t), (s' d + t')] with s the physical
 * index of `site`. d = 2 only (ORC_E_STATE otherwise). */
int  orc_expectation2(orc_mps* s, int site, const double* O, double* re_im);
/* NEXT-1: exact canonicalisation: two sweeps of exact identity-gate two-site updates
 * (right to left, then left to right) with no truncation and no ledger entry; afterwards every B_i
 * (i >= 1) is right-orthonormal and every lambda_b holds the exact Schmidt values of bond b. */
int  orc_canonicalize(orc_mps* s);
/* the last gate's sorted spectrum (for parity on isolated updates) */
int  orc_last_spectrum(orc_mps*, int gate_in_layer, double* sigma_sorted, int cap, int* n);

#ifdef __cplusplus
}
#endif
#endif
