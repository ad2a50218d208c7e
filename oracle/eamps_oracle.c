/* eamps_oracle.c -- CPU oracle of the entanglement-aware MPS/MPO two-site gate update.
 *
 * TEST INFRASTRUCTURE ONLY (see eamps_oracle.h). complex128, plain loops, no BLAS/LAPACK.
 * It follows the paper step by step, in the paper's order (§V-§VI):
 *   contract the two tensors neighbouring the bond -> SVD with singular values in
 *   decreasing order (M = U Lambda V^dagger) -> pick the smallest rank
 *   whose truncation fidelity is "as close to but not lower than" the target with
 *   the target from E14 updated per strategy -> truncate and
 *   renormalise -> multiply the running estimate by f (E12).
 * Readings where the paper is silent or garbled are SURVEY.md §8(c) items 1-16; DESIGN.md lists
 * them. The state is kept in Vidal/Hastings B-lambda form.
 */
#include "eamps_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

/* ------------------------------------------------------------------------------------------ */
/* One-sided (Hestenes) Jacobi SVD, cyclic row order, SURVEY §8(c) algorithm item 3.          */
/* ------------------------------------------------------------------------------------------ */
int orc_jacobi_svd(int m, int n, double* A_, double* V_, double* sigma, int max_sweeps, int* sweeps) {
  cplx* A = (cplx*)A_;
  cplx* V = (cplx*)V_;
  double normF2 = 0.0;
  for (long i = 0; i < (long)m * n; ++i) normF2 += creal(A[i]) * creal(A[i]) + cimag(A[i]) * cimag(A[i]);
  /* skip pairs whose smaller column is below the rounding floor (eps*||A||_F)^2, eps = 2^-53 */
  const double eps = ldexp(1.0, -53);
  const double skip = eps * eps * normF2;
  /* convergence: |gamma| <= tol * sqrt(alpha beta), tol = max(1e-15, sqrt(m) 2^-52) */
  double tol = sqrt((double)(m > 0 ? m : 1)) * ldexp(1.0, -52);
  if (tol < 1e-15) tol = 1e-15;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) V[(long)j * n + i] = (i == j) ? 1.0 : 0.0;
  int sw = 0, converged = (n < 2);
  for (sw = 0; sw < max_sweeps && !converged; ++sw) {
    long rotated = 0;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        cplx* ap = A + (long)p * m;
        cplx* aq = A + (long)q * m;
        double alpha = 0.0, beta = 0.0;
        cplx gamma = 0.0;
        for (int i = 0; i < m; ++i) {
          alpha += creal(ap[i]) * creal(ap[i]) + cimag(ap[i]) * cimag(ap[i]);
          beta += creal(aq[i]) * creal(aq[i]) + cimag(aq[i]) * cimag(aq[i]);
          gamma += conj(ap[i]) * aq[i];
        }
        if ((alpha < beta ? alpha : beta) <= skip) continue;
        double g = cabs(gamma);
        if (!(g > tol * sqrt(alpha * beta))) continue;
        ++rotated;
        /* after the phase e, the 2x2 Gram is real; t solves t^2 + 2 zeta t - 1 = 0 */
        cplx e = gamma / g;
        double zeta = (beta - alpha) / (2.0 * g);
        double sg = (zeta >= 0.0) ? 1.0 : -1.0; /* sgn(0) = +1 */
        double t = sg / (fabs(zeta) + hypot(1.0, zeta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = c * t;
        cplx ce = conj(e);
        for (int i = 0; i < m; ++i) {
          cplx x = ap[i], y = aq[i];
          ap[i] = c * x - s * ce * y;
          aq[i] = s * x + c * ce * y;
        }
        cplx* vp = V + (long)p * n;
        cplx* vq = V + (long)q * n;
        for (int i = 0; i < n; ++i) {
          cplx x = vp[i], y = vq[i];
          vp[i] = c * x - s * ce * y;
          vq[i] = s * x + c * ce * y;
        }
      }
    }
    if (rotated == 0) converged = 1;
  }
  for (int j = 0; j < n; ++j) {
    double a = 0.0;
    for (int i = 0; i < m; ++i) {
      cplx z = A[(long)j * m + i];
      a += creal(z) * creal(z) + cimag(z) * cimag(z);
    }
    sigma[j] = sqrt(a);
  }
  if (sweeps) *sweeps = sw;
  return converged ? ORC_OK : ORC_E_NOCONV;
}

/* ------------------------------------------------------------------------------------------ */
/* Sort descending + tail sums (SURVEY §8(c) algorithm item 4)             */
/* ------------------------------------------------------------------------------------------ */
void orc_sort_tails(int n, const double* sigma, int32_t* pi, double* T) {
  for (int j = 0; j < n; ++j) pi[j] = j;
  /* plain insertion sort: obviously stable on ties (lower index first) */
  for (int a = 1; a < n; ++a) {
    int32_t v = pi[a];
    int b = a - 1;
    while (b >= 0 && (sigma[pi[b]] < sigma[v] || (sigma[pi[b]] == sigma[v] && pi[b] > v))) {
      pi[b + 1] = pi[b];
      --b;
    }
    pi[b + 1] = v;
  }
  T[n] = 0.0;
  for (int k = n - 1; k >= 0; --k) T[k] = T[k + 1] + sigma[pi[k]] * sigma[pi[k]];
}

/* ------------------------------------------------------------------------------------------ */
/* Ledger: target truncation fidelity, SURVEY §8(c) algorithm item 5 (SPEC.md:423 in logs)    */
/*   naive:   log t = log F_min / n                           (E14)          */
/*   global:  log t = min(0, (log F_min - log E)/R)            R = n - j   */
/*   nearest: log t = min(0, log F_min - log E - (R-1) log F_min / n)                         */
/*   fixed:   log t = log f_fixed    (config-2 microbench: per-update target, no ledger)      */
/* ------------------------------------------------------------------------------------------ */
int orc_target_log(int strategy, double log_fmin, int64_t n_planned, double log_E, int64_t j,
                   double log_f_fixed, double* log_t) {
  if (strategy == ORC_STRAT_FIXED) {
    *log_t = log_f_fixed < 0.0 ? log_f_fixed : 0.0;
    return ORC_OK;
  }
  if (j >= n_planned) return ORC_E_STATE;
  double R = (double)(n_planned - j);
  double lt;
  switch (strategy) {
    case ORC_STRAT_NAIVE: lt = log_fmin / (double)n_planned; break;
    case ORC_STRAT_GLOBAL: lt = (log_fmin - log_E) / R; break;
    case ORC_STRAT_NEAREST: lt = log_fmin - log_E - (R - 1.0) * log_fmin / (double)n_planned; break;
    default: return ORC_E_INVAL;
  }
  *log_t = lt < 0.0 ? lt : 0.0;
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Selection rule (SURVEY §8(c) algorithm item 6; readings 1-2 of E10/E11):                    */
/*   pure : f(k) = 1 - T_k/P          tau = 1 - t                                             */
/*   wang : f(k) = sqrt(1 - T_k/P)    tau = 1 - t^2                                           */
/*   ratio: f(k) = 1 - T_k/P          tau = 1 - t   (the MPO with the pure formula)           */
/*   k = min{k >= 1 : T_k <= tau P}; t = 1 -> k = max(1, #{sigma > 1e-14 sigma_0})*/
/* ------------------------------------------------------------------------------------------ */
void orc_select(int rule, int n, const double* s, const double* T, double log_t, int chi_cap,
                int kmax, int* k_out, double* f_out, double* dlogE, int* capped) {
  double P = T[0];
  int k;
  *capped = 0;
  if (n <= 0 || !(P > 0.0)) {
    *k_out = 1; *f_out = 1.0; *dlogE = 0.0;
    return;
  }
  double tau = (rule == ORC_RULE_WANG) ? -expm1(2.0 * log_t) : -expm1(log_t);
  if (tau <= 0.0) {
    k = 0;
    for (int j = 0; j < n; ++j)
      if (s[j] > 1e-14 * s[0]) ++k;
    if (k < 1) k = 1;
  } else {
    k = n;
    for (int kk = 1; kk <= n; ++kk)
      if (T[kk] <= tau * P) { k = kk; break; }
  }
  if (kmax > 0 && k > kmax) k = kmax;
  if (chi_cap > 0 && k > chi_cap) { k = chi_cap; *capped = 1; }
  double r = T[k] / P;
  if (rule == ORC_RULE_WANG) {
    *f_out = sqrt(1.0 - r);
    *dlogE = 0.5 * log1p(-r);
  } else {
    *f_out = 1.0 - r;
    *dlogE = log1p(-r);
  }
  *k_out = k;
}

/* ------------------------------------------------------------------------------------------ */
/* State                                                                                       */
/* ------------------------------------------------------------------------------------------ */
struct orc_mps {
  int N, d;
  orc_config cfg;
  double log_fmin, logE;
  int64_t j;
  int guarantee_held;
  int32_t *chl, *chr; /* per-site bond extents */
  cplx** B;           /* per site, row-major (chl, d, chr) */
  int32_t* lamlen;    /* per bond b in [-1, N-1] at index b+1 */
  double** lam;
  orc_record* rec;
  int64_t nrec, caprec;
  /* spectra of the last layer (per gate, in ascending-site order) */
  int last_count;
  double** last_sig;
  int* last_n;
};

static double* ones(int n) {
  double* x = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) x[i] = 1.0;
  return x;
}

int orc_create(int n_sites, int d, const orc_config* cfg, orc_mps** out) {
  if (n_sites < 2 || (d != 2 && d != 4) || !cfg || !out) return ORC_E_INVAL;
  if (!(cfg->f_min > 0.0 && cfg->f_min <= 1.0)) return ORC_E_INVAL;
  orc_mps* s = (orc_mps*)calloc(1, sizeof(orc_mps));
  s->N = n_sites; s->d = d; s->cfg = *cfg;
  if (s->cfg.max_sweeps <= 0) s->cfg.max_sweeps = 60;
  s->log_fmin = log(cfg->f_min);
  s->logE = 0.0; s->j = 0; s->guarantee_held = 1;
  s->chl = (int32_t*)malloc(sizeof(int32_t) * n_sites);
  s->chr = (int32_t*)malloc(sizeof(int32_t) * n_sites);
  s->B = (cplx**)calloc(n_sites, sizeof(cplx*));
  s->lamlen = (int32_t*)malloc(sizeof(int32_t) * (n_sites + 1));
  s->lam = (double**)calloc(n_sites + 1, sizeof(double*));
  /* |0...0>: B_i[0,0,0] = 1, lambda = [1] (SURVEY §8(c) algorithm item 1); for the MPO the
   * site index s = 2 sigma + sigma' = 0 is rho = |0..0><0..0|. */
  for (int i = 0; i < n_sites; ++i) {
    s->chl[i] = s->chr[i] = 1;
    s->B[i] = (cplx*)calloc(d, sizeof(cplx));
    s->B[i][0] = 1.0;
  }
  for (int b = 0; b <= n_sites; ++b) { s->lamlen[b] = 1; s->lam[b] = ones(1); }
  s->caprec = 1024;
  s->rec = (orc_record*)malloc(sizeof(orc_record) * s->caprec);
  *out = s;
  return ORC_OK;
}

static void free_last(orc_mps* s) {
  for (int g = 0; g < s->last_count; ++g) free(s->last_sig[g]);
  free(s->last_sig); free(s->last_n);
  s->last_sig = NULL; s->last_n = NULL; s->last_count = 0;
}

void orc_destroy(orc_mps* s) {
  if (!s) return;
  for (int i = 0; i < s->N; ++i) free(s->B[i]);
  for (int b = 0; b <= s->N; ++b) free(s->lam[b]);
  free(s->B); free(s->lam); free(s->lamlen); free(s->chl); free(s->chr); free(s->rec);
  free_last(s);
  free(s);
}

int orc_set_lambda(orc_mps* s, int bond, const double* lam, int len) {
  if (bond < -1 || bond > s->N - 1 || len < 1) return ORC_E_RANGE;
  free(s->lam[bond + 1]);
  s->lam[bond + 1] = (double*)malloc(sizeof(double) * len);
  memcpy(s->lam[bond + 1], lam, sizeof(double) * len);
  s->lamlen[bond + 1] = len;
  return ORC_OK;
}

int orc_import_site(orc_mps* s, int site, const double* B, const int32_t* dims3) {
  if (site < 0 || site >= s->N) return ORC_E_RANGE;
  if (dims3[1] != s->d || dims3[0] < 1 || dims3[2] < 1) return ORC_E_INVAL;
  long len = (long)dims3[0] * s->d * dims3[2];
  free(s->B[site]);
  s->B[site] = (cplx*)malloc(sizeof(cplx) * len);
  memcpy(s->B[site], B, sizeof(cplx) * len);
  s->chl[site] = dims3[0]; s->chr[site] = dims3[2];
  /* lambdas whose extent no longer matches are reset to ones (import is a test/bench facility) */
  if (s->lamlen[site] != dims3[0]) { free(s->lam[site]); s->lam[site] = ones(dims3[0]); s->lamlen[site] = dims3[0]; }
  if (s->lamlen[site + 1] != dims3[2]) { free(s->lam[site + 1]); s->lam[site + 1] = ones(dims3[2]); s->lamlen[site + 1] = dims3[2]; }
  return ORC_OK;
}

int orc_export_site(orc_mps* s, int site, double* B, int32_t* dims3) {
  if (site < 0 || site >= s->N) return ORC_E_RANGE;
  dims3[0] = s->chl[site]; dims3[1] = s->d; dims3[2] = s->chr[site];
  if (B) memcpy(B, s->B[site], sizeof(cplx) * (long)s->chl[site] * s->d * s->chr[site]);
  return ORC_OK;
}

int orc_apply_gate1(orc_mps* s, int site, const double* U_) {
  if (site < 0 || site >= s->N) return ORC_E_RANGE;
  const cplx* U = (const cplx*)U_;
  int d = s->d, l = s->chl[site], r = s->chr[site];
  cplx* B = s->B[site];
  cplx* tmp = (cplx*)malloc(sizeof(cplx) * d);
  for (int a = 0; a < l; ++a)
    for (int c = 0; c < r; ++c) {
      for (int x = 0; x < d; ++x) {
        cplx acc = 0.0;
        for (int y = 0; y < d; ++y) acc += U[x * d + y] * B[((long)a * d + y) * r + c];
        tmp[x] = acc;
      }
      for (int x = 0; x < d; ++x) B[((long)a * d + x) * r + c] = tmp[x];
    }
  free(tmp);
  return ORC_OK;
}

/* per-gate workspace of one layer */
typedef struct {
  int site, m, n, l, mid, r, k, capped, status, sweeps;
  cplx *Tp, *th, *V;   /* Theta' (m x n), theta -> theta V (m x n), V (n x n), column-major */
  double *sig, *T;      /* sigma (unsorted), tails (n+1) */
  int32_t* pi;
  double f, t, dlogE;
} gate_ws;

/* Contract: Theta'[(a,s),(t,c)] = sum U[s d + t, s' d + t'] B_i[a,s',b] B_{i+1}[b,t',c];
 * theta = diag(lambda_{i-1} (x) 1_d) Theta'   (SURVEY §8(c) algorithm item 2). */
static void contract(const orc_mps* s, gate_ws* w, const cplx* U) {
  int d = s->d, i = w->site;
  int l = w->l, mid = w->mid, r = w->r, m = w->m, n = w->n;
  const cplx* Bi = s->B[i];
  const cplx* Bj = s->B[i + 1];
  const double* lam = s->lam[i];
  /* C[(a,s'),(t',c)] = sum_b B_i[a,s',b] B_{i+1}[b,t',c] */
  cplx* C = (cplx*)calloc((long)m * n, sizeof(cplx));
  for (int a = 0; a < l; ++a)
    for (int sp = 0; sp < d; ++sp)
      for (int b = 0; b < mid; ++b) {
        cplx x = Bi[((long)a * d + sp) * mid + b];
        const cplx* row = Bj + (long)b * d * r; /* row b of B_{i+1} as (t',c) */
        cplx* crow = C + ((long)a * d + sp) * n;   /* row-major temp */
        for (int col = 0; col < n; ++col) crow[col] += x * row[col];
      }
  for (int a = 0; a < l; ++a)
    for (int c = 0; c < r; ++c)
      for (int ss = 0; ss < d; ++ss)
        for (int tt = 0; tt < d; ++tt) {
          cplx acc = 0.0;
          for (int sp = 0; sp < d; ++sp)
            for (int tp = 0; tp < d; ++tp)
              acc += U[(long)(ss * d + tt) * d * d + (sp * d + tp)] * C[((long)a * d + sp) * n + (tp * r + c)];
          long row = (long)a * d + ss, col = (long)tt * r + c;
          w->Tp[col * m + row] = acc;
          w->th[col * m + row] = lam[a] * acc;
        }
  free(C);
}

/* Hastings update (SURVEY §8(c) algorithm item 7; PAPER.md:65 left/right-normalised factors):
 *   nu = sqrt(sum_{j<k} sigma_pi_j^2); lambda_i <- sigma_pi[0:k]/nu;
 *   B_{i+1}[j,t,c] <- conj(V[(t,c), pi_j]);  B_i[(a,s), j] <- (Theta' V_{:,pi_j}) / nu          */
static void reabsorb(orc_mps* s, gate_ws* w) {
  int d = s->d, i = w->site, m = w->m, n = w->n, k = w->k;
  double nu2 = 0.0;
  for (int j = 0; j < k; ++j) nu2 += w->sig[w->pi[j]] * w->sig[w->pi[j]];
  double nu = sqrt(nu2);
  double* lam = (double*)malloc(sizeof(double) * k);
  for (int j = 0; j < k; ++j) lam[j] = w->sig[w->pi[j]] / nu;
  cplx* Bn = (cplx*)malloc(sizeof(cplx) * (long)k * n);       /* (k, d, r) */
  for (int j = 0; j < k; ++j)
    for (int col = 0; col < n; ++col) Bn[(long)j * n + col] = conj(w->V[(long)w->pi[j] * n + col]);
  cplx* Bm = (cplx*)malloc(sizeof(cplx) * (long)m * k);       /* (l, d, k) */
  for (int row = 0; row < m; ++row)
    for (int j = 0; j < k; ++j) {
      cplx acc = 0.0;
      const cplx* v = w->V + (long)w->pi[j] * n;
      for (int col = 0; col < n; ++col) acc += w->Tp[(long)col * m + row] * v[col];
      Bm[(long)row * k + j] = acc / nu;
    }
  free(s->B[i]); free(s->B[i + 1]);
  s->B[i] = Bm; s->B[i + 1] = Bn;
  s->chr[i] = k; s->chl[i + 1] = k;
  free(s->lam[i + 1]);
  s->lam[i + 1] = lam; s->lamlen[i + 1] = k;
  (void)d;
}

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

int orc_apply_layer(orc_mps* s, int G, const int32_t* sites, const double* Us_) {
  if (G < 0) return ORC_E_INVAL;
  if (G == 0) return ORC_OK;
  int d = s->d, dd = d * d;
  const cplx* Us = (const cplx*)Us_;
  /* validate: in range, disjoint (SURVEY §8(b) conventions) */
  int* ord = (int*)malloc(sizeof(int) * G * 2);
  for (int g = 0; g < G; ++g) {
    if (sites[g] < 0 || sites[g] >= s->N - 1) { free(ord); return ORC_E_RANGE; }
    ord[2 * g] = sites[g]; ord[2 * g + 1] = g;
  }
  qsort(ord, G, 2 * sizeof(int), cmp_int);
  for (int g = 1; g < G; ++g)
    if (ord[2 * g] < ord[2 * (g - 1)] + 2) { free(ord); return ORC_E_INVAL; }
  for (int g = 0; g < G; ++g) {
    int i = ord[2 * g];
    if (s->chr[i] != s->chl[i + 1] || s->lamlen[i] != s->chl[i]) { free(ord); return ORC_E_INVAL; }
  }
  if (s->cfg.strategy != ORC_STRAT_FIXED && s->j + G > s->cfg.n_planned) { free(ord); return ORC_E_STATE; }
  for (long x = 0; x < (long)G * dd * dd; ++x)
    if (!isfinite(creal(Us[x])) || !isfinite(cimag(Us[x]))) { free(ord); return ORC_E_INVAL; }

  gate_ws* W = (gate_ws*)calloc(G, sizeof(gate_ws));
  for (int g = 0; g < G; ++g) {
    gate_ws* w = &W[g];
    w->site = ord[2 * g];
    w->l = s->chl[w->site]; w->mid = s->chr[w->site]; w->r = s->chr[w->site + 1];
    w->m = w->l * d; w->n = d * w->r;
  }
  /* phase 1 (independent gates): contract + SVD + sort/tails */
#pragma omp parallel for schedule(dynamic, 1)
  for (int g = 0; g < G; ++g) {
    gate_ws* w = &W[g];
    const cplx* U = Us + (long)ord[2 * g + 1] * dd * dd;
    w->Tp = (cplx*)malloc(sizeof(cplx) * (long)w->m * w->n);
    w->th = (cplx*)malloc(sizeof(cplx) * (long)w->m * w->n);
    w->V = (cplx*)malloc(sizeof(cplx) * (long)w->n * w->n);
    w->sig = (double*)malloc(sizeof(double) * w->n);
    w->T = (double*)malloc(sizeof(double) * (w->n + 1));
    w->pi = (int32_t*)malloc(sizeof(int32_t) * w->n);
    contract(s, w, U);
    w->status = orc_jacobi_svd(w->m, w->n, (double*)w->th, (double*)w->V, w->sig, s->cfg.max_sweeps, &w->sweeps);
    orc_sort_tails(w->n, w->sig, w->pi, w->T);
  }
  int status = ORC_OK;
  for (int g = 0; g < G; ++g)
    if (W[g].status != ORC_OK) status = W[g].status;
  /* phase 2 (sequential, ascending site = canonical ledger order) */
  if (status == ORC_OK) {
    for (int g = 0; g < G; ++g) {
      gate_ws* w = &W[g];
      double log_t;
      int rc = orc_target_log(s->cfg.strategy, s->log_fmin, s->cfg.n_planned, s->logE, s->j,
                              log(s->cfg.f_fixed > 0 ? s->cfg.f_fixed : 1.0), &log_t);
      if (rc != ORC_OK) { status = rc; break; }
      double* ssorted = (double*)malloc(sizeof(double) * w->n);
      for (int j = 0; j < w->n; ++j) ssorted[j] = w->sig[w->pi[j]];
      int kmax = w->m < w->n ? w->m : w->n;
      orc_select(s->cfg.rule, w->n, ssorted, w->T, log_t, s->cfg.chi_cap, kmax, &w->k, &w->f, &w->dlogE, &w->capped);
      free(ssorted);
      w->t = exp(log_t);
      if (w->capped) s->guarantee_held = 0;
      s->logE += w->dlogE;
      if (s->nrec == s->caprec) {
        s->caprec *= 2;
        s->rec = (orc_record*)realloc(s->rec, sizeof(orc_record) * s->caprec);
      }
      orc_record* rr = &s->rec[s->nrec++];
      rr->gate_index = s->j; rr->bond = w->site; rr->chi_before = w->mid; rr->chi_after = w->k;
      rr->capped = w->capped; rr->target_f = w->t; rr->achieved_f = w->f;
      rr->discarded_weight = w->T[0] > 0 ? w->T[w->k] / w->T[0] : 0.0;
      s->j += 1;
    }
  }
  /* phase 3 (independent gates): reabsorb */
  if (status == ORC_OK) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int g = 0; g < G; ++g) reabsorb(s, &W[g]);
    free_last(s);
    s->last_count = G;
    s->last_sig = (double**)malloc(sizeof(double*) * G);
    s->last_n = (int*)malloc(sizeof(int) * G);
    for (int g = 0; g < G; ++g) {
      s->last_n[g] = W[g].n;
      s->last_sig[g] = (double*)malloc(sizeof(double) * W[g].n);
      for (int j = 0; j < W[g].n; ++j) s->last_sig[g][j] = W[g].sig[W[g].pi[j]];
    }
  }
  for (int g = 0; g < G; ++g) {
    free(W[g].Tp); free(W[g].th); free(W[g].V); free(W[g].sig); free(W[g].T); free(W[g].pi);
  }
  free(W); free(ord);
  return status;
}

int orc_apply_gate2(orc_mps* s, int site, const double* U) {
  int32_t st = site;
  return orc_apply_layer(s, 1, &st, U);
}

int orc_bond_dims(orc_mps* s, int32_t* out) {
  for (int i = 0; i < s->N - 1; ++i) out[i] = s->chr[i];
  return ORC_OK;
}

int orc_schmidt_values(orc_mps* s, int bond, double* out, int cap, int* len) {
  /* bonds -1 and N-1 are the trivial boundary vectors [1] (readable like set_lambda's range) */
  if (bond < -1 || bond > s->N - 1) return ORC_E_RANGE;
  int L = s->lamlen[bond + 1];
  *len = L;
  for (int j = 0; j < L && j < cap; ++j) out[j] = s->lam[bond + 1][j];
  return ORC_OK;
}

int orc_estimate(orc_mps* s, double* log_est, int64_t* n_done, int* guarantee_held) {
  *log_est = s->logE; *n_done = s->j; *guarantee_held = s->guarantee_held;
  return ORC_OK;
}

/* Ledger token plumbing for the multi-rank tests: replace (log E, j, guarantee).
 * No arithmetic: the next truncation reads these exactly as if the preceding gates had run here. */
int orc_set_ledger(orc_mps* s, double log_E, int64_t j, int guarantee_held) {
  if (!(log_E <= 0.0) || j < 0) return ORC_E_INVAL;
  s->logE = log_E; s->j = j; s->guarantee_held = guarantee_held;
  return ORC_OK;
}

int orc_records(orc_mps* s, orc_record* out, int64_t cap, int64_t* len) {
  *len = s->nrec;
  for (int64_t r = 0; r < s->nrec && r < cap; ++r) out[r] = s->rec[r];
  return ORC_OK;
}

/* <digits|psi> = prod_i B_i[:, digit_i, :] (B = Gamma lambda, E2 PAPER.md:38-41) */
int orc_amplitude(orc_mps* s, const uint8_t* digits, double* re_im) {
  if (s->chl[0] != 1 || s->chr[s->N - 1] != 1) return ORC_E_STATE;
  int d = s->d;
  cplx* v = (cplx*)malloc(sizeof(cplx));
  v[0] = 1.0;
  for (int i = 0; i < s->N; ++i) {
    if (digits[i] >= d) { free(v); return ORC_E_INVAL; }
    int l = s->chl[i], r = s->chr[i];
    cplx* nv = (cplx*)calloc(r, sizeof(cplx));
    for (int a = 0; a < l; ++a)
      for (int c = 0; c < r; ++c) nv[c] += v[a] * s->B[i][((long)a * d + digits[i]) * r + c];
    free(v);
    v = nv;
  }
  re_im[0] = creal(v[0]); re_im[1] = cimag(v[0]);
  free(v);
  return ORC_OK;
}

/* full d^N vector, site 0 the most significant digit (SURVEY §8(c) algorithm item 1) */
int orc_statevector(orc_mps* s, double* out, int64_t n_complex) {
  if (s->chl[0] != 1 || s->chr[s->N - 1] != 1) return ORC_E_STATE;
  int d = s->d;
  int64_t total = 1;
  for (int i = 0; i < s->N; ++i) total *= d;
  if (n_complex < total) return ORC_E_RANGE;
  /* S has rows = prefix index, cols = bond */
  int64_t rows = 1;
  int cols = 1;
  cplx* S = (cplx*)malloc(sizeof(cplx));
  S[0] = 1.0;
  for (int i = 0; i < s->N; ++i) {
    int r = s->chr[i];
    cplx* NS = (cplx*)calloc((size_t)rows * d * r, sizeof(cplx));
    for (int64_t p = 0; p < rows; ++p)
      for (int a = 0; a < cols; ++a) {
        cplx x = S[p * cols + a];
        if (x == 0.0) continue;
        for (int sd = 0; sd < d; ++sd)
          for (int c = 0; c < r; ++c) NS[(p * d + sd) * r + c] += x * s->B[i][((long)a * d + sd) * r + c];
      }
    free(S);
    S = NS; rows *= d; cols = r;
  }
  memcpy(out, S, sizeof(cplx) * total);
  free(S);
  return ORC_OK;
}

int orc_last_spectrum(orc_mps* s, int g, double* sig, int cap, int* n) {
  if (g < 0 || g >= s->last_count) return ORC_E_RANGE;
  *n = s->last_n[g];
  for (int j = 0; j < s->last_n[g] && j < cap; ++j) sig[j] = s->last_sig[g][j];
  return ORC_OK;
}

/* ---- observables (NEXT-4) -------------------------------------------------------------------- */
/* E_{i+1}[a',b'] = sum_s sum_{a,b} conj(A_i[a,s,a']) E_i[a,b] B_i[b,s,b'], E_0 = [1] (E2 with the bra
 * conjugated: PAPER.md:38-41, 91-93). Plain loops. Returns the 1 x 1 result. */
static int transfer_overlap(const orc_mps* a, const orc_mps* b, cplx* out) {
  if (a->N != b->N || a->d != b->d) return ORC_E_INVAL;
  if (a->chl[0] != 1 || b->chl[0] != 1 || a->chr[a->N - 1] != 1 || b->chr[b->N - 1] != 1) return ORC_E_STATE;
  const int d = a->d;
  cplx* E = (cplx*)malloc(sizeof(cplx));
  E[0] = 1.0;
  int la = 1, lb = 1;
  for (int i = 0; i < a->N; ++i) {
    const int ra = a->chr[i], rb = b->chr[i];
    cplx* En = (cplx*)calloc((size_t)ra * rb, sizeof(cplx));
    for (int s2 = 0; s2 < d; ++s2)
      for (int x = 0; x < la; ++x)
        for (int y = 0; y < lb; ++y) {
          const cplx e = E[(long)x * lb + y];
          if (e == 0.0) continue;
          for (int xp = 0; xp < ra; ++xp) {
            const cplx ca = conj(a->B[i][((long)x * d + s2) * ra + xp]) * e;
            for (int yp = 0; yp < rb; ++yp) En[(long)xp * rb + yp] += ca * b->B[i][((long)y * d + s2) * rb + yp];
          }
        }
    free(E);
    E = En;
    la = ra;
    lb = rb;
  }
  *out = E[0];
  free(E);
  return ORC_OK;
}

int orc_overlap(orc_mps* a, orc_mps* b, double* re_im) {
  cplx v;
  int st = transfer_overlap(a, b, &v);
  if (st != ORC_OK) return st;
  re_im[0] = creal(v);
  re_im[1] = cimag(v);
  return ORC_OK;
}

/* Tr rho = sum over sigma of <sigma sigma'|rho> with sigma = sigma': per site the vector
 * v_{i+1}[c] = sum_a v_i[a] (B_i[a,0,c] + B_i[a,3,c])  (s = 2 sigma + sigma') */
int orc_trace(orc_mps* s, double* re_im) {
  if (s->d != 4) return ORC_E_STATE;
  if (s->chl[0] != 1 || s->chr[s->N - 1] != 1) return ORC_E_STATE;
  cplx* v = (cplx*)malloc(sizeof(cplx));
  v[0] = 1.0;
  for (int i = 0; i < s->N; ++i) {
    const int l = s->chl[i], r = s->chr[i];
    cplx* nv = (cplx*)calloc(r, sizeof(cplx));
    for (int x = 0; x < l; ++x)
      for (int c = 0; c < r; ++c) nv[c] += v[x] * (s->B[i][((long)x * 4 + 0) * r + c] + s->B[i][((long)x * 4 + 3) * r + c]);
    free(v);
    v = nv;
  }
  re_im[0] = creal(v[0]);
  re_im[1] = cimag(v[0]);
  free(v);
  return ORC_OK;
}

/* E5, arbitrary gauge: L = left environment of sites < k (transfer of psi with
 * itself), R = right environment of sites > k+1 (right-to-left transfer), then
 * <O> = sum L[a,a''] conj(theta[a,s,t,c]) O[st,s't'] theta[a'',s',t',c''] R[c,c''] / <psi|psi>,
 * theta[a,s,t,c] = sum_b B_k[a,s,b] B_{k+1}[b,t,c]. */
int orc_expectation2(orc_mps* s, int k, const double* Od, double* re_im) {
  if (s->d != 2) return ORC_E_STATE;
  if (k < 0 || k >= s->N - 1) return ORC_E_RANGE;
  if (s->chl[0] != 1 || s->chr[s->N - 1] != 1) return ORC_E_STATE;
  const int d = 2;
  const cplx* O = (const cplx*)Od;
  /* left environment L (chl[k] x chl[k]) */
  cplx* L = (cplx*)malloc(sizeof(cplx));
  L[0] = 1.0;
  int l = 1;
  for (int i = 0; i < k; ++i) {
    const int r = s->chr[i];
    cplx* Ln = (cplx*)calloc((size_t)r * r, sizeof(cplx));
    for (int s2 = 0; s2 < d; ++s2)
      for (int x = 0; x < l; ++x)
        for (int y = 0; y < l; ++y) {
          const cplx e = L[(long)x * l + y];
          if (e == 0.0) continue;
          for (int xp = 0; xp < r; ++xp) {
            const cplx ca = conj(s->B[i][((long)x * d + s2) * r + xp]) * e;
            for (int yp = 0; yp < r; ++yp) Ln[(long)xp * r + yp] += ca * s->B[i][((long)y * d + s2) * r + yp];
          }
        }
    free(L);
    L = Ln;
    l = r;
  }
  /* right environment R (chr[k+1] x chr[k+1]): R_i[c,c''] = sum_s B_i[c,s,x] conj... from the right */
  cplx* R = (cplx*)malloc(sizeof(cplx));
  R[0] = 1.0;
  int rr = 1;
  for (int i = s->N - 1; i > k + 1; --i) {
    const int li = s->chl[i];
    cplx* Rn = (cplx*)calloc((size_t)li * li, sizeof(cplx));
    for (int s2 = 0; s2 < d; ++s2)
      for (int x = 0; x < li; ++x)
        for (int y = 0; y < li; ++y) {
          cplx acc = 0.0;
          for (int xp = 0; xp < rr; ++xp)
            for (int yp = 0; yp < rr; ++yp)
              acc += conj(s->B[i][((long)x * d + s2) * rr + xp]) * R[(long)xp * rr + yp] *
                     s->B[i][((long)y * d + s2) * rr + yp];
          Rn[(long)x * li + y] += acc;
        }
    free(R);
    R = Rn;
    rr = li;
  }
  /* theta (l, d, d, rr) */
  const int mid = s->chr[k];
  cplx* th = (cplx*)calloc((size_t)l * d * d * rr, sizeof(cplx));
  for (int a = 0; a < l; ++a)
    for (int s1 = 0; s1 < d; ++s1)
      for (int b = 0; b < mid; ++b) {
        const cplx u = s->B[k][((long)a * d + s1) * mid + b];
        for (int t = 0; t < d; ++t)
          for (int c = 0; c < rr; ++c)
            th[(((long)a * d + s1) * d + t) * rr + c] += u * s->B[k + 1][((long)b * d + t) * rr + c];
      }
  /* O theta */
  cplx* Oth = (cplx*)calloc((size_t)l * d * d * rr, sizeof(cplx));
  for (int a = 0; a < l; ++a)
    for (int c = 0; c < rr; ++c)
      for (int st = 0; st < d * d; ++st)
        for (int sp = 0; sp < d * d; ++sp)
          Oth[((long)a * d * d + st) * rr + c] += O[st * d * d + sp] * th[((long)a * d * d + sp) * rr + c];
  cplx num = 0.0, den = 0.0;
  for (int a = 0; a < l; ++a)
    for (int a2 = 0; a2 < l; ++a2) {
      const cplx la = L[(long)a * l + a2];
      if (la == 0.0) continue;
      for (int st = 0; st < d * d; ++st)
        for (int c = 0; c < rr; ++c)
          for (int c2 = 0; c2 < rr; ++c2) {
            const cplx w = la * conj(th[((long)a * d * d + st) * rr + c]) * R[(long)c * rr + c2];
            num += w * Oth[((long)a2 * d * d + st) * rr + c2];
            den += w * th[((long)a2 * d * d + st) * rr + c2];
          }
    }
  free(L); free(R); free(th); free(Oth);
  if (den == 0.0) return ORC_E_STATE;
  const cplx v = num / den;
  re_im[0] = creal(v);
  re_im[1] = cimag(v);
  return ORC_OK;
}

/* ---- NEXT-1: exact canonicalisation ------------------------------------------------
 * "We apply QR to each tensor ... and similarly apply a RQ ... The state is now in canonical form"
 * (PAPER.md:76); "the canonical form ... is enforced throughout". In the B-lambda form
 * (reading 4) this is two sweeps of exact two-site updates with the identity gate, no
 * truncation (t = 1: keep every sigma > 1e-14 sigma_0) and no ledger entry:
 *   right to left (bonds N-2 .. 0): B_{i+1} <- V^H  -> every B_1 .. B_{N-1} right-orthonormal;
 *   left to right (bonds 0 .. N-2): theta = lambda_{i-1} B_i B_{i+1} is then the exact Schmidt
 *     decomposition at bond i (left basis orthonormal by induction, right environment right-canonical),
 *     so lambda_i <- its singular values (renormalised) are the exact Schmidt values.
 * The represented vector is unchanged up to the global scale. */
int orc_canonicalize(orc_mps* s) {
  const int d = s->d, dd = d * d, N = s->N;
  const orc_config keep = s->cfg;
  const double logE = s->logE;
  const int64_t j = s->j, nrec = s->nrec;
  const int gh = s->guarantee_held;
  s->cfg.strategy = ORC_STRAT_FIXED;
  s->cfg.f_fixed = 1.0;
  s->cfg.chi_cap = 0;
  double* ident = (double*)calloc((size_t)2 * dd * dd, sizeof(double));
  for (int x = 0; x < dd; ++x) ident[2 * (x * dd + x)] = 1.0;
  int st = ORC_OK;
  for (int i = N - 2; i >= 0 && st == ORC_OK; --i) st = orc_apply_gate2(s, i, ident);
  for (int i = 0; i <= N - 2 && st == ORC_OK; ++i) st = orc_apply_gate2(s, i, ident);
  free(ident);
  s->cfg = keep;
  s->logE = logE;
  s->j = j;
  s->nrec = nrec;
  s->guarantee_held = gh;
  return st;
}
