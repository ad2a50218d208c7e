/* eamps.h -- C ABI of the B200-native entanglement-aware MPS/MPO two-site gate update.
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, the LaTeX of arXiv:2307.16870):
 *   a two-qubit gate on sites (i, i+1) of an MPS (E2) or of a vectorised MPO
 *   (E4, local dimension d = 4) is applied by "contracting both tensors
 *   neighbouring the bond" and "performing its SVD", then truncating to the
 *   smallest rank whose truncation fidelity (E10 pure / E11 mixed) is "as close
 *   to but not lower than" a target f_t. The target comes from the input fidelity
 *   F_min and the number n of two-qubit gates (E14) and is updated after
 *   every truncation by the chosen strategy (naive / nearest / global). The running
 *   product of truncation fidelities estimates the final state fidelity (E12/E13,
 *   PAPER.md:132-139). A bond-dimension cap may force deeper cuts, in which case the guarantee is
 *   lost.
 * Readings where the paper is silent or garbled are listed in DESIGN.md ("Readings").
 *
 * Memory model. Every device byte the library touches lives inside ONE caller-provided device
 * slab (cfg.dev_slab, cfg.slab_bytes; e.g. torch.empty(bytes, dtype=uint8, device="cuda")). The
 * caller keeps it alive until mps_destroy. Site tensors and Schmidt vectors are carved from it by
 * a device-side pool allocator; per-layer workspace from its top. Host pointers passed in are
 * read before the call returns (the caller may free them at once); outputs go to caller buffers.
 * All work is issued on cfg.stream (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream).
 *
 * Layouts. Complex numbers are interleaved (re, im) float32 ("c64") unless stated. A site tensor
 * B_i is row-major (chi_l, d, chi_r). A gate U is row-major d^2 x d^2 with
 * U[(s*d+t), (s'*d+t')], s the physical index of `site` (the left / more significant one).
 * For d = 4 the physical index is s = 2*sigma + sigma' (ket, bra) and the "gate" is the 16x16
 * superoperator S (workloads.mpo_gate). The represented vector is psi = B_0 B_1 ... B_{N-1}
 * with site 0 the most significant digit.
 *
 * Errors. Argument errors are returned synchronously. Device-side errors (Jacobi
 * non-convergence, non-finite values, pool exhaustion) are sticky and reported by the next
 * synchronising call (mps_apply_layer's end-of-layer readback, mps_fidelity_estimate,
 * mps_amplitude, mps_to_statevector, mps_sync). After MPS_E_CUDA the handle is poisoned: only
 * mps_destroy is legal. One handle is single-writer (not thread-safe).
 */
#ifndef EAMPS_H
#define EAMPS_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct mps_handle* mps_t;
typedef int32_t mps_status;

enum {
  MPS_OK = 0,
  MPS_E_INVAL = -1,   /* bad argument: overlapping gates, non-finite gate entry, bad dims */
  MPS_E_RANGE = -2,   /* site / bond index out of range */
  MPS_E_NOMEM = -3,   /* slab or device pool exhausted */
  MPS_E_CUDA = -4,    /* CUDA runtime error (handle poisoned) */
  MPS_E_NCCL = -5,    /* reserved (never returned: the boundary exchange runs above this ABI) */
  MPS_E_NOCONV = -6,  /* Jacobi SVD did not converge within max_sweeps */
  MPS_E_NUMERIC = -7, /* non-finite singular value */
  MPS_E_STATE = -8,   /* more truncations than n_planned, or bad query state */
  MPS_E_TOOBIG = -9   /* query too large (statevector with d^N > 2^26) */
};
/* target-update strategies: PAPER.md:153 (Fig. 1 caption) and 158; FIXED = per-update target
 * f_fixed with no ledger feedback (the BASELINE config-2 microbench). */
enum { MPS_STRAT_NAIVE = 0, MPS_STRAT_NEAREST = 1, MPS_STRAT_GLOBAL = 2, MPS_STRAT_FIXED = 3 };
/* truncation fidelity rule: PURE = E10 read as 1 - T_k/P; WANG = E11 read as sqrt(1 - T_k/P)
 * (Wang fidelity E9 of rho vs the truncated rho); RATIO = 1 - T_k/P applied to an MPO. */
enum { MPS_RULE_PURE = 0, MPS_RULE_WANG = 1, MPS_RULE_RATIO = 2 };

typedef struct {
  double f_min;        /* (0, 1]; 1 = exact mode (E14 with F_min = 1) */
  int64_t n_planned;   /* number of two-qubit gates to be applied */
  int32_t strategy;    /* MPS_STRAT_* */
  int32_t rule;        /* MPS_RULE_* (MPO default: WANG) */
  int32_t chi_cap;     /* <= 0: no cap; else bond cap */
  int32_t max_sweeps;  /* Jacobi safety limit (<= 0: 60) -> MPS_E_NOCONV */
  double f_fixed;      /* per-update target for MPS_STRAT_FIXED */
  void* stream;        /* cudaStream_t; NULL = legacy default stream */
  void* dev_slab;      /* device memory owned by the caller */
  size_t slab_bytes;   /* the site-block sharding of SURVEY §8(e) runs ABOVE this ABI: one handle per
                        * rank holds that rank's block (paper_2307_16870_b200/sharded.py) */
} mps_config;

/* One row per truncation (SPEC.md:189-193 TruncationRecord). */
typedef struct {
  int64_t gate_index;  /* ledger index j (0-based, canonical order: layer-major, ascending site) */
  int32_t bond;        /* bond i = the gate's left site */
  int32_t chi_before;  /* chi_i before the gate */
  int32_t chi_after;   /* kept rank k */
  int32_t capped;      /* 1 if chi_cap forced a deeper cut */
  double target_f;     /* issued target t_j */
  double achieved_f;   /* f_j */
  double discarded_weight; /* T_k / P */
} mps_record;

/* |0...0> (MPO: rho = |0..0><0..0|), every bond extent 1. d in {2, 4}. */
mps_status mps_create(int32_t n_sites, int32_t d, const mps_config* cfg, mps_t* out);
mps_status mps_destroy(mps_t);

/* Single-site gate (d x d, row-major c64, host pointer), no truncation. */
mps_status mps_apply_gate1(mps_t, int32_t site, const float* U);
/* A layer of single-site gates on distinct sites (the one-qubit layers of the paper's random
 * circuits, "alternates randomly chosen layers of one- and two-qubit gates"; for d = 4
 * the 4 x 4 superoperator, e.g. (D (x) D)-free U (x) U* followed by a one-qubit channel): sites[g]
 * (host, int32, distinct, in [0, N)), Us (host, n_gates * d^2 c64 row-major). One launch for the
 * layer; no truncation (single-site gates do not change bond dimensions). Synchronous.
 * MPS_E_RANGE / MPS_E_INVAL (repeated site, non-finite entry). */
mps_status mps_apply_layer1(mps_t, int32_t n_gates, const int32_t* sites, const float* Us);
/* One two-site gate on (site, site+1): contract -> SVD -> fidelity-driven truncation ->
 * reabsorb. U host pointer, d^2 x d^2 c64 row-major. */
mps_status mps_apply_gate2(mps_t, int32_t site, const float* U);
/* All gates of one layer: sites[g] (host, int32), Us (host, n_gates * d^4 c64). Sites must be
 * disjoint pairs (|site_a - site_b| >= 2) and in [0, N-1). Truncations are ledgered in
 * ascending-site order (reading "canonical order"). Synchronises the stream at the end
 * of the layer (the new bond profile drives the next layer's bucketing). */
mps_status mps_apply_layer(mps_t, int32_t n_gates, const int32_t* sites, const float* Us);

/* The same layer in two halves, so that a caller can pass the ledger between calls (the
 * multi-rank token chain of SURVEY §8(e)): mps_layer_begin validates and
 * plans exactly like mps_apply_layer and issues the first wave's contract + SVD (steps a0-a3)
 * without waiting for them; *n_waves = 1 if work was issued (0 for an empty layer).
 * mps_layer_step runs the current wave's select + ledger + reabsorb (a4-a5, reading the ledger
 * as it stands on the device), synchronises, and issues the next wave's a0-a3 if any;
 * *remaining = gates not yet committed (0 = layer done). While a layer is in flight, imports,
 * set_lambda and snapshot_load return MPS_E_STATE. mps_apply_layer == begin + step until 0. */
mps_status mps_layer_begin(mps_t, int32_t n_gates, const int32_t* sites, const float* Us, int32_t* n_waves);
mps_status mps_layer_step(mps_t, int32_t* remaining);
/* Ledger token (E12 running product in log space, next truncation index j, guarantee flag).
 * get synchronises; set writes the device ledger (MPS_E_INVAL if log_E is not finite or > 0). */
mps_status mps_ledger_get(mps_t, double* log_E, int64_t* j, int32_t* guarantee);
mps_status mps_ledger_set(mps_t, double log_E, int64_t j, int32_t guarantee);

/* Planning introspection (host only; no handle, no device work): the SVD regime the layer planner
 * picks for an m x n theta (3 QR-preconditioned, 0 small, 2 medium, 1 tcgen05 large), the lane-group
 * size and rows per lane of its bucket (0 for the large regime / the generic path) and the padded
 * column count. MPS_E_INVAL for m, n < 1 or NULL outputs. */
mps_status mps_plan_regime(int32_t m, int32_t n, int32_t* regime, int32_t* gt, int32_t* rpl, int32_t* n_pad);

/* Running estimate (E12/E13): est = exp(log_est); n_done = truncations so far; guarantee_held =
 * no cap fired; is_lower_bound = 1 for the MPO (noisy) regime (E13). Any pointer may be NULL. */
mps_status mps_fidelity_estimate(mps_t, double* est, double* log_est, int64_t* n_done,
                                 int32_t* guarantee_held, int32_t* is_lower_bound);
/* <digits|psi> = the coefficient C_{sigma_1..sigma_N} of E1 evaluated from the MPS
 * product of E2 as a left-to-right chain of chi-vectors (MPO: the vectorised
 * element <<digits|rho>> of the density-matrix expansion); digits: N values in
 * [0, d). re_im: 2 doubles (host). Synchronising; MPS_E_RANGE for a digit >= d. */
mps_status mps_amplitude(mps_t, const uint8_t* digits, double* re_im);
/* The full coefficient vector C of E1, contracted from the MPS of E2
 * (PAPER.md:38-41): d^N interleaved complex128 values in `out` (host, n_doubles >= 2 d^N), site 0
 * the most significant digit; MPS_E_TOOBIG if d^N > 2^26 (small-N verification only). */
mps_status mps_to_statevector(mps_t, double* out, size_t n_doubles);
/* The bond dimensions chi_1 .. chi_{N-1} of E2 as they stand (host mirror, no
 * device work); out: N-1 int32 (host). */
mps_status mps_bond_dims(mps_t, int32_t* out /* N-1 */);
/* Exact canonicalisation (NEXT-1; PAPER.md:76 QR / RQ sweeps, :84 "enforced
 * throughout"): after truncations or non-unitary MPO maps the B-lambda form is canonical only
 * approximately (reading 4); two sequential sweeps of exact identity-gate two-site updates
 * (right to left, then left to right; the same kernels as mps_apply_layer) make every B_i, i >= 1,
 * right-orthonormal and every lambda the exact Schmidt values of its bond. No truncation beyond the
 * exact-mode floor (sigma > 1e-6 sigma_0), no ledger entry (log E, j, guarantee, records restored).
 * 2 (N - 1) sequential single-gate waves: an occasional operation ("every L layers"), not per layer.
 * Synchronous; device errors as for mps_apply_layer. */
mps_status mps_canonicalize(mps_t);
/* ---- observables (NEXT-4); synchronising, FP64 accumulation on the device ----
 * <a|b> = sum_sigma conj(C^a_sigma) C^b_sigma by left-to-right transfer matrices
 * E_{i+1} = sum_s A_i^{s dagger} E_i B_i^s (E2): the overlap behind the pure-state
 * fidelity E7 |<a|b>|^2; for d = 4 the Hilbert-Schmidt product Tr(rho_a^dagger
 * rho_b) of the vectorised density operators, from which the Wang fidelity E9
 * is |<<a|b>>| / sqrt(<<a|a>> <<b|b>>). Both handles on the same device, same N and d
 * (MPS_E_INVAL otherwise); re_im: 2 doubles (host). Scratch is taken from the top of a's slab
 * (MPS_E_NOMEM if the pool has grown into it). */
mps_status mps_overlap(mps_t a, mps_t b, double* re_im);
/* Tr rho = <<vec(I)|rho>> of a vectorised MPO (d = 4: per site the digits s = 2 sigma + sigma'
 * with sigma = sigma', s in {0, 3}); MPS_E_STATE for d = 2. re_im: 2 doubles (host). */
mps_status mps_trace(mps_t, double* re_im);
/* Two-site expectation value <psi|O_{site,site+1}|psi> / <psi|psi> (E5) in the
 * state's actual gauge (full left and right environments: exact also after truncations, when the
 * B-lambda form is no longer exactly canonical, reading 4). O: host, d^2 x d^2 row-major
 * interleaved complex64, O[(s d + t), (s' d + t')] with s the physical index of `site`. d = 2 only
 * (MPS_E_STATE for d = 4); MPS_E_RANGE for site outside [0, N-1); MPS_E_INVAL for a non-finite O. */
mps_status mps_expectation2(mps_t, int32_t site, const float* O, double* re_im);
/* Schmidt vector lambda of `bond` (float32, descending; bond -1..N-1, the outer two are [1]): the
 * kept, renormalised singular values of the last SVD at that bond ("singular values in decreasing
 * order"; the Lambda of the canonical form, PAPER.md:65 and E10 PAPER.md:117-118).
 * out may be NULL to query *len; MPS_E_RANGE for a bond outside -1..N-1. */
mps_status mps_schmidt_values(mps_t, int32_t bond, float* out, int32_t cap, int32_t* len);
mps_status mps_truncation_log(mps_t, mps_record* rows, int64_t cap, int64_t* len);
/* Sorted singular values (float64, descending, all n of them) of gate g (ascending-site order)
 * of the most recent layer -- the parity export for the SVD step. Readable for the gates of the
 * layer's final wave (a layer larger than the slab's workspace runs in waves); MPS_E_STATE for
 * earlier waves, whose workspace was reused. */
mps_status mps_last_spectrum(mps_t, int32_t g, double* out, int32_t cap, int32_t* len);
/* Parity switch for layers that run in several waves: with on != 0 every wave copies its gates'
 * sorted sigma^2 (the SVD step's output) to host memory before its workspace is
 * reused, and mps_last_spectrum then serves every gate of the last layer (one small D2H copy per
 * gate and wave: tests only, off by default). MPS_E_STATE inside a split layer. */
mps_status mps_keep_spectra(mps_t, int32_t on);
/* Site tensors for tests / checkpoints. dims3 = {chi_l, d, chi_r}. B: c64 row-major. The
 * pointer kind (host or device) is detected with cudaPointerGetAttributes. lam (float32, may be
 * NULL) = Schmidt vector of the bond right of `site`. Import resets the lambda of a bond whose
 * extent changed to ones. */
mps_status mps_export_site(mps_t, int32_t site, float* B, int32_t* dims3);
mps_status mps_import_site(mps_t, int32_t site, const float* B, const int32_t* dims3);
/* Bulk import of `count` consecutive sites starting at `first`: B holds the tensors back to back
 * (c64, row-major each; host -- pinned or pageable -- or device pointer), dims holds count x 3
 * extents (host). One H2D copy plus one device allocation/scatter launch pair. */
mps_status mps_import_sites(mps_t, int32_t first, int32_t count, const float* B, const int32_t* dims);
/* Bulk export, the reverse of mps_import_sites: the site tensors B_first .. B_{first+count-1} (the
 * B tensors of E1/E2; the B_i', B_{i+1}' an update writes) packed back
 * to back in site order (c64, row-major (chl, d, chr) each) into B -- host (pinned or pageable) or
 * device pointer, caller-owned, cap_elems complex elements -- by one device gather launch plus,
 * for a host B, one D2H copy. dims (host, count x 3) receives the extents and *elems_out (may be
 * NULL) the total complex elements; B == NULL only reports them. MPS_E_RANGE if cap_elems is too
 * small, MPS_E_STATE while a split layer is in flight. */
mps_status mps_export_sites(mps_t, int32_t first, int32_t count, float* B, size_t cap_elems, int32_t* dims,
                            size_t* elems_out);
mps_status mps_set_lambda(mps_t, int32_t bond /* -1..N-1 */, const float* lam, int32_t len);
/* Device-side snapshot of the whole state (site store, ledger, pool) into a caller device buffer
 * and back; *bytes_needed reports the size when buf == NULL. */
mps_status mps_snapshot_save(mps_t, void* dev_buf, size_t buf_bytes, size_t* bytes_needed);
mps_status mps_snapshot_load(mps_t, const void* dev_buf, size_t buf_bytes);
/* Kernel launches issued by this handle since creation (the bench's gpu_launches). */
mps_status mps_launch_count(mps_t, int64_t* count);
/* Jacobi sweeps of gate g of the last layer. */
mps_status mps_last_sweeps(mps_t, int32_t g, int32_t* sweeps);
/* Phase timers: with profiling on, apply_layer records CUDA events on cfg.stream around each
 * phase and accumulates device milliseconds: ms[0] contract, ms[1] SVD (small / medium / QR
 * regimes), ms[2] SVD (large regime), ms[3] select, ms[4] reabsorb (counts[p] = waves timed);
 * and sub-phases of the SVD (counts[p] = launch groups timed): ms[5] preconditioner (FP64 Gram +
 * Cholesky + B = L), ms[6] the Jacobi kernel, ms[7] spectrum (Rayleigh + polish + sort); the
 * eigen route (mps_set_svd_route): ms[8] its Householder tridiagonalisation kernel, ms[9] the rest
 * of it (FP64 theta and Gram, bisection, spectrum, eigenvectors after the select). A sub-phase is
 * timed for the regimes whose kernels are launched from the layer planner (the QR regime, the
 * eigen route and the fused large regime). mps_set_profiling resets the accumulators. */
mps_status mps_set_profiling(mps_t, int32_t on);
/* SVD route of the large regime (a2, "performing its SVD"; reading 20):
 * route 0 (default) takes large-regime theta with 128 < n <= 4096 through the FP64 Gram eigensolver (sigma^2 =
 * eigenvalues of theta^H theta, V for the kept columns by inverse iteration + back-transformation),
 * falling back to the Jacobi route for spectra deeper than 3e-6 sigma_max; route 1 takes every large
 * theta through the tcgen05 block Jacobi (+ the FP64 refinements). Applies from the next layer;
 * MPS_E_STATE inside a layer, MPS_E_INVAL for another route. */
mps_status mps_set_svd_route(mps_t, int32_t route);
mps_status mps_phase_times(mps_t, double* ms /* [10] */, int64_t* counts /* [10], may be NULL */);
mps_status mps_sync(mps_t);
const char* mps_last_error(mps_t);
const char* mps_status_string(mps_status);

#ifdef __cplusplus
}
#endif
#endif
