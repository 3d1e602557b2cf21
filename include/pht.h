/*
 * pht.h — C ABI of the B200-native polyhedral-homotopy hot path (arXiv 2111.14317).
 *
 * The library evaluates the polyhedral homotopy (Eq. (1))
 *
 *     h_k(x, t) = sum_{a in S_k} c_{k,a} x^a t^{omega_k(a)},    k = 1..n,
 *
 * together with dH/dx and dH/dt at large batches of points, in the logarithmic
 * formulation of §5 (z = log x, monomials = exp(z_hat A_hat), derivatives =
 * the same monomial row contracted against B_k, x-derivatives via diag(e^{-z})), and
 * computes the consolidated Euler + Newton directions of §6 by solving
 * Jx [dE | dN] = -[dH/dt | H] for both right-hand sides at once.  A fixed-protocol
 * Euler-Newton step runs entirely on the device.
 *
 * Conventions (all functions):
 *   - n = number of equations = number of variables (square systems).
 *   - complex values are interleaved (re, im) double pairs — the memory layout of
 *     torch.complex128 / numpy.complex128.  "c128[...]" below means 2*... doubles.
 *   - Batched arrays are row-major, point-major: x[p][n], H[p][n], Jx[p][n][n] with Jx[q][k][j]
 *     = dh_k/dx_j at point q (ledger R11 fixes the paper's vec() order).
 *   - All point/output pointers are DEVICE pointers on the system's device, owned by the
 *     caller; calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy default
 *     stream) and never synchronise the host (except the *_host variants).
 *   - A NULL output pointer skips that output.
 *   - Device arrays must be naturally aligned: complex (c128) arrays to 16 bytes (they are moved as
 *     16-byte vectors; torch/cudaMalloc allocations always are), double and int64 arrays to 8,
 *     int32 arrays to 4; otherwise PHT_EINVAL.
 *   - API misuse returns a negative pht_status synchronously; numerical conditions are
 *     reported per point in `status` (PHT_PT_* bits) and never abort the batch.
 *   - The handle is immutable after creation and may be used from several streams.
 */
#ifndef PHT_H
#define PHT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pht_system pht_system;

typedef enum {
    PHT_OK = 0,
    PHT_EINVAL = -1,       /* bad argument (NULL, negative size, non-finite data)        */
    PHT_ESHAPE = -2,       /* n_eq != n_var, n outside [1, PHT_MAX_N], bad offsets        */
    PHT_EDUPLICATE = -3,   /* duplicate (exponent vector, lifting) term in an equation */
    PHT_EEMPTY = -4,       /* an equation has no term with a nonzero coefficient   */
    PHT_ERANGE = -5,       /* |exponent| > PHT_MAX_EXP or lifting < 0                    */
    PHT_ECUDA = -6,        /* a CUDA runtime call failed (see pht_last_cuda_error)        */
    PHT_ENOMEM = -7,       /* device or host allocation failed                           */
    PHT_EUNSUPPORTED = -8, /* option not supported by this build                         */
    PHT_EJIT = -9          /* run-time compilation failed (NVRTC log: pht_last_cuda_error)  */
} pht_status;

/* per-point / per-path status bits */
enum {
    PHT_PT_OK = 0,
    PHT_PT_ZERO_COORD = 1,     /* a coordinate is 0: outside (C*)^n          */
    PHT_PT_NONFINITE = 2,      /* non-finite input or result                               */
    PHT_PT_SINGULAR = 4,       /* |pivot| <= 1e-14 * (row max) in the direction solve       */
    PHT_PT_STEP_UNDERFLOW = 8, /* tracker: step size fell below dtau_min                    */
    PHT_PT_MAX_STEPS = 16,     /* tracker: step budget exhausted                            */
    PHT_PT_DIVERGED = 32,      /* tracker: endpoint not refined or ||x||_inf > inf_norm      */
    PHT_PT_FLOOR = 64          /* tracker: finite endpoint whose final refinement reached only
                                  newton_tol, not final_tol, within final_iters (the accuracy
                                  floor of the log/exp evaluation, reading R30); the
                                  endpoint is returned, counted apart from PHT_PT_OK            */
};

#define PHT_MAX_N 24     /* largest n with a compiled kernel                              */
#define PHT_MAX_EXP 1024 /* largest |exponent| accepted                                    */

/*
 * Load a system (Alg. 1 "Initialize").  All inputs are HOST pointers, copied.
 *   n_eq, n_var   number of equations / variables; must be equal, 1..PHT_MAX_N.
 *   eq_offsets    int64[n_eq+1], eq_offsets[0] = 0, non-decreasing; the terms of equation k
 *                 are [eq_offsets[k], eq_offsets[k+1]) (per-equation supports S_k).
 *   exponents     int32[M][n_var], M = eq_offsets[n_eq]; Laurent exponents a (may be < 0).
 *   coeffs        c128[M] coefficients c_{k,a}.  Terms with c = 0 are dropped.
 *   lifting       double[M] liftings omega_k(a) >= 0 (real values allowed on the GPU).
 *   device        CUDA device ordinal that will own the tables and run every call.
 *   out           receives the handle on success.
 * Returns PHT_OK or a negative pht_status; *out is untouched on failure.
 */
int pht_system_create(int32_t n_eq, int32_t n_var, const int64_t *eq_offsets,
                      const int32_t *exponents, const double *coeffs, const double *lifting,
                      int32_t device, pht_system **out);

/*
 * Projective system: the same inputs as pht_system_create (the AFFINE system),
 * lifted into P^n as in Eq. (3): y in C^{n+1} with the homogenising coordinate LAST,
 * exponents a^ = (a, deg(f_k) - 1^T a), deg(f_k) = max 1^T a over S_k.  Every entry point then
 * works in homogeneous coordinates with n_var = n_eq + 1 columns (pht_system_info reports it):
 *   pht_evaluate        H (n+1 entries, the last 0), Jx = the bordered (n+1) x (n+1) matrix
 *                       [dH^/dy ; y^*] (last row: conjugated coordinates), Jt (last 0);
 *   pht_euler_newton    the projective Euler / Newton directions of P:237-252 / P:277-291
 *                       (bordered 2-RHS solve: dH^/dy E = -dH^/dtau ... with y^* E = 0);
 *   pht_pc_step         the Euler-Newton step in y with y renormalised to ||y|| = 1 after every
 *                       update (reading R29);
 *   pht_track           y state only (log_state / pht_track_cells: PHT_EUNSUPPORTED); norm-
 *                       relative corrector tests; an endpoint is finite iff |y_n| >= 1/inf_norm
 *                       (||y|| = 1), else PHT_PT_DIVERGED: a solution at infinity, which the
 *                       projective tracker reaches instead of losing the path.
 * Requires n_eq + 1 <= PHT_MAX_N.  No FP64 tensor-core evaluation path.
 */
int pht_system_create_projective(int32_t n_eq, int32_t n_var, const int64_t *eq_offsets,
                                 const int32_t *exponents, const double *coeffs, const double *lifting,
                                 int32_t device, pht_system **out);

/* Affine points of a projective system's n_eq variables onto P^n: y = (x, 1) / ||(x, 1)||
 * (homogenising coordinate last), x = e^z when log_input (z = log x, e.g. the endpoints of
 * pht_track_cells).  x: c128[p][n_eq] device, y: c128[p][n_eq + 1] device, async on stream.
 * PHT_EINVAL if sys is not projective. */
int pht_homogenize(const pht_system *sys, int64_t p, const double *x, int32_t log_input, double *y,
                   void *stream);

/* Free the device tables.  NULL is a no-op.  No call may be in flight on the handle. */
void pht_system_destroy(pht_system *sys);

/* Query: n, number of packed terms M, largest equation size, owning device. */
#define PHT_SYS_DENSE 1 /* the FP64 tensor-core (DMMA) evaluation tables exist: affine systems
                           with n >= 10, or after pht_system_set_kernels(PHT_KERNELS_DENSE) */
#define PHT_SYS_SPECIALIZED 2 /* system-specialised kernels loaded (pht_system_specialize) */
#define PHT_SYS_PROJECTIVE 4  /* created by pht_system_create_projective */
int pht_system_flags(const pht_system *sys); /* PHT_SYS_* bits, or a negative pht_status */

/*
 * System-specialised kernels: the one-time "Initialize" step of Alg. 1 extended to
 * write the system's rows (a2-a4) as straight-line CUDA with the exponents,
 * liftings and coefficients as literals, so that only the nonzero exponents are touched
 * (nnz(A)/M = 1.6-5 on the benchmark systems vs n for the table-driven kernels), compiled at
 * run time with NVRTC for sm_100a and loaded on the system's device.  Afterwards every entry
 * point selected by `what` runs the specialised kernels on this handle; results agree with the
 * generic kernels to rounding (same arithmetic per term, different summation order; rows keep
 * the row_exp2 convention with the exponent taken from the row's largest term).
 *   what   bit set of PHT_SPEC_* (0 = all): EVAL = pht_evaluate / pht_evaluate_log,
 *          STEP = pht_euler_newton / pht_pc_step, TRACK = pht_track / pht_track_cells.
 * Host-synchronous; compile time grows with the number of terms (about 4 s for the n = 10
 * benchmark systems; images are cached per process by generated source).  Calling it again with
 * a subset of the compiled kernels is a no-op.  The tracker uses the specialised kernel only
 * when the batch fills at least one wave of its (larger) tiles (pht_system_set_kernels(
 * PHT_KERNELS_SPECIALIZED) forces the specialised kernels on every entry point they implement).
 * Returns PHT_OK, PHT_EJIT (NVRTC failed: log in pht_last_cuda_error), PHT_ECUDA (load failed),
 * PHT_EUNSUPPORTED (the generated code would exceed sum_terms (nnz(a) + 8) > 8000 units, e.g.
 * random dense 20 x 50: minutes of compile time and instruction-cache bound; such systems keep
 * the generic and FP64 tensor-core kernels) or PHT_EINVAL.
 */
#define PHT_SPEC_EVAL 1
#define PHT_SPEC_STEP 2
#define PHT_SPEC_TRACK 4
#define PHT_SPEC_ALL 7
int pht_system_specialize(pht_system *sys, int32_t what);

/* Code-generator checks without a GPU (same inputs as pht_system_create, HOST pointers):
 * pht_specialize_compile generates and compiles the specialised kernels (no load) and stores
 * the cubin size; pht_specialize_source copies the generated CUDA source into buf (capacity
 * cap, NUL-terminated, truncated) and returns the full length + 1, or a negative pht_status. */
int pht_specialize_compile(int32_t n_eq, int32_t n_var, const int64_t *eq_offsets, const int32_t *exponents,
                           const double *coeffs, const double *lifting, int32_t what, int64_t *cubin_bytes);
int64_t pht_specialize_source(int32_t n_eq, int32_t n_var, const int64_t *eq_offsets,
                              const int32_t *exponents, const double *coeffs, const double *lifting,
                              char *buf, int64_t cap);

int pht_system_info(const pht_system *sys, int32_t *n, int64_t *M, int32_t *max_terms,
                    int32_t *device);

/*
 * Direction solver used by pht_euler_newton, pht_pc_step(_host), pht_track(_cells) on this
 * handle (a5; both solve G [dE | dN] = -[G_tau | h] in log coordinates):
 *   PHT_SOLVER_LU (default)  Gauss-Jordan with partial pivoting, one warp-lane per matrix row
 *                            (the consolidated 2-RHS elimination of BASELINE.json north_star).
 *   PHT_SOLVER_QR            the paper's own mechanism (Alg. 3):
 *                            Householder QR (no pivoting, backward stable), one lane per column,
 *                            the right-hand sides carried through Q^H, then back substitution.
 *                            Singular: |R_kk| <= 1e-14 ||G||_F (reading R26).  About twice the
 *                            cost of LU; a robustness path for ill-conditioned Jx.
 * Not synchronised with calls in flight on the handle.  Returns PHT_OK or PHT_EINVAL.
 */
#define PHT_SOLVER_LU 0
#define PHT_SOLVER_QR 1
int pht_system_set_solver(pht_system *sys, int32_t solver);

/*
 * Kernel family used by every entry point on this handle (explicit selection; results of all
 * families agree to rounding, tests/test_gpu_warp_kernels.py, tests/test_gpu_parity.py):
 *   PHT_KERNELS_AUTO (default)  the measured-best family per entry point and n:
 *        evaluation: specialised kernels if loaded, FP64 tensor cores for n >= 11 (and
 *        pht_evaluate_log from n = 10), else the warp-per-group kernel (n <= 12) or the tile
 *        kernel; directions / step / tracking: warp-per-group kernels (n <= 12, LU, affine, Euler
 *        predictor), the specialised kernels where those do not apply, else the tile kernels.
 *   PHT_KERNELS_TILE            tile kernels (k_phte, k_pht, k_track) for every entry point.
 *   PHT_KERNELS_WARP            warp-per-group kernels (k_stepw, k_trackw) wherever they apply,
 *                               AUTO elsewhere (same as AUTO without specialised kernels).
 *   PHT_KERNELS_DENSE           pht_evaluate / pht_evaluate_log on the FP64 tensor cores (builds the
 *                               tables on first selection; PHT_EUNSUPPORTED for projective
 *                               systems); AUTO for the other entry points.
 *   PHT_KERNELS_SPECIALIZED     the system-specialised kernels for every entry point they were
 *                               compiled for (PHT_EUNSUPPORTED before pht_system_specialize).
 *   PHT_KERNELS_LANE            pht_evaluate / pht_evaluate_log on the point-per-lane kernel (a warp
 *                               owns 32 points and walks the equations; rows leave through TMA
 *                               tensor stores), n <= 12; AUTO for the other entry points.
 * Host-synchronous (PHT_KERNELS_DENSE may upload tables); not synchronised with calls in flight.
 * Returns PHT_OK, PHT_EINVAL, PHT_EUNSUPPORTED, PHT_ENOMEM or PHT_ECUDA.  pht_system_kernels
 * returns the current family.
 */
#define PHT_KERNELS_AUTO 0
#define PHT_KERNELS_TILE 1
#define PHT_KERNELS_WARP 2
#define PHT_KERNELS_DENSE 3
#define PHT_KERNELS_SPECIALIZED 4
#define PHT_KERNELS_LANE 5
int pht_system_set_kernels(pht_system *sys, int32_t family);
int pht_system_kernels(const pht_system *sys);

/*
 * Batched evaluation of H, dH/dx, dH/dt (§5, Alg. 2).
 *   p         number of points (>= 0; 0 is a no-op).
 *   x         c128[p][n] points in (C*)^n.
 *   t         double[p], t in (0, 1] (real homotopy parameter, ledger R2/R16; any t > 0 works).
 *   H         c128[p][n]        h_k
 *   Jx        c128[p][n][n]     dh_k/dx_j
 *   Jt        c128[p][n]        dh_k/dt
 *   row_exp2  int32[p][n] or NULL.  NULL: outputs are plain IEEE values (may overflow).
 *             Non-NULL: every output of row k of point q is scaled by 2^-row_exp2[q][k]
 *             (true row = returned row * 2^row_exp2, ledger R7); no overflow occurs.
 *   status    uint8[p] PHT_PT_* bits, or NULL.
 */
int pht_evaluate(const pht_system *sys, int64_t p, const double *x, const double *t,
                 double *H, double *Jx, double *Jt, int32_t *row_exp2, uint8_t *status,
                 void *stream);

/*
 * The same in logarithmic coordinates: input z = log x (any branch;
 * Im z is wrapped to (-pi, pi]) and tau = log t; outputs H, Jz = dH/dz = Jx diag(x),
 * Jtau = dH/dtau = t dH/dt.  Range-safe with row_exp2 for |Re z| far beyond double range.
 */
int pht_evaluate_log(const pht_system *sys, int64_t p, const double *z, const double *tau,
                     double *H, double *Jz, double *Jtau, int32_t *row_exp2, uint8_t *status,
                     void *stream);

/*
 * Consolidated Euler + Newton directions (§6, affine form P:219-276):
 *   Jx dE = -dH/dt   (dE = dx/dt, Davidenko)       Jx dN = -H   (Newton)
 * computed from ONE elimination with two right-hand sides (partial pivoting).
 *   x c128[p][n], t double[p] inputs; dE, dN c128[p][n] outputs; status as above
 *   (PHT_PT_SINGULAR when a pivot is tiny; outputs of that point are then unspecified).
 */
int pht_euler_newton(const pht_system *sys, int64_t p, const double *x, const double *t,
                     double *dE, double *dN, uint8_t *status, void *stream);

/*
 * The paper's simplified Euler-Newton step in tau = log t (Eq. (2)):
 *   x~ = x + dtau * dx/dtau (Euler prediction),  tau~ = tau + dtau,
 *   then newton_iters times:  x~ = x~ + dN(x~, tau~).
 *   x         c128[p][n] in/out.
 *   tau       double[p] in/out.
 *   dtau      double[p] step sizes (tau + dtau should be <= 0).
 *   newton_iters  K >= 0 Newton iterations (the paper's protocol uses 1).
 *   status    uint8[p] or NULL (bits OR-ed over the step's solves).
 *   dn_norm   double[p] or NULL: ||dN||_2 of the last Newton iteration.
 */
int pht_pc_step(const pht_system *sys, int64_t p, double *x, double *tau, const double *dtau,
                int32_t newton_iters, uint8_t *status, double *dn_norm, void *stream);

/*
 * pht_pc_step on HOST buffers (end-to-end entry point): copies x, tau, dtau to a device
 * workspace owned by the handle, runs the step, copies x, tau, status, dn_norm back and
 * synchronises.  Pipelined (P:807-824 batch pipelining): the points are cut into chunks that
 * run copy-in -> step -> copy-out on three internal streams ordered after `stream`, so copies in
 * both directions overlap the kernels (requires pinned host memory; pageable memory works but
 * does not overlap).  Results are identical to pht_pc_step.  Serialised per handle.
 */
int pht_pc_step_host(const pht_system *sys, int64_t p, double *x, double *tau,
                     const double *dtau, int32_t newton_iters, uint8_t *status,
                     double *dn_norm, void *stream);

/*
 * pht_pc_step_host without the final synchronisation: returns once the pipeline is enqueued.
 * The host buffers x, tau, dtau, status, dn_norm belong to the copy engines until
 * pht_host_wait(sys, stream) returns (do not read or write them before).  Consecutive calls on one
 * handle chain through the handle's internal streams: chunk c of a call starts copying in as soon
 * as the previous call's chunk c has been copied out (same p; in-place x, tau), so one batch's
 * copy-in overlaps the previous batch's kernels and copy-out instead of the whole pipeline
 * filling and draining per call.  Orders itself after the work already submitted to `stream`.
 * Results are identical to pht_pc_step_host.  Errors as pht_pc_step_host.  pht_system_destroy
 * waits for host steps still in flight.
 */
int pht_pc_step_host_async(const pht_system *sys, int64_t p, double *x, double *tau,
                           const double *dtau, int32_t newton_iters, uint8_t *status,
                           double *dn_norm, void *stream);

/* Orders `stream` after every host step of this handle submitted so far and synchronises it
 * (the end of pht_pc_step_host_async chains).  PHT_OK when there was none. */
int pht_host_wait(const pht_system *sys, void *stream);

/*
 * Adaptive path tracking tau0 -> 0 on the device (step control = DESIGN.md
 * reading R14, the same algorithm as the oracle's tracker).  One persistent kernel: each slot
 * of each CTA runs one path (Euler predictor from dx/dtau, up to newton_iters Newton
 * corrections, accept -> grow dtau by `grow` after `grow_after` successes, reject -> shrink),
 * lands exactly on tau = 0, then refines with up to final_iters Newton steps at t = 1;
 * finished slots take the next path from an atomic queue.
 *   x       c128[p][n] start points in (on their paths at tau), endpoints out (z = log x
 *           instead of x when opts->log_state).
 *   tau     double[p] start parameters tau0 <= 0 in; final tau (0 when tracked) out.
 *   opts    options; NULL = defaults (pht_track_opts_default).
 *   stats   int64[p][4] or NULL: accepted steps, rejected steps, evaluations (each one
 *           evaluate + 2-RHS solve), final Newton iterations.
 *   status  uint8[p]: PHT_PT_OK = finite endpoint refined to final_tol; PHT_PT_FLOOR = finite
 *           endpoint refined only to newton_tol (accuracy floor, counted apart); PHT_PT_SINGULAR,
 *           PHT_PT_STEP_UNDERFLOW, PHT_PT_MAX_STEPS, PHT_PT_DIVERGED (refinement failed or
 *           ||x||_inf > inf_norm), PHT_PT_NONFINITE (non-finite tau0).
 * PHT_EINVAL for non-positive step sizes, shrink outside (0, 1), grow < 1, newton_iters,
 * grow_after, max_steps or final_iters < 1.
 * Asynchronous on `stream`; uses a stream-ordered 8-byte device counter.
 */
typedef struct {
    double dtau_init;   /* 0.05   initial step in tau                                   */
    double dtau_min;    /* 1e-12  step underflow threshold (events sit at |tau| ~ 1/omega)  */
    double dtau_max;    /* 0.5                                                           */
    double newton_tol;  /* 1e-10  corrector: max_j |dN_j|/|x_j| <= newton_tol             */
    double shrink;      /* 0.5                                                           */
    double grow;        /* 2.0                                                           */
    double final_tol;   /* 1e-13  final refinement: max_j |dN_j|/|x_j| <= final_tol       */
    double inf_norm;    /* 1e8    endpoints with ||x||_inf above this are DIVERGED         */
    int32_t newton_iters; /* 4    max corrector iterations per step (K)                  */
    int32_t grow_after;   /* 3                                                           */
    int32_t max_steps;    /* 10000                                                       */
    int32_t final_iters;  /* 5    (>= 1)                                                  */
    int32_t log_state;    /* 0: x holds points x; 1: x holds z = log x (any branch) — for start
                             points far outside double range (|Re z| > ~700); the steps are the
                             same affine updates, applied as z <- z + log(1 + dx/x)            */
    int32_t pred_log;     /* Euler predictor chart: 0 affine x + h dx/dtau (the paper's form,
                             P:254-259); 1 log chart z + h dz/dtau (exact for the toric paths
                             x ~ e^{tau alpha} y near tau0); -1 (default) = log_state          */
    double pred_tol;      /* 0      step-size control (reading R14): > 0: after an accepted step the
                             next step is dtau * clamp(sqrt(pred_tol / e1), shrink, grow), e1 =
                             size of the first corrector update (the Euler predictor's error,
                             O(dtau^2)); <= 0 (default): grow by `grow` after `grow_after`
                             successes (measured faster on the benchmark systems).
                             A corrector iterate is accepted when its update, or the update
                             times the observed contraction (quadratic convergence estimate),
                             is <= newton_tol.                                               */
    int32_t predictor;    /* 0 (default) Euler (the paper's protocol); 1 cubic Hermite
                             extrapolation in the log chart through the previous and the current
                             accepted point and their Euler directions (log chart
                             only, i.e. pred_log = 1: Euler otherwise)                        */
    int32_t reuse_tangent; /* 0 (default); 1: the consolidated solve of the last corrector iteration
                             also yields the Euler direction at that iterate; it
                             serves as the next step's predictor direction, one evaluation fewer
                             per accepted step (first-order different from the tangent at the
                             accepted point; Euler predictor, affine systems)                    */
} pht_track_opts;

void pht_track_opts_default(pht_track_opts *opts);

int pht_track(const pht_system *sys, int64_t p, double *x, double *tau, const pht_track_opts *opts,
              int64_t *stats, uint8_t *status, void *stream);

/*
 * Tracking in cell coordinates ("rescaled" polyhedral homotopy).  For a start path of the mixed
 * cell with inner normal (alpha, 1) and lower values beta_k, the substitution x = e^{tau alpha} e^w
 * and row scaling by e^{-tau beta_k} turn Eq. (2) into the polyhedral homotopy
 *     h'_k(w, tau) = sum_i c_i e^{<a_i, w>} e^{tau omega'_i},  omega'_i = omega_i + <a_i, alpha> - beta_k,
 * whose start values w = log y are O(1) and which equals F(e^w) at tau = 0 (so w = log x there).
 * It is the same path, with no cancellation between huge <a, log x> and omega tau.
 *   w          c128[p][n] start values w0 = log y (log state; opts->log_state is implied), out: z = log x.
 *   tau        double[p] tau0 in, 0 out.
 *   cell_lift  DEVICE double[ncells][M] shifted liftings omega' of every term (M = packed term count
 *              = input term count; systems with zero coefficients are rejected, PHT_EINVAL).
 *   path_cell  DEVICE int32[p] cell of each path (out-of-range ids give status PHT_PT_NONFINITE).
 * Other arguments as pht_track.
 */
int pht_track_cells(const pht_system *sys, int64_t p, double *w, double *tau, const double *cell_lift,
                    int64_t ncells, const int32_t *path_cell, const pht_track_opts *opts,
                    int64_t *stats, uint8_t *status, void *stream);

/* Number of kernels this library has launched in the calling process (all handles). */
int64_t pht_launch_count(void);

/* Human-readable text for a pht_status; last CUDA error string for PHT_ECUDA. */
const char *pht_strerror(int code);
const char *pht_last_cuda_error(void);

/* ABI version (incremented on any signature change). */
int pht_version(void); /* 4: pht_pc_step_host_async, pht_host_wait; 3: pht_track_opts.reuse_tangent; 2: pht_system_set_kernels, PHT_PT_FLOOR */

#ifdef __cplusplus
}
#endif

#endif /* PHT_H */
