/* bsfem.h — C ABI of the B200 (sm_100a) quadratic B-spline cloth assembly library.
 *
 * Method: arXiv 2506.18867 "Efficient B-Spline Finite Elements for Cloth Simulation"
 * (/root/reference/PAPER.md, cited as PAPER.md:<line>).  The library evaluates, for one sheet (or
 * one row slab of a sheet),
 *     E(C)   = sum_q w_q Psi_FBW(F_q) + sum_q' w_q' 1/2 mu_bd |Lap phi_q'|^2       (PAPER.md:240-243,
 *                                                                                  264-275, 551-566)
 *     g      = dE/dC,      H = d^2E/dC^2  (optionally PSD-projected per FBW term, D7)
 * at the paper's reduced quadrature points (Fig. `fig: quadrature`,
 * PAPER.md:301-545) and assembles H into a 3x3-block sparse matrix whose pattern is fixed at
 * create time.
 *
 * Conventions (all calls):
 *  - Control point a = (i, j), 0 <= i < n_u, 0 <= j < n_v, has global index a = j*n_u + i.
 *  - Positions d_x: device, f64, row-major [rows][n_u][3] covering cp rows [x_row_begin, x_row_end)
 *    = [max(0,row_begin-2), min(n_v,row_end+2)) (the owned slab plus a 2-row halo; for a whole sheet
 *    simply [0, n_v)).  C^alpha in the paper's notation.
 *  - Gradient d_grad: device, f64 [row_end-row_begin][n_u][3] (owned rows only).
 *  - Hessian d_vals: device, f64 [nnzb][3][3], block b of block-row r (local row r = a - row_begin*n_u)
 *    holds d^2E / dC_{a,p} dC_{col_idx[b],q} at [b][p][q].  Full storage (both triangles), diagonal
 *    block always present, col_idx ascending within a row (global cp indices).
 *  - Energy d_energy: device, one f64: the sum over quadrature points whose lowest stencil row is
 *    owned (so the slabs of a partition sum to the sheet's energy).
 *  - Ownership: every d_* buffer belongs to the CALLER (e.g. torch tensors); the handle owns only
 *    its precomputed tables and scratch, released by bsf_destroy.
 *  - Asynchrony: compute calls validate arguments synchronously, enqueue kernels on `stream` and
 *    return without synchronising; asynchronous CUDA faults surface as BSF_E_CUDA on a later call.
 *    All compute calls are CUDA-graph capturable once the handle has run one call of the same batch
 *    size outside the capture (that call sizes the handle's scratch: energy partials, CTA lists).
 *  - Errors: every call returns bsf_status; bsf_last_error() gives a thread-local message.
 *  - Thread safety: one handle may be used by one host thread / stream at a time.
 */
#ifndef BSFEM_H
#define BSFEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bsf_sheet* bsf_handle;
typedef void* bsf_stream; /* a cudaStream_t (0 = legacy default stream) */

typedef enum {
  BSF_OK = 0,
  BSF_E_INVALID_ARG = -1,
  BSF_E_KNOTS = -2,             /* knots not open, uniform, integer        */
  BSF_E_TOO_SMALL = -3,         /* < 3 spans per direction with a REDUCED rule                   */
  BSF_E_DEGENERATE_GEOMETRY = -4, /* det J <= 0 at a quadrature point (rest map not regular)     */
  BSF_E_SINGULAR_STRETCH = -5,  /* |F e_beta| < 1e-12 at a membrane point (FBW undefined; SPEC.md:290
                                   clamps, this library reports): detected by the kernels, returned by
                                   the handle's next compute call or bsf_poll_status                 */
  BSF_E_CUDA = -6,
  BSF_E_OOM = -7,
  BSF_E_NCCL = -8,
  BSF_E_NO_DEVICE = -9
} bsf_status;

typedef enum {
  BSF_RULE_REDUCED = 0,       /* paper's rules: PAPER.md:290-293 (membrane), 571-573 (bending)   */
  BSF_RULE_G2_INTERIOR = 1,   /* ablation (A) of Fig. `fig:time_breakdown`:
                                 2x2 Gauss on interior spans, boundary frame as REDUCED           */
  BSF_RULE_G3_FULL = 2        /* 3x3 Gauss on every span, both energies                         */
} bsf_rule;

enum {
  BSF_PROJECT_PSD = 1,   /* per-term PSD projection of the FBW F-space Hessian (D7)  */
  BSF_NO_MEMBRANE = 2,   /* debug: drop the membrane terms                                       */
  BSF_NO_BENDING = 4,    /* debug: drop the bending terms                                        */
  BSF_GENERIC_PATH = 8,  /* force the generic point/gather kernels instead of the fused tile path; handles
                            with >= 2^23 points per rule (e.g. G3-FULL at 1024^2) do not build that path and
                            return BSF_E_INVALID_ARG for this flag */
  BSF_TILE_ONLY = 16,    /* debug: the tile kernel on the whole sheet, without the interior core kernel (and
                            not the G3-FULL kernel k_g3); falls back to the generic path where the tile
                            kernel does not fit */
  BSF_ASYNC_STAGE = 32   /* bsf_eval_all_batch_host only: the upload into d_x_stage waits only for the previous
                            host-buffer call on this handle that read the same d_x_stage (not for all work
                            queued on `stream`), so alternating two staging buffers overlaps one call's
                            upload with the previous call's assembly */
};

/* Stiffness symbols of Eq. `eq: FBW stretching and shearing energy` and
 * Eq. `eq: general bending energy`, per unit material area (Q9). */
typedef struct {
  double mu_st1, mu_st2, mu_sh, mu_bd;
} bsf_material;

/* Material map (D6; the paper's supplement is missing): mu_st1 = mu_st2 = E h / 2,
 * mu_sh = G h / 2 with G = shear_E if shear_E >= 0 else E / (2 (1 + nu)),
 * mu_bd = E_b h^3 / (12 (1 - nu^2)) with E_b = bend_E if bend_E >= 0 else E (pinned by the plate
 * formula PAPER.md:1149).  Errors: BSF_E_INVALID_ARG if E <= 0, h <= 0 or nu outside (-1, 0.5). */
bsf_status bsf_material_from_young(double E, double nu, double h, double shear_E, double bend_E,
                                   bsf_material* out);

/* Create a handle for one sheet / one owned row slab.
 *  n_u, n_v       control points per direction (>= 5 for REDUCED rules, i.e. >= 3 spans)
 *  knots_u/v      host, n_u+3 / n_v+3 doubles, must be (0,0,0,1,...,S-1,S,S,S)
 *  rest_xy        host, [n_v][n_u][2] material control points X^alpha, the
 *                 whole sheet even when a slab is owned
 *  mat            stiffness symbols (may be changed later with bsf_set_material)
 *  membrane_rule, bending_rule   quadrature rules (bsf_rule)
 *  row_begin, row_end            owned control-point rows [row_begin, row_end); 0, n_v for a sheet
 *  device         CUDA device ordinal the tables are uploaded to; -1 = host-only handle (sizes
 *                 and pattern queries only; compute calls return BSF_E_NO_DEVICE)
 *  out            receives the handle
 * The handle precomputes the quadrature points, the per-point basis / inverse-map coefficients
 * ("can be precomputed"), the BSR pattern (set union of structural stencils, DESIGN.md
 * Q10) and the gather tables, and uploads them.  Synchronous. */
bsf_status bsf_create(int n_u, int n_v, const double* knots_u, const double* knots_v,
                      const double* rest_xy, const bsf_material* mat, int membrane_rule,
                      int bending_rule, int row_begin, int row_end, int device, bsf_handle* out);

bsf_status bsf_destroy(bsf_handle h);

bsf_status bsf_set_material(bsf_handle h, const bsf_material* mat);

/* Sizes: number of owned block rows (= (row_end-row_begin)*n_u), nnzb, and the membrane /
 * bending quadrature points whose stencils touch the owned rows. Any pointer may be NULL. */
bsf_status bsf_get_sizes(bsf_handle h, int64_t* n_rows, int64_t* nnzb, int64_t* n_membrane,
                         int64_t* n_bending);

/* Copy the pattern (host buffers): row_ptr[n_rows+1] (int32, starts at 0), col_idx[nnzb]. */
bsf_status bsf_get_pattern(bsf_handle h, int32_t* row_ptr, int32_t* col_idx);

/* Batched fused pass over nbatch independent states of the same sheet (e.g. the states of many sheet
 * instances, or the line-search candidates of one Newton iteration; successive Newton iterates depend on
 * each other and are separate calls): item b reads d_x + b*x_stride and writes d_energy[b], d_grad + b*grad_stride,
 * d_vals + b*vals_stride (strides in doubles, >= one item's size).  One kernel launch covers all
 * items on the tile path.  Outputs may be NULL. */
bsf_status bsf_eval_all_batch(bsf_handle h, int nbatch, const double* d_x, int64_t x_stride,
                              double* d_energy, double* d_grad, int64_t grad_stride, double* d_vals,
                              int64_t vals_stride, int flags, bsf_stream stream);

/* Batch of DIFFERENT sheets that share the handle's grid size, rules and pattern, each with its own
 * affine rest map and stiffness (e.g. config C5: 64 flat sheets of side L_s and material E_s, nu_s).
 * d_params: device, [nbatch][9] doubles = G00 G01 G10 G11 (G = (dX/d(u,v))^-1 of the item's affine
 * rest map), det(dX/d(u,v)), mu_st1, mu_st2, mu_sh, mu_bd.  Requires an affine handle (flat
 * Greville sheet); BSF_E_INVALID_ARG otherwise.  Other arguments as bsf_eval_all_batch. */
bsf_status bsf_eval_all_batch_params(bsf_handle h, int nbatch, const double* d_x, int64_t x_stride,
                                     const double* d_params, double* d_energy, double* d_grad,
                                     int64_t grad_stride, double* d_vals, int64_t vals_stride, int flags,
                                     bsf_stream stream);

/* Step a2 of a flat affine sheet (J = dX/d(u,v), G = J^-1, w = what det J) for one item of
 * bsf_eval_all_batch_params: the rest map (rest_xy: host, [n_v][n_u][2]) is evaluated at the centre of every
 * knot span and must have one constant J (to 1e-11 of |J|) and vanishing second derivatives.
 * out9: host, G00 G01 G10 G11 det J mu_st1 mu_st2 mu_sh mu_bd.  Host call.  Errors: BSF_E_TOO_SMALL (< 3
 * control points per direction), BSF_E_DEGENERATE_GEOMETRY (det J <= 0), BSF_E_INVALID_ARG (not affine). */
bsf_status bsf_affine_params(int n_u, int n_v, const double* rest_xy, const bsf_material* mat, double* out9);

/* Host-buffer variant (end-to-end use): the positions of the nbatch states come from HOST memory h_x
 * (item b at h_x + b*x_stride; page-locked memory lets the upload overlap the computation) and are
 * uploaded into the caller's device buffer d_x_stage (same layout) in chunks of `chunk` items (0: batch/10,
 * then doubling each chunk)
 * on an internal copy stream, each chunk's assembly starting as soon as its positions have arrived.
 * By default the upload starts after all work already queued on `stream`; with BSF_ASYNC_STAGE in flags
 * it waits only for the last host-buffer call on this handle that read the same d_x_stage (the caller
 * must not use d_x_stage for anything else meanwhile), and chunk 0 means one chunk (the previous call's
 * assembly hides this call's upload).
 * d_params: optional per-item parameters (as bsf_eval_all_batch_params; device).  Energies go to d_energy
 * (device, nbatch doubles; required if h_energy is given) and, if h_energy is not NULL, are copied back to
 * the host buffer h_energy at the end of `stream` (valid after the stream synchronises).  Gradient and
 * Hessian outputs stay on the device as in bsf_eval_all_batch.  Asynchronous w.r.t. the host. */
bsf_status bsf_eval_all_batch_host(bsf_handle h, int nbatch, const double* h_x, int64_t x_stride, double* d_x_stage,
                                   const double* d_params, double* h_energy, double* d_energy, double* d_grad,
                                   int64_t grad_stride, double* d_vals, int64_t vals_stride, int flags, int chunk,
                                   bsf_stream stream);

/* ---- Incremental potential (Q13/Q14) ------------------------------------
 * E(x) = E_elastic(x) + sum_a m_a/(2 dt^2) |x_a - xhat_a|^2 - sum_a m_a g.x_a
 * with the lumped mass m_a = sum_b M_ab, M_ab = int R0 N_a N_b dX (3x3 Gauss per
 * knot span), the minimised objective of one implicit-Euler step; its Hessian adds m_a/dt^2 I3 to the
 * diagonal blocks.  Pinned control points are eliminated: gradient rows 0, Hessian rows and columns 0 and
 * the diagonal block I3 (the energy is unchanged).
 *
 * bsf_set_inertia: areal_density R0 (mass per rest area, >= 0), time step dt (> 0), gravity: host, 3 doubles
 * (NULL = none), pinned: host, [n_v][n_u] bytes over ALL rows (nonzero = pinned; NULL = none).  Computes the
 * lumped masses of the owned control points (host) and uploads them with the pinned lists; may be called
 * again to change any of them.  Works on a host-only handle (masses only).
 * bsf_get_lumped_mass: host m[owned rows][n_u] of the last bsf_set_inertia.
 * bsf_eval_ip_batch: as bsf_eval_all_batch plus the terms above; d_xhat: device, the predicted positions
 * x^ = x^n + dt v^n of the owned control points, [owned rows][n_u][3] per item, item stride xhat_stride
 * (doubles).  d_params: optional (device, as bsf_eval_all_batch_params, affine sheets): a batch of
 * different sheets of this grid; each item's masses are the handle's scaled by its det(dX/d(u,v)) over the
 * handle's (the same areal density).  BSF_E_INVALID_ARG before bsf_set_inertia. */
bsf_status bsf_set_inertia(bsf_handle h, double areal_density, double dt, const double* gravity,
                           const uint8_t* pinned);
bsf_status bsf_get_lumped_mass(bsf_handle h, double* m);
bsf_status bsf_eval_ip_batch(bsf_handle h, int nbatch, const double* d_x, int64_t x_stride, const double* d_xhat,
                             int64_t xhat_stride, const double* d_params, double* d_energy, double* d_grad,
                             int64_t grad_stride, double* d_vals, int64_t vals_stride, int flags,
                             bsf_stream stream);

/* ---- Linear algebra on the assembled Hessian (solve.cu) --------------------------------
 * The projected Newton step solves (H_inertia + H_elasticity) dC = -g; the paper
 * factorises (CHOLMOD), this library offers device block-Jacobi PCG on the BSR values it assembled.
 * bsf_bsr_spmv: d_y[owned rows][n_u][3] = H d_x, d_x in the position layout (owned rows plus the 2-row halo
 *   of a slab, like bsf_eval_all's d_x); d_vals: the handle's pattern.  Asynchronous.
 * bsf_gershgorin: host lo / hi with spec(H) within [lo, hi] (union of the scalar rows' Gershgorin discs,
 *   the bound PAPER.md:884-888 gates its Neumann split with).  Synchronises `stream`.
 * bsf_pcg: whole-sheet handles only; solves H x = b for SPD H (e.g. the PSD-projected Hessian plus inertia),
 *   d_b / d_x: device [n_v][n_u][3], d_x holds the initial guess on entry and the solution on return;
 *   stops at |b - Hx| <= rtol |b| or after max_iter iterations (check *relres); *iters, *relres: host (may
 *   be NULL).  BSF_E_INVALID_ARG if H is found not SPD.  Synchronises `stream` every 16 iterations. */
bsf_status bsf_bsr_spmv(bsf_handle h, const double* d_vals, const double* d_x, double* d_y, bsf_stream stream);

/* Direct solve (the paper factorises) and its Neumann split (Eq. `eq: Neumann
 * expansion`).  Whole-sheet handles only.  In control-point-major DOF order the Hessian is banded (half-bandwidth
 * 6 n_u + 5 DOFs for the reduced rules) and Cholesky keeps the band, so the factor is a device band matrix of
 * 3 n_v n_u x (half-bandwidth + 513) doubles (C2 128^2: 0.5 GB; C3 226^2: 2.3 GB); BSF_E_OOM if that exceeds
 * half the free device memory (e.g. C4).
 * bsf_chol_factor: factorises the SPD matrix D given by d_vals (the handle's pattern), e.g. the PSD-projected
 *   Hessian plus inertia, with cuSOLVER potrf / cuBLAS trsm + syrk panels (loaded at run time), and records the
 *   Gershgorin lower bound of D's spectrum.  Synchronises `stream`.  BSF_E_INVALID_ARG if D is not positive
 *   definite (names the pivot).
 * bsf_chol_solve: d_x = D^-1 d_b (device [n_v][n_u][3]; d_x may equal d_b).  Asynchronous.
 * bsf_neumann_solve: solves (D + B) x = b with the factorised D and B = d_vals_B (same pattern, symmetric) by the
 *   Neumann series x = sum_k (-D^-1 B)^k D^-1 b (as the fixed point x <- D^-1 (b - B x)), after the paper's gate:
 *   |D^-1 B| <= lambda_max(B) / lambda_min(D), both from Gershgorin discs; *gate (host) receives that bound and
 *   BSF_E_INVALID_ARG is returned if it is >= 1 (factorise D + B instead).  Stops when the step is <= rtol |x| or
 *   after max_terms terms (*terms, host, may be NULL).  Synchronises `stream` once per term. */
bsf_status bsf_chol_factor(bsf_handle h, const double* d_vals, bsf_stream stream);
bsf_status bsf_chol_solve(bsf_handle h, const double* d_b, double* d_x, bsf_stream stream);
bsf_status bsf_neumann_solve(bsf_handle h, const double* d_vals_B, const double* d_b, double* d_x, int max_terms,
                             double rtol, double* gate, int* terms, bsf_stream stream);

/* ---- Contact Hessian pullback to the control points (contact.cu) -------------------------
 * The contact mesh is embedded in the sheet: vertex alpha sits at a fixed parametric point (u_alpha, v_alpha)
 * and moves as x^alpha = sum_ij N_ij(u_alpha, v_alpha) C^ij (Eq. `eq: trig mesh node from
 * control points`), so a contact barrier's gradient and Hessian on the mesh pull back by the chain rule
 * (Eq. `eq: gradient and hessian of contact barrier`), assembled as in Alg. 1 (PAPER.md:
 * 792-846) in two levels: vertex-pair blocks, then control-point-pair blocks.  Contact detection and the
 * barrier itself are the caller's.  Whole-sheet device handles only; every output value is summed by one
 * thread in a fixed order (sorted keys, stable), so results are deterministic.
 * bsf_contact_mesh: uv: host [n_vert][2] parameters in [0, S_u] x [0, S_v] (the knot-span units of the sheet;
 *   on a knot line the right limit, as the energies).  Precomputes each vertex's 3x3 control-point window and
 *   weights.  BSF_E_INVALID_ARG if a vertex lies outside the domain.  Replaces the previous mesh.
 * bsf_contact_positions: d_xv[n_vert][3] = the vertices' positions for control points d_x [n_v][n_u][3]
 *   (device).  Asynchronous.
 * bsf_contact_assemble: n_pairs active pairs; d_verts: device int32 [n_pairs][4] mesh vertex indices (-1 = a slot
 *   without control-point DOFs, e.g. an obstacle vertex; index >= n_vert -> BSF_E_INVALID_ARG); d_H: device
 *   [n_pairs][12][12] the barrier Hessian of each pair w.r.t. its 4 vertex slots (row 3 s + r), d_g: device
 *   [n_pairs][12] its gradient, or NULL.  Outputs: d_grad (device [n_v][n_u][3], or NULL): += the pulled-back
 *   gradient; d_vals (device, the handle's BSR pattern, or NULL): its diagonal blocks += the pulled-back
 *   Hessian's diagonal blocks (the paper's H_barrier,d, merged into D); the off-diagonal blocks (H_barrier,od,
 *   the paper's B) stay in the handle as a BSR matrix of n_v n_u block rows in its own pattern, columns
 *   ascending, *nnzb_off (host, may be NULL) blocks.  Synchronises `stream` (the pattern's size is data
 *   dependent).
 * bsf_contact_get: copies that matrix out: d_row_ptr [n_v n_u + 1], d_col_idx [nnzb_off], d_vals [nnzb_off][9]
 *   (device; any may be NULL).  Asynchronous.
 * bsf_contact_neumann_solve: as bsf_neumann_solve with B = that off-diagonal contact matrix and D the matrix of
 *   the last bsf_chol_factor (e.g. inertia + elasticity + the merged contact diagonal). */
bsf_status bsf_contact_mesh(bsf_handle h, int n_vert, const double* uv);
bsf_status bsf_contact_positions(bsf_handle h, const double* d_x, double* d_xv, bsf_stream stream);
bsf_status bsf_contact_assemble(bsf_handle h, int n_pairs, const int32_t* d_verts, const double* d_H,
                                const double* d_g, double* d_grad, double* d_vals, int64_t* nnzb_off,
                                bsf_stream stream);
bsf_status bsf_contact_get(bsf_handle h, int32_t* d_row_ptr, int32_t* d_col_idx, double* d_vals, bsf_stream stream);
bsf_status bsf_contact_neumann_solve(bsf_handle h, const double* d_b, double* d_x, int max_terms, double rtol,
                                     double* gate, int* terms, bsf_stream stream);
bsf_status bsf_gershgorin(bsf_handle h, const double* d_vals, double* lo, double* hi, bsf_stream stream);
bsf_status bsf_pcg(bsf_handle h, const double* d_vals, const double* d_b, double* d_x, int max_iter, double rtol,
                   int* iters, double* relres, bsf_stream stream);

/* Energy only (the line-search call). d_energy: device, 1 double (overwritten).  Calls without
 * Hessian values (this one, bsf_eval_gradient, any call with d_vals = NULL) skip the per-point A entries, their
 * projection and the Hessian gather; energy-only calls also skip the gradient and run a point-parallel kernel
 * (C4: 0.04 ms energy, 0.21 ms gradient against 0.45 ms for all three).  Gradients are bit-identical to the full
 * call's; energies equal them to rounding (another summation order). */
bsf_status bsf_eval_energy(bsf_handle h, const double* d_x, double* d_energy, int flags,
                           bsf_stream stream);

/* Gradient only. d_grad overwritten. */
bsf_status bsf_eval_gradient(bsf_handle h, const double* d_x, double* d_grad, int flags,
                             bsf_stream stream);

/* Hessian values only, into the fixed pattern. d_vals overwritten. */
bsf_status bsf_assemble_hessian(bsf_handle h, const double* d_x, double* d_vals, int flags,
                                bsf_stream stream);

/* Fused hot path: energy, gradient and Hessian in one pass.  Any output may be NULL to skip it. */
bsf_status bsf_eval_all(bsf_handle h, const double* d_x, double* d_energy, double* d_grad,
                        double* d_vals, int flags, bsf_stream stream);

/* ---- Multi-GPU row slabs.  NCCL is loaded at run time
 * (libnccl.so.2 of the process, e.g. torch's); without it these calls return BSF_E_NCCL. */

/* Rank 0 creates a 128-byte NCCL unique id (host buffer) to broadcast to the other ranks. */
bsf_status bsf_nccl_get_unique_id(void* out128);

/* Create this rank's communicator (ranks = slabs in row order) on CUDA device `device`. */
bsf_status bsf_nccl_comm_init(int nranks, const void* id128, int rank, int device, void** comm);
bsf_status bsf_nccl_comm_destroy(void* comm);

/* The halo exchange plan of this slab as rank `rank` of `nranks` (row slabs in order): plan8[4 d + k] for
 * d = 0 (the peer below, rank-1) and d = 1 (the peer above, rank+1): k = 0 peer rank (-1: no exchange on that
 * side), 1 send offset, 2 receive offset, 3 count, all in doubles of the slab's position buffer d_x.  The
 * slab sends its first / last (<= 2) owned rows and receives the peer's into its halo rows.  bsf_halo_exchange
 * executes exactly this plan over NCCL; other transports (e.g. torch.distributed) can execute it too.  Host
 * call; works on host-only handles. */
bsf_status bsf_halo_plan(bsf_handle h, int rank, int nranks, int64_t* plan8);

/* Halo exchange: sends the 2 first / last owned rows to the previous / next slab and receives
 * theirs into d_x's halo rows (layout as above), as one NCCL group on `stream`.  Every slab must
 * own >= 2 rows.  No Hessian data is communicated (each slab recomputes the <= 2 rows of shared
 * quadrature points). */
bsf_status bsf_halo_exchange(bsf_handle h, double* d_x, void* nccl_comm, int rank, int nranks,
                             bsf_stream stream);

/* Halo exchange overlapped with the assembly (SURVEY §8(e) "Overlap"): the exchange runs on an internal
 * stream while the core kernel assembles the rows [r0+4, r1-4) that need no halo (a row's gather reads
 * control-point rows j-4 .. j+3); the remaining core rows, the bands and the corners wait for it.  Outputs
 * as bsf_eval_all (the slab's energy; sum it over ranks with bsf_allreduce_sum).  nranks == 1: no exchange
 * (nccl_comm may be NULL).  Falls back to exchange-then-assemble when the core path does not apply. */
bsf_status bsf_eval_all_slab(bsf_handle h, double* d_x, void* nccl_comm, int rank, int nranks, double* d_energy,
                             double* d_grad, double* d_vals, int flags, bsf_stream stream);

/* In-place sum all-reduce of n doubles (the slab energies) over the communicator. */
bsf_status bsf_allreduce_sum(double* d_buf, int64_t n, void* nccl_comm, bsf_stream stream);

/* Interior rectangle covered by the core kernel: rect4 = {i0, i1, j0, j1}, control
 * points [i0,i1) x [j0,j1) of the owned rows; all zero if the handle has no core region (non-affine
 * rest shape, non-REDUCED rules, small sheet, host-only handle).  Host call, no device work. */
bsf_status bsf_get_core_rect(bsf_handle h, int32_t* rect4);

/* Live per-kernel timing for the roofline of the dominant kernel (bench.py): with ncalls > 0 every
 * following call on the core + band path records CUDA events around the k_core launch (on the caller's
 * stream) and the k_band launch (on the side stream), in a ring of the last ncalls calls; ncalls = 0 turns
 * it off.  bsf_get_kernel_timing synchronises on those events and writes the durations in ms of the last
 * min(n, recorded) calls, oldest first (either pointer may be NULL); returns the count. */
bsf_status bsf_set_kernel_timing(bsf_handle h, int ncalls);
int bsf_get_kernel_timing(bsf_handle h, float* core_ms, float* band_ms, int n);

/* Number of kernel launches the most recent compute call enqueued (for the bench's claim). */
int bsf_last_launch_count(bsf_handle h);

/* BSF_E_SINGULAR_STRETCH (with bsf_last_error naming the quadrature point: its anchor knot span and batch
 * item) if a COMPLETED earlier call on this handle met |F e_beta| < 1e-12 at a membrane point whose energy
 * it owns, else BSF_OK.  The report is consumed (the next compute call would otherwise return it and
 * enqueue nothing).  Host read of mapped memory: no synchronisation, so synchronise the call's stream first
 * to be sure to see it. */
bsf_status bsf_poll_status(bsf_handle h);

/* Thread-local description of the most recent failure; never NULL. */
const char* bsf_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BSFEM_H */
