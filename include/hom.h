/*
 * hom.h -- C-ABI of libhom.so, the B200 (sm_100a) hot path of the monolithic
 * FE^2 homogenization of Hesch, Schmidt & Schuss, arXiv 2312.12771.
 *
 * The path: a batch of independent RVE problems, one per macro
 * Gauss point (Dirac macro basis), whose fluctuation DOFs
 * are removed by static condensation -- the paper's null-space reduction
 * P = [I, -D L^-1]^T -- followed by the condensed macro solve
 * [K - D L^-1 E] dq = -[R_macro - D L^-1 R_micro] (eq:solution2)
 * and the fluctuation update dw = -L^-1 [R_micro + E dq].
 *
 * Conventions used by every call:
 *  - All floating point is IEEE binary64 (FP64).
 *  - Host pointers (setup inputs) are copied during hom_setup; the caller may
 *    free them when it returns.  Device pointers (d_*) are caller-owned,
 *    contiguous, 8-byte aligned, on the context's device; the library never
 *    frees them.  The context owns all scratch (K_ff chunk pool, influence
 *    store X, CSR matrix, CG vectors, fluctuation state).
 *  - Every call enqueues on `stream` (a cudaStream_t, NULL = legacy default)
 *    and returns after enqueue, except where a call is documented to
 *    synchronise (error flags, solver info).
 *  - B = number of RVEs = n_macro_elems * 2^dim, RVE b = e * 2^dim + q,
 *    Gauss points 2 per direction at +-1/sqrt(3), qp order x fastest.
 *  - m = 3 (2-D Voigt [e11, e22, g12]), 6 (3-D Voigt [e11, e22, e33, g23,
 *    g13, g12], engineering shear), 4 (2-D finite strain, F row-major
 *    [F11, F12, F21, F22]).
 *  - RVE fluctuation layout [B][N_pad]: N_pad = dim * n_indep, entry
 *    dim*p + c for periodic independent node p (nodes of the RVE mesh with no
 *    coordinate on an upper face, numbered in RVE-node order) and component
 *    c; the corner class (independent node of the lowest corner) is fixed
 *     and its entries are 0.
 *  - Return value: HOM_OK or a hom_status code; details via hom_last_error.
 *    No call aborts or throws.  One context per host thread.
 */
#ifndef HOM_H
#define HOM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hom_ctx hom_ctx; /* opaque */

typedef enum {
  HOM_OK = 0,
  HOM_ERR_INVALID_ARG = 1,     /* bad sizes, NULL where required, unsupported element */
  HOM_ERR_MESH = 2,            /* unmatched periodic faces, det J <= 0, no lower corner */
  HOM_ERR_NOT_SPD = 3,         /* Cholesky pivot <= 0 in an RVE (hom_error_info.rve, .row) */
  HOM_ERR_JACOBIAN = 4,        /* micro J <= 0 at a quadrature point (finite strain) */
  HOM_ERR_CG_NOT_CONVERGED = 5,/* macro CG hit max_iter before rtol */
  HOM_ERR_CG_BREAKDOWN = 6,    /* p^T K p <= 0 in the macro CG */
  HOM_ERR_CUDA = 7,            /* a CUDA runtime error (hom_error_info.cuda_error) */
  HOM_ERR_OOM = 8              /* device allocation failed */
} hom_status;

/* Macro mesh.  Q1 (4 nodes, counter-clockwise) in 2-D,
 * hex8 (bottom face CCW, then top face) in 3-D.  Dirichlet DOFs are
 * dof = node*dim + comp with prescribed values (Gamma^phi); body_force
 * is a constant body load per unit reference volume (eq:weakMech). */
typedef struct {
  int32_t dim;              /* 2 or 3 */
  int32_t n_nodes;
  int32_t n_elems;
  int32_t nodes_per_elem;   /* 4 (2-D) or 8 (3-D) */
  const double* coords;     /* host [n_nodes][dim] */
  const int32_t* conn;      /* host [n_elems][nodes_per_elem] */
  int32_t n_dirichlet;
  const int32_t* dirichlet_dof;   /* host [n_dirichlet] */
  const double* dirichlet_value;  /* host [n_dirichlet] (total prescribed value) */
  const double* body_force;       /* host [dim] or NULL */
  const double* nodal_force;      /* host [n_nodes*dim] or NULL: external nodal forces, e.g. the
                                     consistent nodal loads of a surface traction on Gamma^sigma */
} hom_macro_mesh;

/* RVE mesh: an axis-aligned box meshed with Q1/hex8 elements whose opposite
 * faces carry matching nodes; the periodic pairing (eq:Con (iii)) is
 * found in hom_setup by coordinate matching.  Any such mesh (graded, distorted interior) is
 * accepted.  Small strain: elements are grouped into geometry types (element matrices equal to
 * 1e-13 relative; a uniform grid has one); when the per-(type, phase) matrices fit K1's 96 KB
 * shared-memory tables (e.g. <= 69 types x 2 phases in 2-D, <= 8 in 3-D) K1 reads them from
 * shared memory, otherwise it combines the geometry tables (global memory, L2) with the element's
 * (lambda, mu) on the fly. */
typedef struct {
  int32_t dim;
  int32_t n_nodes;
  int32_t n_elems;
  int32_t nodes_per_elem;
  const double* coords;     /* host [n_nodes][dim] */
  const int32_t* conn;      /* host [n_elems][nodes_per_elem] */
} hom_rve_mesh;

/* Phase id per RVE element; per_rve = 1: [B][n_rve_elems], 0: [n_rve_elems] shared. */
typedef struct {
  int32_t per_rve;
  const uint8_t* phase;     /* host */
} hom_phase_field;

/* Materials per phase.  kind 0: linear isotropic (E, nu), plane strain in 2-D.
 * kind 1: the paper's Cook energy with beta = 0 (R11),
 *   Psi = alpha (F:F - 2) + kappa/2 (J - 1)^2 - 2 alpha ln J, params (alpha, kappa), 2-D only.
 * kind 2: the paper's Cook energy,
 *   Psi = alpha (F:F - 2) + beta (F:F + J^2 - 3) + kappa/2 (J - 1)^2 - 2 (alpha + 2 beta) ln J,
 *   params (alpha, beta, kappa) [n_phases][3], 2-D only. */
typedef struct {
  int32_t kind;
  int32_t n_phases;
  int32_t per_rve;          /* 1: [B][n_phases][2], 0: [n_phases][2] */
  const double* params;     /* host [B|1][n_phases][2] (kind 0, 1) or [..][3] (kind 2) */
} hom_materials;

typedef struct {
  int32_t finite_strain;    /* must equal (materials.kind >= 1) */
  double cg_rtol;           /* relative residual ||r||/||b|| (default 1e-13 if <= 0) */
  int32_t cg_max_iter;      /* default 20000 if <= 0 */
  int32_t rve_chunk;        /* RVEs condensed per pass; <= 0: automatic (memory budget) */
  int32_t check_info;       /* 1: hom_condense synchronises once to report NOT_SPD / JACOBIAN */
  double mem_budget_gb;     /* K_ff pool budget for automatic chunking; <= 0: 96 GB (chunks are then a whole
                               number of condensation waves, as few launches as the budget allows) */
  int32_t tile_sparse;      /* 0: dense blocked factorisation of every lower 64x64 tile of K_ff
                               (BASELINE north_star).  1: tile-sparse -- only the tiles of the
                               symbolic tile-level fill of K_ff's structural pattern are stored
                               and factored; identical arithmetic on those tiles,
                               the skipped products are exact zeros. */
  int32_t rve_begin;        /* RVE sharding (multi-GPU): this context condenses and */
  int32_t rve_count;        /* recovers RVEs [rve_begin, rve_begin + rve_count) only (rve_count <= 0:
                               all B).  C_eff / P_eff / w rows of the other RVEs are left untouched,
                               so the caller all-gathers C_eff (and P_eff) before hom_macro_solve,
                               which always solves the full macro problem. */
  int32_t macro_basis;      /* macro interpolation of the fluctuations:
                               0 = Dirac pulses at the macro Gauss points (one RVE per qp, B = 2^dim
                               n_elems, classical FE^2); 1 = piecewise constant per macro element
                               (eq:constSolution1/2, one RVE per element, B = n_elems; small strain
                               only).  With 1, the RVE index is the element, hom_condense also keeps
                               <C> per element, the macro stiffness is
                               K_e = sum_q eta B_q^T <C>_e B_q - |B_e| Bbar^T (<C>_e - C_eff,e) Bbar
                               (Bbar = element-average strain operator) and kinematics / recovery use
                               the element-average strain. */
  int32_t rve_ordering;     /* internal order of the RVE's independent nodes (the rows of K_ff):
                               0 = folded (default): along every axis the periodic images are
                               interleaved 0, r-1, 1, r-2, ... (slowest axis first), so wrap-around
                               neighbours are adjacent and K_ff is banded without a periodic frame
                               (fewer fill tiles for tile_sparse); 1 = natural
                               (first appearance in the mesh).  The layout of w at the API (d_w of
                               hom_recover_fluctuations / hom_set_fluctuations / hom_get_fluctuations)
                               is always the natural one. */
  int32_t macro_precond;    /* preconditioner of the macro PCG (a6): 2 = two-level: node-block Jacobi + an
                               additive coarse space of node aggregates with their rigid-body modes,
                               A_c = P^T K_M P formed and inverted on the device every solve (DESIGN.md
                               §5.4.1; meshes with >= 1024 DOFs in 2-D / 3-D, otherwise Jacobi);
                               1 = node-block Jacobi only; 0 = auto (default): two-level when fewer than
                               a quarter of the macro DOFs are prescribed (few Dirichlet anchors: the slow
                               low-frequency modes the coarse space removes), else Jacobi -- measured:
                               config 2 (3 % prescribed) 0.69 vs 0.98 ms, config 4 (53 % prescribed) 0.48
                               vs 0.86 ms.  The solution is the same (rtol), only the iteration count and
                               the time differ. */
} hom_options;

typedef struct {
  int32_t n_rve;            /* B */
  int32_t m;                /* tangent size */
  int32_t n_pad;            /* fluctuation entries per RVE */
  int32_t n_tiles;          /* 64x64 tiles per K_ff dimension */
  int32_t n_macro_dof;
  int32_t n_macro_free;
  int32_t macro_nnz;        /* scalar CSR entries of the macro stiffness */
  int32_t rve_chunk;
  double rve_volume;        /* |Omega| */
  int32_t rve_begin;        /* local RVE range of this context (options.rve_begin / rve_count) */
  int32_t rve_count;
} hom_sizes;

/* Work per RVE of the condensation, from the tile structure (hom_get_work).  Tile counts
 * are per RVE; a "product" is one 64x64x64 tile GEMM. */
typedef struct {
  int32_t a_tiles;          /* structurally nonzero lower tiles of K_ff (assembled by K1) */
  int32_t g_tiles;          /* lower tiles processed / stored for G (all lower tiles if dense) */
  int32_t diag_tiles;       /* diagonal tiles (factor + inverse each) */
  int32_t syrk_tiles;       /* diagonal-update products G_JK G_JK^T */
  int32_t gemm_tiles;       /* off-diagonal update products G_IK G_JK^T */
  int32_t trsm_tiles;       /* off-diagonal tiles G_IJ = S_IJ G_JJ^-T */
  double flop_dense;        /* algorithmic dense count n^3/3 + 2 n^2 m + n m^2 (n = n_f) */
  double flop_executed;     /* DMMA flops k_condense executes for this tile structure */
} hom_work;
typedef struct {
  int32_t iterations;
  double rel_residual;      /* ||r|| / ||b|| at exit */
  double rhs_norm;          /* ||b|| */
} hom_solve_info;

typedef struct {
  int32_t code;
  int32_t rve;              /* offending RVE or -1 */
  int32_t row;              /* NOT_SPD: the fluctuation DOF (natural [N_pad] layout) whose pivot
                               failed in the factorisation order; JACOBIAN: micro qp; or -1 */
  int32_t cuda_error;
  char message[256];
} hom_error_info;

/* Build a context: validates the meshes, finds the periodic pairing and the
 * fixed corner, precomputes shape-gradient tables and the macro CSR pattern,
 * copies phases and materials to the device and allocates all scratch.
 * Synchronises `stream` before returning. */
int hom_setup(hom_ctx** out, const hom_macro_mesh* macro, const hom_rve_mesh* rve,
              const hom_phase_field* phases, const hom_materials* materials,
              const hom_options* options, void* stream);

int hom_get_sizes(const hom_ctx* ctx, hom_sizes* out);
int hom_get_work(const hom_ctx* ctx, hom_work* out);

/* Macro kinematics at every macro qp: d_u [n_macro_dof] -> d_kin [B][m]:
 * Voigt strain eps = B u (small strain) or F = I + grad u (finite strain). */
int hom_macro_kinematics(hom_ctx* ctx, const double* d_u, double* d_kin, void* stream);

/* Condense every RVE (eq:solution1/2): assemble K_ff, K_fe (, r_f) (eq:discreteSys_D/L,
 * P:348-358), factor K_ff = G G^T, Y = G^-1 [K_fe | r_f], X = G^-T Y (stored in the
 * context for recovery) and
 *   d_C_eff [B][m][m] = <C> - Y^T Y / |Omega|     (row-major),
 *   d_P_eff [B][m]    = <P> - K_Ff K_ff^-1 r_f / |Omega|   (finite strain; NULL otherwise),
 *   d_P_avg [B][m]    = <P>                                 (finite strain; nullable).
 * Small strain: d_kin is ignored (may be NULL).  Finite strain: d_kin = F per RVE [B][4];
 * the current fluctuation state (hom_set_fluctuations / hom_recover_fluctuations) is used.
 * With options.check_info the call synchronises once and returns HOM_ERR_NOT_SPD or
 * HOM_ERR_JACOBIAN for the first failing RVE. */
int hom_condense(hom_ctx* ctx, const double* d_kin, double* d_C_eff, double* d_P_eff,
                 double* d_P_avg, void* stream);

/* Solve the condensed macro system by CG on the free DOFs, preconditioned by the inverses of the
 * dim x dim diagonal node blocks (Dirichlet components removed; one thread-block cluster holds the
 * whole solve for meshes up to ~17k DOFs in 2-D, grid-wide kernels beyond; deterministic sums):
 *   K_FF x_F = -R_F - K_FD x_D,   K = sum_qp eta B^T D_b B,  R = sum_qp eta B^T S_b - f_body,
 * with x_D = dirichlet_scale * dirichlet_value.  d_D = C_eff/A_eff [B][m][m]; d_S [B][m] or NULL.
 * Linear: d_S = NULL, scale = 1 -> x = u.  Newton: d_S = P_eff, scale = increment -> x = du.
 * d_x [n_macro_dof] is written in full (x_D included).  If `info` is non-NULL the call
 * synchronises and fills it; CG failure is returned as a status either way (synchronising). */
int hom_macro_solve(hom_ctx* ctx, const double* d_D, const double* d_S, double dirichlet_scale,
                    double* d_x, hom_solve_info* info, void* stream);

/* External-load factor lambda (load stepping T_k = k T / n_l): the residual
 * is R = sum_qp eta B^T S_b - lambda (f_body + f_nodal).  Default 1; host-side, no sync. */
int hom_set_load_factor(hom_ctx* ctx, double load_factor);
/* Assemble the macro stiffness K = sum_qp eta B^T D_b B (K5) into
 * the context's CSR matrix (node-block pattern over all DOFs) without solving.  Enqueue only. */
int hom_macro_assemble(hom_ctx* ctx, const double* d_D, void* stream);
/* d_y [n_macro_dof] = K_FF d_x on the free rows of the last assembled macro matrix, 0 on the
 * Dirichlet rows (K6, the SpMV of the macro CG).  Enqueue only. */
int hom_macro_spmv(hom_ctx* ctx, const double* d_x, double* d_y, void* stream);
/* Inspection of K1 (test / verification use): assembles RVE `rve` (small strain only) with the
 * production kernel into the context's scratch pool and expands its lower K_ff tiles into the
 * dense symmetric d_Kff [N_pad][N_pad] in the natural fluctuation layout (PAPER.md
 * eq:discreteSys_L, un-normalised: sum_e sum_qp eta~ B_f^T C B_f; the corner class is an
 * identity pad).  Overwrites the scratch pool (call between condensations); synchronises. */
int hom_debug_rve_kff(hom_ctx* ctx, int rve, double* d_Kff, void* stream);
/* ||R_F||_2 with R = sum_qp eta B^T S_b - f_body (macro residual, eq:linSys); synchronises. */
int hom_macro_residual_norm(hom_ctx* ctx, const double* d_S, double* norm, void* stream);

/* Fluctuation recovery (eq:reduction P:388-390 / P:424-427), local RVE range only.
 * Small strain: d_w [B][N_pad] = -X_b eps_b(d_x)           (d_x = u).
 * Finite strain: w += -(X_b dF_b(d_x) + K_ff^-1 r_f,b)       (d_x = du), internal state;
 *                copied to d_w if non-NULL. */
int hom_recover_fluctuations(hom_ctx* ctx, const double* d_x, double* d_w, void* stream);

/* Finite-strain Newton update of both scales: u += du and
 * w += -(X_b dF_b(du) + K_ff^-1 r_f,b), using the factorisation of the last
 * hom_condense.  d_u, d_du [n_macro_dof]. */
int hom_newton_update(hom_ctx* ctx, double* d_u, const double* d_du, void* stream);

/* Finite-strain fluctuation state [B][N_pad] (checkpoint / parity-per-state). */
int hom_set_fluctuations(hom_ctx* ctx, const double* d_w, void* stream);
int hom_get_fluctuations(hom_ctx* ctx, double* d_w, void* stream);

/* max_b ||r_f,b||_2 / |Omega| of the last finite-strain hom_condense: the micro residual R_micro of
 * eq:constSolution2 / P:313-315, which carries the 1/|Omega| of eq:discreteSys_L (with the
 * Dirac basis the macro integral reduces to the value at the Gauss point by the shifting property,
 * P:248-250), i.e. the RVE-averaged residual (R21).  Synchronises. */
int hom_micro_residual_max(hom_ctx* ctx, double* out, void* stream);

/* Macro-only update d_u += d_du [n_macro_dof] (the q <- q + dq of P:342 without the fluctuation
 * update; used by the classical staggered scheme's no-predictor variant).  Enqueue only. */
int hom_macro_update(hom_ctx* ctx, double* d_u, const double* d_du, void* stream);

/* Replace the phase field and/or material table (same shapes and per_rve flags as at
 * setup) from HOST memory (pinned recommended) with asynchronous copies on `stream`;
 * either pointer may be NULL to keep the current data.  This is the per-step input
 * of an end-to-end run.  Phase ids are validated on the host first (HOM_ERR_INVALID_ARG
 * if any id >= n_phases; nothing is copied then). */
int hom_set_phases(hom_ctx* ctx, const uint8_t* h_phase, const double* h_params, void* stream);

/* Constant macro basis (options.macro_basis = 1) only: the per-element volume average <C>_e
 * [B][m][m] that hom_condense keeps for the macro stiffness (eq:constSolution1/2).
 * With RVE sharding a context holds only its local rows, so the caller all-gathers them next to
 * C_eff: get copies the local rows [rve_begin, rve_begin + rve_count) into d_cavg (other rows
 * untouched), set replaces all B rows from d_cavg.  Enqueue only; HOM_ERR_INVALID_ARG for the
 * Dirac basis. */
int hom_get_element_cavg(hom_ctx* ctx, double* d_cavg, void* stream);
int hom_set_element_cavg(hom_ctx* ctx, const double* d_cavg, void* stream);

/* Kernel launches enqueued by this context since creation (for launch accounting). */
int64_t hom_launch_count(const hom_ctx* ctx);

/* Per-kernel-class device time, measured with CUDA events recorded around each launch
 * on the launching stream while profiling is enabled. */
enum {
  HOM_PROF_RVE_ASSEMBLE = 0, /* K1 (and the finite-strain material pass) */
  HOM_PROF_CONDENSE = 1,     /* K2-K4 fused Cholesky / solves / Schur */
  HOM_PROF_MACRO_ASSEMBLE = 2,/* K5 + right-hand side */
  HOM_PROF_CG = 3,           /* K6/K7 */
  HOM_PROF_RECOVER = 4,      /* K8 + kinematics */
  HOM_PROF_OTHER = 5,
  HOM_PROF_N = 6
};
int hom_profile_enable(hom_ctx* ctx, int enable);
/* Synchronises on the last recorded event, writes the accumulated milliseconds and
 * launch counts per class (arrays of HOM_PROF_N), and resets the accumulators. */
int hom_profile_read(hom_ctx* ctx, double* ms, int64_t* launches);

int hom_last_error(const hom_ctx* ctx, hom_error_info* out);
void hom_destroy(hom_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HOM_H */
