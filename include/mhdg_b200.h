/*
 * mhdg_b200.h -- C ABI of the B200 macro-element HDG operator library
 * (libmhdg_b200.so).
 *
 * The reference (macrohdg, pure Python) has no FFI; its drop-in surface is
 * the duck-typed Discretization / LinearizedSystem object API.  Each entry
 * point below replaces one method of that API (cited per function); the
 * Python shim `paper_2507_22195_b200.assembly` binds them with ctypes and
 * keeps the reference's method names, argument meaning and exceptions.
 *
 * Conventions
 *  - All array pointers are caller-owned DEVICE buffers of float64 in the
 *    reference layouts: w (E, nc, 5), trace (F, nt, 5), offset
 *    (E, n_sub, nq, 5).  Lin buffers are caller-allocated with the sizes
 *    reported by mhdg_lin_sizes().
 *  - `stream` is a cudaStream_t (may be NULL = legacy default stream).
 *    Calls are stream-ordered; calls that return a status synchronize the
 *    stream before returning, the others do not.
 *  - Return codes map 1:1 onto the reference's exception classes
 *    (macrohdg/errors.py); details come back in mhdg_status.
 */
#ifndef MHDG_B200_H
#define MHDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mhdg_code {
  MHDG_OK = 0,
  MHDG_NON_ADMISSIBLE = 1,          /* NonAdmissibleState            */
  MHDG_NON_ADMISSIBLE_ENTROPY = 2,  /* NonAdmissibleEntropyState     */
  MHDG_SINGULAR_LOCAL = 3,          /* SingularLocalMatrix(macro)    */
  MHDG_SINGULAR_BLOCK = 4,          /* SingularBlock(face)           */
  MHDG_INVALID_CONFIG = 5,          /* InvalidConfig                 */
  MHDG_CUDA_ERROR = 6,
  MHDG_OUT_OF_MEMORY = 7
};

/* where_kind: 0 = "volume sub <index>", 1 = "face tile <index>",
 *             2 = "trace tile <index>" (assembly.py:428-438, :471-531) */
typedef struct {
  int code;
  int where_kind;
  int where_index;
  int64_t item; /* first offending macro (residual / local factor) or face */
  int n_unsym;  /* face blocks not symmetric (debug log, assembly.py:1025) */
} mhdg_status;

/* Host-side tables of one Discretization (paper_2507_22195_b200/tables.py),
 * uploaded once by mhdg_create.  Integer maps are int64 as in the reference. */
typedef struct {
  int dim, p, m;
  int n_macros, n_faces;
  int nn, nq, nfn, nqf, n_st, n_sub;
  int formulation; /* 0 conservative, 1 entropy        */
  int flux_kind;   /* 0 lf, 1 ec, 2 es, 3 kepes        */
  double gamma;
  const double* phi;          /* (nq, nn)        */
  const double* dphi;         /* (nq, nn, 3)     */
  const double* quad_wts;     /* (nq)            */
  const double* phi_face;     /* (n_st, nqf, nfn)*/
  const double* fphi;         /* (nqf, nfn)      */
  const double* facet_wts;    /* (nqf)           */
  const int64_t* face_rows;   /* (n_st, nfn)     */
  const double* sub_det;      /* (E)             */
  const double* sub_inv_jac;  /* (E, 3, 3)       */
  const double* face_normals; /* (E, n_st, 3)    */
  const double* face_area;    /* (E, n_st) area*(d-1)! */
  const int64_t* face_id_st;  /* (E, n_st)       */
  const int64_t* trace_idx;   /* (E, n_st, nfn)  */
  const uint8_t* boundary_st; /* (E, n_st)       */
  const int64_t* face_sides;  /* (F, 2) macro*n_st+tile, -1 if none */
  const double* freestream;   /* (5) conservative far-field state or NULL */
  int n_owned_faces;          /* faces [0, n_owned) get preconditioner blocks;
                                 0 = all (single partition)                   */
  /* viscous closure (gas.py:48-77) and reference operators of the gradient
   * equation (assembly.py:326-371), NULL / 0 for inviscid runs            */
  int has_visc;
  double reynolds, mach, prandtl, mu;
  const double* minv_ref;     /* (nn, nn)  inverse reference mass matrix  */
  const double* pref;         /* (3, nn, nn) Mref^-1 Kref_k               */
  const double* kref;         /* (3, nn, nn) Kref_k[j][i]                 */
  const double* eref;         /* (n_st, nfn, nfn) Eref_k[i][j]            */
  /* m > 1 macro subdivision (reference fem.py:550-724,
   * assembly.py:155-324); ignored for m = 1.  nc / nt: macro C0 nodes and
   * trace nodes per face; scatter: element node -> macro node per
   * sub-element; per-(macro, sub-element) geometry; CSR lists giving, per
   * trace entry (face * nt + node), the tile-contribution slots
   * ((macro * n_st + tile) * nfn + facet node) in the reference's np.add.at
   * order, and per face its tiles (macro * n_st + tile). */
  int nc, nt;
  const int64_t* scatter;        /* (n_sub, nn)          */
  const double* sub_det_all;     /* (E, n_sub)           */
  const double* sub_inv_jac_all; /* (E, n_sub, 3, 3)     */
  const int64_t* trace_ptr;      /* (F * nt + 1)         */
  const int64_t* trace_list;     /* (E * n_st * nfn)     */
  const int64_t* face_ptr;       /* (F + 1)              */
  const int64_t* face_list;      /* (E * n_st)           */
} mhdg_tables;

typedef struct mhdg_ctx mhdg_ctx;

/* Caller-allocated storage of one linearization (LinearizedSystem). */
typedef struct {
  double* sinv; /* (E, 5nc, 5nc) S^-1 per macro, column-major          */
  double* hw;   /* (E, n_st, nqf, 5, 5) dF^/dw at face quadrature      */
  double* hhat; /* (E, n_st, nqf, 5, 5) dF^/dw^                        */
  double* hh;   /* (E, n_st, nqf, 5, 5) hhat + ghost + trace ptc       */
  double* pinv; /* (F, 5nt, 5nt) face-block inverse, column-major      */
  double* wlin; /* (E, nc, 5) state of the linearization (viscous)      */
} mhdg_lin_buffers;

/* Discretization.__init__ (assembly.py:120-153): upload tables. */
mhdg_ctx* mhdg_create(const mhdg_tables* tables, int device, int* err);
void mhdg_destroy(mhdg_ctx* ctx);
/* element counts of the six mhdg_lin_buffers arrays */
void mhdg_lin_sizes(const mhdg_ctx* ctx, int64_t sizes[6]);

/* Discretization.residuals (assembly.py:459-549).  offset may be NULL;
 * has_stage = 0 means stage None.  check = 0 skips the rho/P checks
 * (residuals(check=False)).  sync = 0 leaves the status on the device
 * (retrieve with mhdg_status_fetch).  q / r_q: (E, nc, 5, 3) gradient
 * unknowns and their residual, NULL for inviscid runs. */
int mhdg_residual(mhdg_ctx* ctx, const double* w, const double* trace,
                  const double* q, int has_stage, double alpha,
                  const double* offset, int check, double* r_w,
                  double* r_trace, double* r_q, int sync, mhdg_status* st,
                  void* stream);
/* Discretization.solve_gradient (assembly.py:398-411): q = M^-1 (E w^ - K w) */
int mhdg_solve_gradient(mhdg_ctx* ctx, const double* w, const double* trace,
                        double* q, void* stream);
int mhdg_status_fetch(mhdg_ctx* ctx, mhdg_status* st, void* stream);

/* Discretization.jacobian / LinearizedSystem.__init__ (assembly.py:697-1026):
 * linearization tensors, S assembly, per-macro S^-1, face-block inverses. */
int mhdg_linearize(mhdg_ctx* ctx, const double* w, const double* trace,
                   const double* q, double alpha, double ptc_weight,
                   const mhdg_lin_buffers* lin, mhdg_status* st, void* stream);

/* The two halves of mhdg_linearize, for partitioned runs where the
 * preconditioner blocks of halo faces need the other rank's side:
 * mhdg_linearize_local builds S^-1, hw, hhat, hh; mhdg_precond_factor
 * assembles and inverts the owned face blocks, taking remote sides
 * (face_sides entries <= -2) from hh_remote (n_remote, nqf, 5, 5),
 * tidx_remote (n_remote, nfn) and area_remote (n_remote) device arrays. */
int mhdg_linearize_local(mhdg_ctx* ctx, const double* w, const double* trace,
                         const double* q, double alpha, double ptc_weight,
                         const mhdg_lin_buffers* lin, mhdg_status* st,
                         void* stream);
int mhdg_precond_factor(mhdg_ctx* ctx, const mhdg_lin_buffers* lin,
                        int n_remote, const double* hh_remote,
                        const int32_t* tidx_remote, const double* area_remote,
                        mhdg_status* st, void* stream);

/* Macro-range forms for partitioned runs (no reference counterpart: the
 * reference is single-process; these compute the same operators as
 * Discretization.residuals (assembly.py:459-549) and LinearizedSystem.matvec
 * (assembly.py:1131-1143) restricted to the contributions of macros
 * [e_begin, e_end), accumulated into the trace outputs).  zero = 1 clears
 * r_trace / y (and the residual status) first.  Calling them for the
 * interior macros and then for the halo macros gives results bit-identical
 * to the whole-range call (two contributions per trace node, 0 + a + b),
 * which lets the trace halo exchange overlap the interior work.  matvec
 * stages: bit 0 = face-in + local solve, bit 1 = face-out.  q / r_q: the
 * gradient unknowns and their residual of a viscous context (NULL
 * otherwise). */
int mhdg_residual_range(mhdg_ctx* ctx, const double* w, const double* trace, const double* q,
                        int has_stage, double alpha, const double* offset, int check, double* r_w,
                        double* r_trace, double* r_q, int64_t e_begin, int64_t e_end, int zero,
                        void* stream);
int mhdg_matvec_range(mhdg_ctx* ctx, const mhdg_lin_buffers* lin, const double* x, double* y,
                      int64_t e_begin, int64_t e_end, int stages, int zero, void* stream);

/* LinearizedSystem.matvec (assembly.py:1131-1143): y = A^ x */
int mhdg_matvec(mhdg_ctx* ctx, const mhdg_lin_buffers* lin, const double* x,
                double* y, void* stream);
/* LinearizedSystem.condensed_rhs (assembly.py:1145-1157) */
int mhdg_condensed_rhs(mhdg_ctx* ctx, const mhdg_lin_buffers* lin,
                       const double* r_w, const double* r_trace,
                       const double* r_q, double* b, void* stream);
/* LinearizedSystem.recover (assembly.py:1159-1173): d_w (and d_q if viscous) */
int mhdg_recover(mhdg_ctx* ctx, const mhdg_lin_buffers* lin, const double* r_w,
                 const double* r_q, const double* d_trace, double* d_w,
                 double* d_q, void* stream);
/* LinearizedSystem.apply_preconditioner (assembly.py:1175-1180) */
int mhdg_precond(mhdg_ctx* ctx, const mhdg_lin_buffers* lin, const double* r,
                 double* z, void* stream);

/* Discretization.volume_quad_states (assembly.py:417-426): (E,1,nq,5) */
int mhdg_volume_quad_states(mhdg_ctx* ctx, const double* w, double* out,
                            mhdg_status* st, void* stream);
/* to_conservative / from_conservative on n nodal states (n, 5) */
int mhdg_to_conservative(mhdg_ctx* ctx, int64_t n, const double* w, double* u,
                         mhdg_status* st, void* stream);
int mhdg_from_conservative(mhdg_ctx* ctx, int64_t n, const double* u, double* w,
                           void* stream);
/* Discretization.integrals (assembly.py:595-620): out_host[5] =
 * entropy, thermo_entropy, kinetic_energy, mass, total_energy */
int mhdg_integrals(mhdg_ctx* ctx, const double* w, double* out_host,
                   void* stream);
/* Discretization.entropy_identity_defect (assembly.py:649-672, face term
 * fluxes.py:245-255): out_host = {lhs, rhs, |lhs - rhs|} with
 * lhs = sum v . r_w - sum v_hat . r_trace (r_* = residuals at stage None of
 * the same fields) and rhs = -sum over side tiles and face points of
 * face_w [(v(u_hat) - v(u)) . F^ - (psi_n(u_hat) - psi_n(u))]. */
int mhdg_entropy_identity(mhdg_ctx* ctx, const double* w, const double* trace,
                          const double* r_w, const double* r_trace, double* out_host,
                          void* stream);
/* Discretization.kinetic_energy_dissipation numerator (assembly.py:622-648):
 * out_host[0] = 2 mu_eff * integral of rho |curl V|^2 / 2 (divide by |Omega|) */
int mhdg_dissipation(mhdg_ctx* ctx, const double* w, const double* q,
                     double* out_host, void* stream);

/* FGMRES vector kernels (solver.py:42-118), deterministic reductions.
 * mhdg_dot: out_dev[0] = x . y
 * mhdg_mgs: modified Gram-Schmidt of w against rows 0..j of V (row stride n):
 *   for i<=j: h[i] = V_i . w; w -= h[i] V_i;  h[j+1] = ||w||;
 *   V_{j+1} = w / h[j+1] if h[j+1] > 1e-300.  h_dev has j+2 slots.
 * mhdg_combine: x += sum_i y_dev[i] Z_i, i < k
 * mhdg_scale: y = x * (a_dev ? a_dev[0] : a) ; mhdg_axpby: z = a x + b y */
int mhdg_dot(mhdg_ctx* ctx, int64_t n, const double* x, const double* y,
             double* out_dev, void* stream);
int mhdg_mgs(mhdg_ctx* ctx, int64_t n, int j, double* V, double* w,
             double* h_dev, void* stream);
int mhdg_combine(mhdg_ctx* ctx, int64_t n, int k, const double* Z,
                 const double* y_dev, double* x, void* stream);
int mhdg_scale(mhdg_ctx* ctx, int64_t n, const double* x, double a,
               const double* a_dev, int invert, double* y, void* stream);
int mhdg_axpby(mhdg_ctx* ctx, int64_t n, double a, const double* x, double b,
               const double* y, double* z, void* stream);
/* y -= a_dev[0] * x  (distributed MGS step with an all-reduced scalar) */
int mhdg_axpy_dev(mhdg_ctx* ctx, int64_t n, const double* a_dev,
                  const double* x, double* y, void* stream);

/* Device-resident condensed solve: solver.solve_condensed (solver.py:121-170)
 * = FGMRES(restart, rel_tol, max_outer) preconditioned by an inner
 * GMRES(inner_iters, inner_rtol) sweep that is itself preconditioned by the
 * face-block solve (inner_precond = 0: face-block solve only), all as one
 * CUDA graph with conditional WHILE / IF nodes (no host round trip inside
 * the solve).  The caller allocates the workspace (mhdg_krylov_workspace
 * doubles of device memory).  mhdg_krylov_solve: x = solution for the
 * condensed right-hand side b (both (F, nt, 5) device buffers); the stats
 * are copied to `stats` at the end of the solve: sync = 1 waits for them,
 * sync = 0 returns at once (stats must then be pinned host memory, valid once
 * the stream reaches that point).  The graph is (re)built when `lin` differs
 * from the previous call's buffers. */
typedef struct {
  double rel_tol;
  int restart;
  int max_outer;
  double inner_rtol;
  int inner_iters;
  int inner_precond;
  /* 1: the inner sweep forms its true residual b - A x after the cycle, as
   * solver.py:62-72 does literally (one more matvec per sweep).  0: when the
   * cycle ended on the iteration cap the sweep returns x whatever that
   * residual is (solver.py:68-69: exact), and when it ended on the Arnoldi
   * residual test |g_k| / |b| <= inner_rtol that estimate stands in for the
   * true residual (equal in exact arithmetic); breakdown exits still form
   * the true residual.  The outer level always forms it. */
  int inner_true_residual;
  /* 1 (needs inner_true_residual = 0): the outer column's w = A z for the z an
   * inner sweep returned comes from that sweep's Arnoldi relation,
   * A z = V_{k+1} (H y) with H the sweep's Hessenberg matrix before the
   * rotations (k + 1 vector updates instead of a matvec; the relation holds
   * to working precision whatever the orthogonality of V).  0: w = A z by the
   * operator, as solver.py:86-88 does literally.  Sweeps that took the
   * true-residual path or never updated x always use the operator. */
  int outer_matvec_reuse;
} mhdg_krylov_params;

typedef struct {
  int outer_iterations;  /* SolveStats.outer_iterations */
  int inner_iterations;  /* SolveStats.inner_iterations */
  int converged;         /* SolveStats.converged        */
  int updated;           /* x received a correction      */
  double rel_residual;   /* SolveStats.rel_residual     */
} mhdg_krylov_stats;

typedef struct mhdg_krylov mhdg_krylov;
int64_t mhdg_krylov_workspace(const mhdg_ctx* ctx, const mhdg_krylov_params* prm);
mhdg_krylov* mhdg_krylov_create(mhdg_ctx* ctx, const mhdg_krylov_params* prm,
                                double* workspace, int64_t workspace_len, int* err);
int mhdg_krylov_solve(mhdg_krylov* k, const mhdg_lin_buffers* lin, const double* b,
                      double* x, mhdg_krylov_stats* stats, int sync, void* stream);
void mhdg_krylov_destroy(mhdg_krylov* k);

/* Diagnostic of the last linearization's batched inversions: out[0] / out[1]
 * = S blocks / face blocks that failed the diagonal-pivot ratio check and
 * went through the partial-pivoting pass (synchronizes the stream). */
int mhdg_gj_fallbacks(mhdg_ctx* ctx, int* out, void* stream);

/* Batched in-place inverse of nmat row-major matrices of order n (20, 50 or
 * 100), column-major result: the device replacement of the reference's
 * per-macro lu_factor / lu_solve (assembly.py:718-733) and per-face block
 * factorization (assembly.py:736-752), exposed for direct testing.  Diagonal-
 * pivot pass first, partial pivoting for the matrices that fail its checks
 * (*fallbacks = their number); MHDG_SINGULAR_LOCAL with *item = the first
 * singular matrix.  nmat <= max(macros, faces) of the context.  Synchronizes. */
int mhdg_batched_inverse(mhdg_ctx* ctx, int n, int nmat, double* mats, int* fallbacks,
                         int64_t* item, void* stream);

/* number of library kernels launched since creation (evidence counter) */
int64_t mhdg_launch_count(const mhdg_ctx* ctx);
/* FP64 FMA throughput probe (roofline denominator), returns GFLOP/s */
double mhdg_fp64_probe(int device, void* stream);
/* FP64 tensor-core (mma.sync m8n8k4 f64, SASS DMMA) probe, GFLOP/s */
double mhdg_dmma_probe(int device, void* stream);
/* y[i] = f(x[i]) with the operator's device elementary functions
   (fn 0: exp, 1: log, 2: division 1 / x): accuracy check of the pointwise
   algebra against libm; replaces no reference symbol (numpy's exp / log /
   true_divide inside gas.py / fluxes.py) */
int mhdg_math_eval(int fn, int64_t n, const double* x, double* y, void* stream);
/* Host (CPU) topology kernels of the table builder; no device work.
 * mhdg_pair_sides: skeleton pairing (reference mesh.py:226-299): sides with
 * identical canonical quantised vertex keys (n_sides x key_width int64) are
 * paired, partner[s] = other side or -1; returns the number of key groups
 * with more than two sides (TopologyError when > 0).
 * mhdg_match_points: trace-node matching (reference assembly.py:299-322):
 * match[f][a] = first b minimising |pts_nb[f][a] - pts_own[f][b]|; returns
 * the largest matched distance, or -1 when a face's matching is not a
 * permutation. */
int64_t mhdg_pair_sides(int64_t n_sides, int key_width, const int64_t* keys, int64_t* partner);
double mhdg_match_points(int64_t n_faces, int nt, int dim, const double* pts_nb,
                         const double* pts_own, int64_t* match);
/* mhdg_side_keys: canonical quantised side keys (wrap on periodic max
 * planes, round(x / quantum), rows sorted) of n_sides sides (d x d vertex
 * coordinates each) -> keys (n_sides, d * d); mhdg_face_shift_perm: periodic
 * shift and owner -> neighbour vertex permutation of paired faces (va, vb:
 * (nf, d, d) vertices), returns the largest matched distance or -1 (both:
 * reference mesh.py:226-299, host-only). */
/* mhdg_match_faces: mhdg_match_points with the neighbour points built from
 * the macro maps (origin + J fun[nfl] - shift; fun: (d+1, nt, d) face-unique
 * reference nodes, ne / nfl: neighbour macro and local face per face). */
double mhdg_match_faces(int64_t nf, int nt, int d, const double* fun, const int64_t* ne,
                        const int64_t* nfl, const double* origins, const double* jac,
                        const double* shift, const double* po, int64_t* match);
void mhdg_side_keys(int64_t n_sides, int d, const double* sv, const double* box_hi,
                    const double* extent, const int* periodic, double quantum, int64_t* keys);
double mhdg_face_shift_perm(int64_t nf, int d, const double* va, const double* vb,
                            const double* extent, double* shift, int64_t* perm);
const char* mhdg_version(void);

#ifdef __cplusplus
}
#endif
#endif
