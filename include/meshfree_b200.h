/*
 * meshfree_b200.h -- C ABI of the B200 (sm_100a) RBF-FD hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch types.
 * Each entry point replaces one reference interface (paths relative to the
 * reference checkout, pkg/src/meshfree/...):
 *
 *   mf_knn            geometry/stencils.py:19-93    find_closest_stencils
 *   mf_phs_weights    _phs_batch.py:305-324         batch_phs_weights
 *                     (kernel body _phs_batch.py:142-302, caller storage.py:342-409)
 *   mf_csr_build      storage.py:156-170            WeightStore.matrix (structure)
 *   mf_csr_gather     storage.py:165-168            WeightStore.matrix (values per family)
 *   mf_apply          storage.py:186-188            WeightStore.apply_all (scipy csr_matvec)
 *   mf_apply_rows     storage.py:174-184            WeightStore.apply (selected rows)
 *   mf_plan_*         storage.py:186-188            apply_all through a locality-ordered ELL plan
 *   mf_*_terms        storage.py:174-222            apply / gradient / divergence / vector_laplacian /
 *                                                   grad_div (several families and fields, one pass)
 *   mf_heat_steps     drivers.py:87-110             run_heat_explicit step loop
 *   mf_heat_pack      (none: packed operator for the heat loop, same results)
 *   mf_neumann_values storage.py:226-250            WeightStore.neumann_value (batched)
 *
 * Conventions
 *   - Array arguments are DEVICE pointers unless the parameter is documented
 *     as a host array; they are borrowed, never freed.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All work is
 *     enqueued on it; calls return without synchronising unless noted.
 *   - Workspaces are caller-allocated device buffers sized by the matching
 *     *_workspace_size query; the library performs no allocation.
 *   - Return value: MF_OK or an error code; mf_last_error() describes the last
 *     failure on the calling thread.  Errors detected inside kernels (singular
 *     stencils, blow-up) are reported through status outputs, not return codes.
 */
#ifndef MESHFREE_B200_H
#define MESHFREE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MF_ABI_VERSION 1

#define MF_OK 0
#define MF_ERR_ARG 1
#define MF_ERR_CUDA 2
#define MF_ERR_UNSUPPORTED 3
#define MF_ERR_WORKSPACE 4

/* limits of the batched shape kernel */
#define MF_MAX_DIM 3
#define MF_MAX_FAMILIES 16
#define MF_MAX_MONOMIALS 128

/* family kinds (_phs_batch.py:22-25) and scale codes (_phs_batch.py:27-29) */
#define MF_KIND_IDENTITY 0
#define MF_KIND_D1 1
#define MF_KIND_D2 2
#define MF_KIND_LAPLACIAN 3
#define MF_SCALE_NONE 0
#define MF_SCALE_NEAREST 1
#define MF_SCALE_SUPPORT 2

/* shape-solve modes */
#define MF_PHS_REPLAY 0 /* reference op order, no FMA: ~bitwise with the reference */
#define MF_PHS_FAST 1   /* FMA elimination, parallel back-substitution */
#define MF_PHS_HYBRID 2 /* FAST, then REPLAY for stencils whose conditioning flags them */

int mf_abi_version(void);
const char* mf_last_error(void);
/* number of kernels this library has launched in the process (instrumentation) */
long long mf_launch_count(void);
/* fp64 pipe probe: blocks x threads threads, each 8 chains of 16*iters DFMA;
 * *flops receives the flop count of the launch (timing is the caller's). */
int mf_dfma_probe(int blocks, int threads, int iters, double* out, void* stream, double* flops);

/* ---- stencil selection ------------------------------------------------------
 * For each target t (targets[t] is a node index) select the n pool nodes with
 * the smallest (d2, node index), d2 in numpy-einsum rounding order, with the
 * reference's tie-straddle re-selection and self-first rule
 * (stencils.py:37-91).  out_idx is T x n int32, row-major, stencil order.
 * n_straddle (device int64, nullable) receives the number of straddle rows.
 * Preconditions (checked by the caller as the reference does, stencils.py:28-35):
 * 1 <= n <= P, 1 <= d <= 3.  pos is N x d f64 row-major; targets/pool int64.
 * Ordering: everything is ordered after prior work on `stream` and complete for later
 * work on `stream`; internally the target-side sort runs on a library-owned side stream
 * forked from and joined back into `stream` by events (capturable in a CUDA graph;
 * one fork..join enqueue at a time per device, mutex-guarded). */
int mf_knn_workspace_size(int64_t N, int32_t d, int64_t T, int64_t P, int32_t n, size_t* bytes);
int mf_knn(const double* pos, int64_t N, int32_t d, const int64_t* targets, int64_t T,
           const int64_t* pool, int64_t P, int32_t n, int32_t* out_idx, int64_t* n_straddle,
           void* ws, size_t ws_bytes, void* stream);

/* ---- batched polyharmonic RBF-FD weights -----------------------------------
 * Mirrors batch_phs_weights(pts, rows, stencils, k, even, expos, base_bot,
 * kinds, ax_a, ax_b, orders, scale_code).  expos (l x d int32), base_bot
 * (nf x l f64) and kinds/ax_a/ax_b/orders (nf int32) are HOST arrays.
 * out is m x nf x n f64; status is m int8 (0 ok, 1 singular / non-finite,
 * 2 degenerate scale); first_fail (device int64, nullable) receives the lowest
 * failing row index, or INT64 0x7f7f7f7f7f7f7f7f when every row succeeded.
 * n_replayed (device int64, nullable) counts rows re-solved in REPLAY order
 * (HYBRID mode).  opts (host struct, nullable) sets the HYBRID threshold and
 * an optional per-row conditioning-estimate output.  HYBRID's first pass is
 * the nullspace solve for r^3 with degree >= 1 on the compiled hot shapes,
 * else the FAST LU; requesting kappa selects the FAST LU first pass. */
typedef struct {
    double hybrid_threshold; /* HYBRID re-solve threshold on the sensitivity estimate
                                ||A||_inf ||(A^-1 z)_w||_inf max_f ||x_f||_inf/||w_f||_inf; <= 0: default */
    double* kappa;           /* device, 4*m, nullable: per row ||A||_inf, ||(A^-1 z)_w||_inf,
                                ||A^-1 z||_inf, max_f ||x_f||/||w_f|| (FAST/HYBRID modes) */
    double min_separation;   /* HYBRID also re-solves stencils whose closest node pair is nearer
                                than this fraction of the stencil radius; <= 0: default */
} mf_phs_options_t;
#define MF_PHS_DEFAULT_THRESHOLD 1e8
#define MF_PHS_DEFAULT_MIN_SEPARATION 1e-2
int mf_phs_workspace_size(int64_t m, size_t* bytes);
int mf_phs_weights(const double* pos, int64_t N, int32_t d, const int64_t* rows,
                   const int32_t* stencils, int64_t m, int32_t n, int32_t k, int32_t even,
                   const int32_t* expos, int32_t l, const double* base_bot,
                   const int32_t* kinds, const int32_t* ax_a, const int32_t* ax_b,
                   const int32_t* orders, int32_t nf, int32_t scale_code, int32_t mode,
                   double* out, int8_t* status, int64_t* first_fail, int64_t* n_replayed,
                   const mf_phs_options_t* opts, void* ws, size_t ws_bytes, void* stream);

/* ---- canonical CSR -------------------------------------------------------------
 * Structure of WeightStore.matrix: N x N, rows ascending, columns ascending
 * (stable for equal columns), rows only for the stored nodes `rows` (unique).
 * indptr (N+1 int32), indices (m*n int32), perm (m*n int32: source slot
 * r*n + j in stencil order of each CSR entry).  dup_flag (device int32,
 * nullable) is set non-zero if `rows` repeats a node. */
int mf_csr_workspace_size(int64_t N, size_t* bytes);
int mf_csr_build(const int64_t* rows, const int32_t* stencils, int64_t m, int32_t n, int64_t N,
                 int32_t* indptr, int32_t* indices, int32_t* perm, int32_t* dup_flag,
                 void* ws, size_t ws_bytes, void* stream);
/* data[p] = w[perm[p]] (one family, w in stencil order). */
int mf_csr_gather(const int32_t* perm, const double* w, int64_t nnz, double* data, void* stream);

/* ---- explicit application ----------------------------------------------------
 * y_i = sum over row i in storage order, sequential from 0.0, no FMA: bitwise
 * equal to scipy's csr_matvec on the same CSR.  mf_apply reads the CSR
 * directly (thread per row). */
int mf_apply(const int32_t* indptr, const int32_t* indices, const double* data,
             const double* u, double* y, int64_t N, void* stream);
/* y[k] = (A u)[sel[k]] for a list of rows (WeightStore.apply). */
int mf_apply_rows(const int32_t* indptr, const int32_t* indices, const double* data,
                  const double* u, const int64_t* sel, int64_t count, double* y, void* stream);

/* ---- apply plan (HBM-rate explicit application) ---------------------------------
 * The plan stores the CSR entries ELL-32 slot-major -- entry j of plan row r at
 * ((r/32)*W + j)*32 + r%32, W = max row length -- with the rows renumbered
 * along a Morton curve of the node positions (order: plan row -> node, inv:
 * node -> plan row) so a warp's rows and their columns are spatial neighbours.
 * The addend order inside each row is the CSR's, so sums stay bitwise equal to
 * mf_apply.  order/inv may be NULL (identity).  ell_len (N int32) receives each
 * plan row's length. */
int mf_order_workspace_size(int64_t N, size_t* bytes);
int mf_locality_order(const double* pos, int64_t N, int32_t d, int32_t* order, int32_t* inv,
                      void* ws, size_t ws_bytes, void* stream);
/* ell_idx (ceil(N/32)*32*W int32, nullable), ell_val (same count f64, nullable) */
int mf_plan_build(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N,
                  int32_t W, const int32_t* order, const int32_t* inv, int32_t* ell_idx,
                  double* ell_val, int32_t* ell_len, void* stream);
/* A plan built with order but inv = NULL keeps the columns in node numbering:
 * mf_plan_apply_direct then reads u in node order and writes y[order[r]] (one
 * launch, no permutes; bitwise the same sums). */
int mf_plan_apply_direct(const int32_t* ell_idx, const double* ell_val, const int32_t* ell_len, int64_t N,
                         int32_t W, const int32_t* order, const double* u, double* y, void* stream);
/* y = A u in node order; with an order, u/y are permuted through scratch_u/scratch_y (N each) */
int mf_plan_apply(const int32_t* ell_idx, const double* ell_val, const int32_t* ell_len, int64_t N,
                  int32_t W, const int32_t* order, const double* u, double* y, double* scratch_u,
                  double* scratch_y, void* stream);
/* ---- operator combinations over one stencil structure ----------------------------
 * Every family of a WeightStore shares one CSR structure (and one plan).  A
 * "terms" descriptor lists row sums s_t = (A_{fam[t]} u_{fld[t]})_i, each in
 * the CSR's addend order from 0.0 (WeightStore.apply, storage.py:174-184), and
 * outputs out[o]_i = ((0.0 + s_{t0[o]}) + s_{t0[o]+1}) + ... over the terms
 * t0[o] .. t0[o+1]-1, the accumulation of gradient / divergence /
 * vector_laplacian / grad_div (storage.py:190-222).  Pointer tables are HOST
 * arrays copied at the call; the arrays they point to are device arrays. */
#define MF_MAX_TERMS 16
typedef struct {
    int32_t nterm;                      /* <= MF_MAX_TERMS */
    int32_t nout;                       /* <= MF_MAX_TERMS */
    const double* val[MF_MAX_TERMS];    /* per term: the family's values (plan layout or CSR data) */
    const double* fld[MF_MAX_TERMS];    /* per term: its field (plan order or node order) */
    int32_t out_t0[MF_MAX_TERMS + 1];   /* output o sums terms out_t0[o] .. out_t0[o+1]-1 */
    double* out[MF_MAX_TERMS];          /* per output: N values (plan) or count values (rows) */
} mf_terms_t;
/* Whole field over an apply plan: fields in plan order; outputs in node order
 * when order is given (scattered through it), else in plan order. */
int mf_plan_apply_terms(const int32_t* ell_idx, const int32_t* ell_len, int64_t N, int32_t W,
                        const int32_t* order, const mf_terms_t* terms, void* stream);
/* Selected rows sel[0..count) over the CSR (values = CSR data, fields in node
 * order); output o gets count values. */
int mf_apply_terms_rows(const int32_t* indptr, const int32_t* indices, const int64_t* sel, int64_t count,
                        const mf_terms_t* terms, void* stream);

/* dst[i] = src[order[i]] (scatter = 0) or dst[order[i]] = src[i] (scatter = 1) */
int mf_permute(const double* src, const int32_t* order, int64_t N, int32_t scatter, double* dst,
               void* stream);

/* ---- row-partitioned explicit step (multi-GPU heat loop) --------------------------
 * One forward-Euler step on a block of n rows (drivers.py:88-98 per block):
 * lap = the rows' Laplacian of the gathered field (mf_apply on the rank's CSR
 * rows, global columns), out = interior ? u + dt * (D * lap + f) : u, then g on
 * Dirichlet rows; peak (nullable) max-ed with the IEEE bits of |out|. */
int mf_heat_rows(const double* lap, const double* u, const uint8_t* interior, const uint8_t* dirichlet,
                 const double* g, const double* source, double dt, double diffusivity, int64_t n, double* out,
                 uint64_t* peak, void* stream);

/* ---- explicit Neumann closure ---------------------------------------------------
 * For listed node i with stencil row r = node_row[i] (stencils m x n int32,
 * stencil order, listed as nodes[k]): c_j = sum_a normals[k,a] * w_d1[a*mn + r*n + j]
 * (storage.py:226-234), pivot guard |c_0| < 1e-12 ||c||_2 (storage.py:240-245),
 * value (gn[k] - sum_{j>=1} c_j u[st_j]) / c_0 (storage.py:246-250).
 * out (count, nullable) receives the values; u_scatter (N, nullable) gets
 * u_scatter[nodes[k]] = value; peak (uint64, nullable) is max-ed with the
 * IEEE bits of |value|; bad (device int64) receives the lowest k whose pivot
 * is negligible, else 0x7f7f7f7f7f7f7f7f. */
typedef struct {
    const int32_t* stencils;
    int32_t n;
    const double* w_d1; /* d planes of m*n weights (families d1_0..d1_{d-1}) */
    int64_t mn;
    int32_t d;
    const double* normals; /* count x d, row k = normal of nodes[k] */
    const int64_t* nodes;  /* count */
    const int64_t* node_row; /* N */
    const double* gn;      /* count */
    int64_t count;
    const uint8_t* mask;   /* N: 1 for listed nodes (excluded from the heat kernel's peak) */
} mf_neumann_t;
int mf_neumann_values(const mf_neumann_t* nm, const double* u, double* out, double* u_scatter,
                      uint64_t* peak, int64_t* bad, void* stream);

/* ---- forward-Euler heat stepping -----------------------------------------------
 * `steps` steps of drivers.py:88-110 over an apply plan of the laplacian
 * (every per-node array below is in plan row order), with step-invariant
 * data: interior and dirichlet masks (uint8, N),
 * Dirichlet values g_dir (N), optional source (N, nullable: the reference's
 * `+ 0.0`), optional Neumann closure (nm, nullable; values from the previous
 * field, as drivers.py:99-102; node-order plans only).  u (N) is advanced in
 * place using scratch (N).
 * peaks (steps uint64, device) receives the IEEE bits of max|u| after each
 * step (NaN sorts above inf); once a step exceeds 1e12 or is non-finite the
 * remaining steps do no work.  Dirichlet values must already be applied to u
 * before the first call (drivers.py:84-85). */
typedef struct {
    const int16_t* ell_d16;   /* ELL-32 layout: column - row, or 0 in wide tiles */
    const uint8_t* meta;      /* N: row length | interior << 5 | dirichlet << 6 */
    const uint8_t* tile_wide; /* ceil(N/32): 1 where an offset exceeds int16 (ell_idx is read) */
} mf_heat_pack_t;
/* Optional packed form of a plan for the heat loop (row length <= 16): per-step
 * reads drop by the index bytes halved and the row masks folded into one byte.
 * The result of mf_heat_steps is bitwise the same with or without it. */
int mf_heat_pack(const int32_t* ell_len, const int32_t* ell_idx, const uint8_t* interior,
                 const uint8_t* dirichlet, int64_t N, int32_t W, int16_t* ell_d16, uint8_t* meta,
                 uint8_t* tile_wide, void* stream);
/* pack: nullable; built by mf_heat_pack from the same plan and masks */
int mf_heat_steps(const int32_t* ell_len, const int32_t* ell_idx, const double* ell_val, int64_t N,
                  int32_t W, const uint8_t* interior, const uint8_t* dirichlet, const double* g_dir,
                  const double* source, double dt, double diffusivity, const mf_neumann_t* nm,
                  int64_t steps, double* u, double* scratch, uint64_t* peaks, const mf_heat_pack_t* pack,
                  void* stream);

/* ---- general weight engines (the reference's per-node loop) ---------------------
 * Replaces the per-node engine loop _run_loop (storage.py:325-339) over
 * RbfFd.weights (approx/engines.py:147-201) and WeightedLeastSquares.weights
 * (approx/engines.py:102-145): every configuration batch_phs_weights does not
 * take -- the qr / svd solvers (the reference's default is qr), Gaussian /
 * multiquadric / inverse multiquadric / r^k (k <= 2) kernels, weighted least
 * squares, composite operators (ScaledOperator / OperatorSum / Directional).
 * One warp per stencil; every family is solved from one factorisation.
 * out is m x nf x n f64 in stencil order; status is m x nf int8:
 *   0 ok, 1 non-finite weights, 2 degenerate scale (all nodes on the centre),
 *   3 polyharmonic derivative singular at the centre (k <= 2, basis.py:180-186),
 *   4 least-squares weight function not positive (engines.py:131-132);
 * first_fail (device int64) receives the lowest failing row, or
 * 0x7f7f7f7f7f7f7f7f. */
#define MF_ENGINE_RBFFD 0
#define MF_ENGINE_WLS 1
#define MF_RBF_PHS 0
#define MF_RBF_GAUSSIAN 1
#define MF_RBF_MQ 2
#define MF_RBF_IMQ 3
#define MF_WEIGHT_CONSTANT 0
#define MF_WEIGHT_GAUSSIAN 1
#define MF_SOLVER_LU 0
#define MF_SOLVER_QR 1
#define MF_SOLVER_SVD 2
#define MF_TERM_IDENTITY 0
#define MF_TERM_D1 1
#define MF_TERM_D2 2
#define MF_TERM_LAPLACIAN 3
#define MF_TERM_DIRECTIONAL 4
#define MF_MAX_ENGINE_TERMS 32
typedef struct {
    int32_t engine;       /* MF_ENGINE_* */
    int32_t rbf;          /* MF_RBF_* (RbfFd) */
    int32_t k;            /* polyharmonic exponent (odd: r^k, even: r^k log r) */
    int32_t solver;       /* MF_SOLVER_* */
    int32_t scale_code;   /* MF_SCALE_* */
    int32_t weight;       /* MF_WEIGHT_* (WLS) */
    double sigma;         /* kernel shape parameter (Gaussian / MQ / IMQ) */
    double weight_sigma;  /* Gaussian weight shape parameter (WLS) */
    int32_t d;            /* dimension */
    int32_t l;            /* monomials: RbfFd augmentation (0 = none), WLS basis size */
    int32_t expos[MF_MAX_MONOMIALS * MF_MAX_DIM]; /* exponent of monomial j on axis a at j*MF_MAX_DIM + a */
    int32_t nf;           /* families */
    int32_t term0[MF_MAX_FAMILIES + 1];  /* family f = elementary terms term0[f] .. term0[f+1]-1 */
    int32_t term_kind[MF_MAX_ENGINE_TERMS];
    int32_t term_a[MF_MAX_ENGINE_TERMS];
    int32_t term_b[MF_MAX_ENGINE_TERMS];
    int32_t term_order[MF_MAX_ENGINE_TERMS];
    double term_coeff[MF_MAX_ENGINE_TERMS];
    double term_vec[MF_MAX_ENGINE_TERMS * MF_MAX_DIM]; /* Directional vectors */
} mf_engine_t;
/* eng is a HOST struct (copied at the call) */
int mf_engine_weights(const double* pos, int64_t N, const int64_t* rows, const int32_t* stencils,
                      int64_t m, int32_t n, const mf_engine_t* eng, double* out, int8_t* status,
                      int64_t* first_fail, void* stream);

/* ---- implicit consumer: assembly, ILU(0), BiCGStab ---------------------------------
 * SparseSystem.finalize (assembly.py:91-108): committed rows given as COO in
 * commit order (rows, cols int32, vals f64; columns distinct within a row) ->
 * canonical CSR (rows ascending, columns ascending).  indptr N+1, indices /
 * data nnz. */
int mf_coo_workspace_size(int64_t N, size_t* bytes);
int mf_coo_to_csr(const int32_t* rows, const int32_t* cols, const double* vals, int64_t nnz, int64_t N,
                  int32_t* indptr, int32_t* indices, double* data, void* ws, size_t ws_bytes, void* stream);
/* The row loop of solve_poisson_implicit (drivers.py:138-154) over a weight
 * store's canonical structure (s_indptr / s_indices / s_perm from
 * mf_csr_build, node space): kind[i] = 1 interior (values v_interior, the
 * store's m x n stencil-order term combination), 2 Dirichlet (1 on the
 * diagonal), 3 Neumann (values v_neumann[neumann_row[i]] x n, stencil order),
 * 0 never committed.  mf_assemble_rows writes indptr and *nnz_out (host, the
 * call synchronises) and the lowest node that is uncommitted or lacks a stored
 * row into missing (device int64, 0x7f.. if none); mf_assemble_fill then
 * writes indices / data. */
int mf_assemble_workspace_size(int64_t N, size_t* bytes);
int mf_assemble_rows(const int32_t* s_indptr, const int8_t* kind, int64_t N, int32_t* indptr, int64_t* missing,
                     int64_t* nnz_out, void* ws, size_t ws_bytes, void* stream);
int mf_assemble_fill(const int32_t* s_indptr, const int32_t* s_indices, const int32_t* s_perm, int32_t n,
                     const double* v_interior, const double* v_neumann, const int64_t* neumann_row,
                     const int8_t* kind, int64_t N, const int32_t* indptr, int32_t* indices, double* data,
                     void* stream);
/* ILU(0) preconditioner in multicolour order (replaces spilu's ILUT,
 * solve.py:49-62): the symmetrised pattern is coloured (Jones-Plassmann, at
 * most 128 colours), rows of one colour never couple, so the factorisation and
 * both substitutions run colour by colour.  The struct is filled by
 * mf_ilu0_build (host), its arrays are caller-owned device buffers. */
#define MF_MAX_COLORS 128
typedef struct {
    const int32_t* indptr;
    const int32_t* indices;
    const int8_t* part;   /* nnz: -1 L, 0 diagonal, +1 U */
    const int32_t* diag;  /* N: position of the diagonal entry */
    const double* lu;     /* nnz: unit-L below / U on and above, CSR order */
    const int32_t* order; /* N: rows colour by colour */
    int32_t ncolors;
    int32_t rounds;       /* colouring rounds taken */
    int32_t color_off[MF_MAX_COLORS + 1];
} mf_ilu0_t;
int mf_ilu0_workspace_size(int64_t N, size_t* bytes);
/* color, order, diag: N int32; part: nnz int8; lu: nnz f64.  zero_pivot_row
 * (device int64) receives the lowest row without a diagonal entry or
 * 0x7f7f7f7f7f7f7f7f.  Synchronises (colouring rounds). */
int mf_ilu0_build(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N, int64_t nnz,
                  int32_t* color, int32_t* order, int8_t* part, int32_t* diag, double* lu, mf_ilu0_t* M,
                  int64_t* zero_pivot_row, void* ws, size_t ws_bytes, void* stream);
/* y = M^-1 x */
int mf_ilu0_apply(const mf_ilu0_t* M, const double* x, double* y, void* stream);
/* scipy's bicgstab recurrence (solve.py:96-99) on the device, preconditioned
 * by M (nullable: none), x0 = x on entry, stop at ||r|| < max(atol, rtol ||b||).
 * info: 0 converged, -10 / -11 breakdown, maxiter when exhausted; iterations =
 * completed iterations (the reference's callback count); residual_norm = the
 * last ||r|| the recurrence evaluated.  Synchronises every iteration. */
int mf_bicgstab_workspace_size(int64_t N, size_t* bytes);
int mf_bicgstab(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N, const mf_ilu0_t* M,
                const double* b, double* x, double rtol, double atol, int64_t maxiter, int64_t* iterations,
                int32_t* info, double* residual_norm, void* ws, size_t ws_bytes, void* stream);

/* ---- node generation: fill_interior's acceptance pass ---------------------------
 * fill_interior (geometry/fill.py:204-298) expands a FIFO of nodes generation
 * by generation; each generation's candidates are accepted strictly in order
 * when no node accepted so far lies within gamma * min(h_c, h_j)
 * (_accept_batch_numba, fill.py:38-117).  Nodes live in a uniform grid of
 * linked lists (head: one int32 per cell, -1 empty; nxt: one per node):
 * mf_fill_insert links nodes [a, b); mf_fill_accept decides one generation
 * (M candidates, cand M x d, hc M) -- the same set as the sequential pass --,
 * appends the accepted ones at pos[count..] / hv[count..] in candidate order,
 * links them, and writes their candidate indices to accepted_idx.  head2 is a
 * second all -1 cell array (scratch; left all -1).  Synchronises. */
typedef struct {
    double lo[3];    /* grid origin */
    double cell;     /* cell edge */
    int32_t dims[3]; /* cells per axis (unused axes: 1) */
    int32_t d;
} mf_fill_grid_t;
int mf_fill_workspace_size(int64_t M, size_t* bytes);
int mf_fill_insert(const double* pos, int64_t a, int64_t b, const mf_fill_grid_t* grid, int32_t* head,
                   int32_t* nxt, void* stream);
int mf_fill_accept(double* pos, double* hv, int32_t* nxt, int64_t count, int64_t cap, const mf_fill_grid_t* grid,
                   int32_t* head, int32_t* head2, const double* cand, const double* hc, int64_t M, double gamma,
                   int32_t* accepted_idx, int64_t* n_accepted, int32_t* rounds, void* ws, size_t ws_bytes,
                   void* stream);

/* The same recurrence with every branch decided on the device, so one
 * iteration is a fixed launch sequence that can be captured in a CUDA graph
 * and replayed past convergence without changing a bit (mf_bicgstab's
 * results, bitwise).  state: mf_bicgstab_state_size device bytes, read back by
 * the host as {double atol, rho, rho_prev, alpha, omega, beta, rr, rv, ts,
 * tt; int64 it, maxiter; int32 done, info, pad}: done = 1 finished (info as
 * mf_bicgstab, it = iterations, rr = last ||r||^2), 3 when b = 0 (x = b). */
int mf_bicgstab_state_size(size_t* bytes);
int mf_bicgstab_init(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N, const double* b,
                     const double* x, double rtol, double atol, int64_t maxiter, void* state, void* ws,
                     size_t ws_bytes, void* stream);
int mf_bicgstab_iter(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N,
                     const mf_ilu0_t* M, double* x, void* state, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MESHFREE_B200_H */
