/*
 * hm.h -- C ABI of the B200-native hierarchical block low-rank cavity-radiation hot path.
 *
 * Paper: Baburin, Ballani, Peterson, Knezevic, "Hierarchical block low-rank approximation of
 * cavity radiation" (arXiv 2305.06891), reproduced as PAPER.md.  The hot path is the repeated
 * application, inside every nonlinear/time step, of the compressed radiation operators:
 *     y = F x          (H-matrix-vector product, "x -> F x ... recursively")
 *     z = C^-1 b       (C = I - Lambda F, eq:reflection_matrix PAPER.md:159-162, applied as
 *                        U^-1 (L^-1 b) with one-time block H-LU factors)
 *     q = flux(T)      (eq:qi_new_location: one solve + one apply)
 *
 * Conventions (apply to every entry point):
 *  - Every function returns hm_status; nothing throws across the ABI.  On failure
 *    hm_last_error(ctx) returns a message (it names the facet pair or block when relevant).
 *  - fp64 everywhere.  Vectors are facet-major n x nrhs (row i holds nrhs contiguous values)
 *    in the caller's EXTERNAL facet order (the order of the geometry arrays).
 *  - Setup calls (hm_build_geometry, hm_assemble_aca, hm_factor_hlu) take HOST arrays,
 *    copy what they need, and are synchronous.
 *  - hm_apply_F / hm_solve_C / hm_radiative_flux accept DEVICE pointers (stream-ordered,
 *    asynchronous, no allocation after the first call with a given nrhs) or HOST pointers
 *    (pageable or pinned: the library stages through its own device buffers on `stream` and
 *    synchronises `stream` before returning).  `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - Ownership: the caller owns all argument buffers.  The library owns its handles and all
 *    device memory it allocates; hm_destroy_* / hm_finalize free them.  Handles are immutable
 *    after setup and may be used from one host thread and one stream at a time (the hot-path
 *    calls of an F / LU pair share their device workspace; calls are stream-ordered).
 *  - Asynchronous kernel faults surface as HM_ERR_CUDA at the next synchronising call;
 *    environment HM_DEBUG=1 synchronises after every launch.
 *  - There is no CPU fallback: without a CUDA device hm_init returns HM_ERR_CUDA (device < 0 gives
 *    a host-only context for trees and shard plans; every compute call then returns an error).
 */
#ifndef HM_H_
#define HM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HM_OK = 0,
    HM_ERR_INVALID_ARG = 1,          /* bad size/pointer/parameter; call-order violation     */
    HM_ERR_CUDA = 2,                 /* CUDA runtime error or no device                      */
    HM_ERR_OOM = 3,                  /* device allocation failed (message has byte count)    */
    HM_ERR_NCCL = 4,                 /* collective failure (world > 1)                       */
    HM_ERR_DEGENERATE_GEOMETRY = 5,  /* r^2 == 0 for i != j, A_i <= 0, non-finite input      */
    HM_ERR_SINGULAR = 6,             /* |pivot| < 1e-14 ||block|| in a leaf LU               */
    HM_ERR_NOT_READY = 7,            /* handle not built / wrong handle combination          */
    HM_ERR_UNSUPPORTED = 8           /* configuration outside what this build implements     */
} hm_status;

/* hm_init flags */
#define HM_FLAG_LOCAL_GROUP 0x1u   /* world > 1 inside ONE process: comm_id points to an int64 group
                                      key shared by the ranks (one host thread per rank); the exchange
                                      is done with device copies (tests of the sharded path on one GPU) */
#define HM_FLAG_ASYNC_PINNED 0x2u  /* hot-path calls whose output is PINNED host memory (written in place
                                      by the kernels through its device alias) return without
                                      synchronizing, stream-ordered like cudaMemcpyAsync: the caller
                                      synchronizes the stream before reading the output or rewriting a
                                      pinned input.  Pageable host buffers stay synchronous. */

typedef struct hm_ctx hm_ctx;
typedef struct hm_geom hm_geom;
typedef struct hm_hmat hm_hmat;
typedef struct hm_hlu hm_hlu;
typedef struct hm_proj hm_proj;

/* Alg. 1 / Alg. 2 parameters. */
typedef struct {
    int32_t n_min;     /* leaf iff #tau <= n_min; >= 1                          */
    double eta;        /* admissibility constant c: min(diam,diam) <= c dist */
    int32_t adm_mode;  /* 0: boxes of the centroid point clouds (paper text, default);
                          1: boxes of the facet extents (facet_aabb required; reproduces Fig. 1) */
} hm_tree_params;

/* ACA parameters. */
typedef struct {
    double eps_aca;        /* eq:erel relative tolerance of the partial-pivot ACA stop test     */
    int32_t k_max;         /* rank cap (<= 64; blocks reaching it are stored dense); 0 = 48     */
    int32_t closed_cavity; /* 1: eq:rowsum / eq:clamped_rowsum / eqn:F_closed row scaling       */
    int32_t probes;        /* 0..16: when the partial-pivot stop test fires, first try this many rows
                              spread over the block as pivots (reading R30: catches parts of
                              a block the pivot path missed, e.g. on multi-body geometries); 0 = off
                              (plain step 10, the default; adds ~1.6 % stored bytes on C2)       */
    int32_t pivoting;      /* 0: partial pivoting (default); 1: full pivoting,
                              the paper's variant (NEXT-3): each admissible block is
                              evaluated densely and cross-approximated with full pivoting and the exact
                              Frobenius residual as stop test, so every block meets eq:erel; costs all
                              m n entries of the admissible blocks (moderate n only)                  */
    int32_t recompress;    /* 1: recompress every low-rank block (rank >= 2) after the ACA to its best
                              rank-k' approximation at eps_aca (QR + SVD truncation, Frobenius tail;
                              PAPER.md:642, reading R32): fewer stored bytes, ranks no longer
                              the raw ACA ranks; 0: off (default)                                    */
    int32_t quadrature;    /* 0: one-point centroid rule for every entry (default); 1: the
                              adaptive Gauss quadrature of PAPER.md:156 (reading R35): with d
                              the centroid distance and h the longer of the two facets' longest edges,
                              d >= 10h one point, 4h <= d < 10h the 3-point rule on each triangle,
                              1.5h <= d < 4h the 6-point (Dunavant degree-4) rule, d < 1.5h the 6-point
                              rule on each of the 4 midpoint sub-triangles; each point pair with its own
                              back-facing test.  Needs `vertices`.                                    */
    const double* vertices;/* quadrature = 1: host array n x 9, external order, facet i's triangle
                              (x0 y0 z0 x1 y1 z1 x2 y2 z2); read during the call only; else ignored */
} hm_aca_params;

/* H-LU parameters. */
typedef struct {
    double eps_lu;         /* truncation tolerance of the factor blocks; <= 0 -> eps_aca
                              ("equal to the approximation accuracy used for F")   */
    int32_t cut_level;     /* solve form (reading R27): level-form updates
                              b_t2 -= W^L_t b_t1 (and W^U_t for the backward sweep) for tree levels
                              < cut_level, then ONE block-diagonal solve with the inverse factors
                              of the cut_level diagonal blocks, compressed in F's partition.
                              < 0 (default) -> 0: C^-1 b = U^-1 (L^-1 b) as two H-matrix products;
                              >= depth: pure level form (leaf inverses only).                  */
    int32_t method;        /* 0 (default): hierarchical arithmetic ("stage B", reading R33):
                              the 4-step recursion of PAPER.md:770-775 on the blocks of C in F's
                              partition, recursive substitutions and block products, every low-rank
                              sum truncated at eps_lu; memory O(stored blocks), any
                              n.  1: dense tiles on the GPU ("stage A", reading R28), then truncation
                              block by block; needs ~18 n^2 bytes of device memory (n up to ~1e5);
                              kept as a cross-check.                                             */
} hm_lu_params;

/* Storage / traffic accounting (bytes are fp64 payload bytes actually stored in HBM). */
typedef struct {
    int64_t n, n_leaves, depth;
    int64_t n_blocks, n_dense, n_lowrank, n_adm_dense;
    int64_t rank_max;
    double rank_mean;                 /* over stored low-rank blocks of F                      */
    int64_t bytes_F;                  /* dense + U + V of F                                    */
    int64_t bytes_F_phase1;           /* V^T bytes (phase-1 kernel)                            */
    int64_t bytes_F_phase2;           /* dense + U bytes (phase-2 kernel)                      */
    int64_t bytes_C;                  /* level-form L/U factor blocks + leaf inverses          */
    int64_t bytes_C_leaf;             /* leaf inverses part of bytes_C                         */
    int64_t n_blocks_C, n_lowrank_C;
    int64_t rank_max_C;
    double rank_mean_C;
    int64_t launches_apply_F;         /* kernel launches per hm_apply_F column (engine: 1)      */
    int64_t launches_solve_C;         /* kernel launches per hm_solve_C column (engine: 1)      */
    double setup_seconds[8];          /* tree, aca, dense-fill+pack, rowsum+scale, C-expand,
                                         dense LU+W, W-compress+pack, flux constant g          */
    int64_t bytes_F_local;            /* world > 1: this rank's stored bytes of F (= bytes_F)   */
    int64_t bytes_C_local;            /* world > 1: this rank's bytes of the solve operators    */
    int64_t rank, world;
    int64_t lu_method;                /* 0 hierarchical (stage B), 1 dense tiles (stage A)           */
    int64_t lu_truncations;           /* stage B: low-rank truncations (QR + SVD) of the factorisation */
    int64_t lu_threads;               /* stage B: host threads of the factorisation (0: on rank 0 only) */
} hm_storage;

/* ---- lifetime ------------------------------------------------------------------------- */
/* device: CUDA ordinal (< 0: host-only context: hm_build_geometry / hm_local_range / hm_shard_plan /
   hm_export_* only, no CUDA is touched).  rank / world: SPMD position, world a power of two.
   world > 1 shards the hot path by row cluster: rank r owns the rows
   of tree node r at level log2(world) (hm_local_range) and the vectors of hm_apply_F / hm_solve_C /
   hm_radiative_flux become this rank's SLICE in internal order (n_loc x nrhs, n_loc = end - begin);
   every rank makes the same calls.  comm_id: world == 1: NULL; world > 1: the 128-byte NCCL unique id
   from hm_nccl_unique_id() on rank 0, broadcast by the caller (the library owns its communicator and
   runs ncclAllGather on the call's stream), or with HM_FLAG_LOCAL_GROUP a pointer to an int64 key
   shared by `world` ranks living in this process (one host thread per rank).  Setup is redundant
   on every rank (each keeps only its block rows for the hot path).  Returns HM_ERR_CUDA without a
   device, HM_ERR_NCCL if libnccl.so.2 cannot be opened or the communicator fails. */
hm_status hm_init(int device, int rank, int world, const void* comm_id, uint32_t flags,
                  hm_ctx** ctx);
/* 128-byte ncclUniqueId into id_out (rank 0 of a world > 1 job). */
hm_status hm_nccl_unique_id(void* id_out);
/* Self-test of the NCCL exchanger on one device: a one-rank communicator and the in-place
   ncclAllGather the sharded hot path issues, on `count` doubles, checked exactly.  HM_OK, or
   HM_ERR_NCCL (library missing, communicator or collective failed, data mismatch), HM_ERR_CUDA,
   HM_ERR_OOM, HM_ERR_INVALID_ARG (count < 1). */
hm_status hm_nccl_selftest(int device, int64_t count);
void hm_finalize(hm_ctx* ctx);
const char* hm_status_string(hm_status s);
const char* hm_last_error(const hm_ctx* ctx);
/* Change the call-mode flag HM_FLAG_ASYNC_PINNED after hm_init (0 clears it).  Any other bit:
   HM_ERR_INVALID_ARG (HM_FLAG_LOCAL_GROUP is fixed at hm_init). */
hm_status hm_set_flags(hm_ctx* ctx, uint32_t flags);
/* Optional device allocator hook (e.g. torch's caching allocator); NULL restores cudaMalloc. */
hm_status hm_set_allocator(hm_ctx* ctx, void* (*alloc_fn)(size_t bytes, void* stream, void* user),
                           void (*free_fn)(void* ptr, void* stream, void* user), void* user);

/* ---- setup (timed separately from the hot path) ------------------------------------- */
/* Facets: xyz = collocation points (n x 3), nrm = unit normals INTO the cavity (n x 3),
   area (n), facet_aabb = per-facet lo_xyz,hi_xyz (n x 6; required iff adm_mode == 1).
   Builds Alg. 1 (k-d split on the longest centroid-box axis, median by (coordinate, index),
   left child ceil(m/2)) and Alg. 2 (admissible -> low-rank leaf; a leaf cluster on either
   side -> dense leaf), flattened into level-ordered block lists. */
hm_status hm_build_geometry(hm_ctx* ctx, int64_t n, const double* xyz, const double* nrm,
                            const double* area, const double* facet_aabb,
                            const hm_tree_params* params, hm_geom** out);
/* Dense near field + batched partial-pivot ACA far field of F (eq:Fdef_new_location by the
   one-point centroid rule, or params->quadrature's adaptive Gauss rule), then
   (closed_cavity) row sums F_H 1 / A,
   clamp and row scaling. */
hm_status hm_assemble_aca(hm_ctx* ctx, const hm_geom* geom, const hm_aca_params* params,
                          hm_hmat** F_out);
/* One-time factorisation of C = I - Lambda F (Lambda_ii = (1-eps_i)/A_i, eq:reflection_matrix)
   in the block structure of F, stored for the solve form of params->cut_level (R27):
   W^L_t = L21 L11^-1, W^U_t = U12 U22^-1 per tree node t above the cut, and the inverse factors
   of the cut-level diagonal blocks (cut 0, default: L^-1 and U^-1), compressed to eps_lu in F's
   partition.  emissivity: host array, n, external order, 0 < eps_i <= 1.  params->method:
   hierarchical arithmetic (default, any n; host recursion, OpenMP tasks over independent blocks)
   or dense GPU tiles (HM_ERR_UNSUPPORTED above n ~ 1e5).  HM_ERR_SINGULAR on a leaf pivot below
   1e-14 of its block's largest entry.  Host-only contexts factor an F from hm_hmat_from_host and
   keep the factors for hm_export_factors.  The 4-step recursion, substitutions and truncation
   policy are PAPER.md:751-779. */
hm_status hm_factor_hlu(hm_ctx* ctx, const hm_hmat* F, const double* emissivity,
                        const hm_lu_params* params, hm_hlu** out);

/* ---- hot path ------------------------------------------------------------------------- */
/* y = F x, the H-matrix-vector product of PAPER.md:782 (F of eq:Fdef_new_location, PAPER.md:150-153,
   as stored: closed-cavity-scaled, the paper's convention without 1/A_i, reading R1).  x, y: n x nrhs, external order; x and y must not overlap. */
hm_status hm_apply_F(hm_ctx* ctx, const hm_hmat* F, int32_t nrhs, const double* x, double* y,
                     void* stream);
/* Host buffers (all hot-path calls): inputs are copied to the device on `stream` (a PINNED
   single-vector input of hm_apply_F / hm_solve_C / hm_radiative_flux is read by the program's own
   copy-in pass instead, world == 1); outputs in
   PINNED host memory are written by the kernels directly (device alias), pageable outputs are staged
   and copied back; with any host buffer the call synchronises `stream` before returning. */
/* z ~= C^-1 b by forward then backward substitution with the factors: level-
   scheduled W updates above the cut, then the cut-level inverse factors (R27). */
hm_status hm_solve_C(hm_ctx* ctx, const hm_hlu* LU, int32_t nrhs, const double* b, double* z,
                     void* stream);
/* q = sigma (eps/A) o (F C^-1 (eps o eta) - eta o g), eta = T^4, g = F C^-1 eps (cached at
   factor time): eq:qi_new_location in operator form (R16).
   T in K, q in W/m^2 (sigma = 5.670374419e-8, reading R2).  LU must have been
   factored from F. */
hm_status hm_radiative_flux(hm_ctx* ctx, const hm_hmat* F, const hm_hlu* LU, int32_t nrhs,
                            const double* T, double* q, void* stream);

/* Open cavities (F assembled with closed_cavity = 0): add the radiation to ambient of
   eqn:flux_to_ambient, B_N = sum_i int_{Gamma_i} (1 - c_i)(T^4 - T_inf^4) phi_N dS,
   with sigma and eps_i restored (reading R34): every later hm_radiative_flux on LU returns
   q_i + sigma eps_i (1 - c_i)(T_i^4 - T_inf^4), and hm_cavity_flux / hm_cavity_jacobian include the
   projected term (its T-derivative in the Jacobian).  c_i = clamped row sums of F (eq:clamped_rowsum,
   hm_export_row_sums).  enable = 0 removes the term.  HM_ERR_INVALID_ARG for a closed-cavity F or a
   negative / non-finite T_inf. */
hm_status hm_set_ambient(hm_ctx* ctx, hm_hlu* LU, int32_t enable, double T_inf);

/* ---- cavity operator around the hot path ------------------------ */
/* Facet <- node projection P (n_facets x n_nodes, PAPER.md:175-183 eqn:projection_operator,
   P_iM = (1/A_i) int_{Gamma_i} phi_M dS) as host CSR arrays in EXTERNAL facet order: row_ptr[n+1]
   (int64, row_ptr[0] = 0), col[nnz] node ids in [0, n_nodes), val[nnz].  The library copies them. */
hm_status hm_projection_create(hm_ctx* ctx, const hm_geom* geom, int64_t n_nodes, const int64_t* row_ptr,
                               const int32_t* col, const double* val, hm_proj** out);
void hm_destroy_projection(hm_proj* P);
/* Q = S eta with S = P^T Rbar P and eta_M = T_M^4 (eqn:flux_residual_3, eqn:S_def_matrix; R, Rbar of
   eq:Rdef / eq:Rbardef): Q_N = sum_i q_i A_i P_iN with q of eq:qi_new_location at eta = P T^4 -- one
   projection, one C^-1 solve, one F apply, one transpose projection.  T_nodes, Q_nodes: n_nodes x nrhs
   (device or host, as for hm_radiative_flux).  LU must have been factored from F, P built on F's
   geometry.  world > 1: nodal arrays are NOT sharded -- every rank passes all n_nodes values and
   receives the full Q (each rank reduces over its own facets; the node partials are allgathered and
   summed in rank order). */
hm_status hm_cavity_flux(hm_ctx* ctx, const hm_hmat* F, const hm_hlu* LU, hm_proj* P, int32_t nrhs,
                         const double* T_nodes, double* Q_nodes, void* stream);
/* y = J^cav x = 4 S (T^3 o x) (eq:Jcav): the action GMRES needs,
   without forming the dense n_nodes x n_nodes J^cav.  Same layout as hm_cavity_flux. */
hm_status hm_cavity_jacobian(hm_ctx* ctx, const hm_hmat* F, const hm_hlu* LU, hm_proj* P, int32_t nrhs,
                             const double* T_nodes, const double* x_nodes, double* y_nodes, void* stream);

/* ---- introspection (host buffers) ----------------------------------------------------- */
hm_status hm_export_perm(const hm_geom* geom, int32_t* perm /* n: perm[internal] = external */);
/* Per leaf block, sorted by (row_begin, col_begin), 8 int64 each:
   level, row_begin, row_end, col_begin, col_end, admissible, stored_kind (0 dense, 1 low-rank,
   2 admissible-but-dense), rank.  Call with rows == NULL to get n_blocks only.  F may be NULL
   (then stored_kind = !admissible ? 0 : 1 and rank = 0). */
hm_status hm_export_partition(const hm_geom* geom, const hm_hmat* F, int64_t* n_blocks,
                              int64_t* rows);
/* The stored blocks of one hot-path operator (host buffers), e.g. for the "apply is exact" check of
   PAPER.md:782.  op: HM_OP_F = F as stored (closed-cavity scaled); HM_OP_LINV / HM_OP_UINV = the
   inverse factors of the cut-level diagonal blocks (cut level 0: L^-1 and U^-1 of C, R27);
   HM_OP_WL(l) / HM_OP_WU(l) = the level-form blocks W^L_t / W^U_t of the tree nodes t of level l
   (l < cut level).  The operator is the SUM of the exported items (leaf-row slices of blocks on the
   GPU, whole blocks on a host-only context); rows and columns in internal order (hm_export_perm).
   Call with meta == NULL to get *n_items and *n_doubles, then with meta[6 n_items] =
   (row0, m, col0, n, kind, k) and data[n_doubles]: kind 0 = dense m x n column-major, kind 1 = U
   (m x k) followed by V (n x k), column-major (item = U V^T).  F or LU may be NULL when op does not
   need it.  HM_ERR_INVALID_ARG for an op the handles do not hold. */
#define HM_OP_F 0
#define HM_OP_LINV 1
#define HM_OP_UINV 2
#define HM_OP_WL(l) (3 + 2 * (l))
#define HM_OP_WU(l) (4 + 2 * (l))
hm_status hm_export_factors(const hm_hmat* F, const hm_hlu* LU, int32_t op, int64_t* n_items,
                            int64_t* n_doubles, int64_t* meta, double* data);
/* An F given by the caller in the block partition of geom (host-only contexts, device < 0): one entry
   per block of hm_export_partition's order, kind[b] = 0 dense (m x n column-major at data + offset[b])
   or 1 low rank (U m x k then V n x k column-major at data + offset[b], k = rank[b]), internal order,
   already closed-cavity scaled.  The library copies the payload.  It exists so the hierarchical H-LU
   can be driven and checked without a GPU (tests/test_hlu_host.py).  HM_ERR_UNSUPPORTED on a
   device context, HM_ERR_INVALID_ARG on a kind/rank/size mismatch. */
hm_status hm_hmat_from_host(hm_ctx* ctx, const hm_geom* geom, const int32_t* kind, const int32_t* rank,
                            const int64_t* offset, const double* data, hm_hmat** F_out);
/* Row sums s_i = (F_H 1)_i / A_i before scaling and clamped c_i (external order, n each). */
hm_status hm_export_row_sums(const hm_hmat* F, double* s, double* c);
hm_status hm_storage_report(const hm_hmat* F, const hm_hlu* LU, hm_storage* out);
/* Internal-order shard of `rank` among `world` ranks (tree node at level log2(world)). */
hm_status hm_local_range(const hm_geom* geom, int rank, int world, int64_t* begin, int64_t* end);
/* Shard plan for `world` ranks (host buffers): begin/end[world] internal row ranges, *maxc the padded
   segment length of the exchanged vectors, block_owner[n_blocks] (or NULL) the rank owning each block
   of hm_export_partition's order (-1: its rows straddle ranks). */
hm_status hm_shard_plan(const hm_geom* geom, int world, int64_t* begin, int64_t* end, int64_t* maxc,
                        int64_t* block_owner);

/* ---- measurement support (bench.py) ---------------------------------------------------- */
/* Times the hot-path programs with CUDA events on `stream` (device pointers T, q; nrhs = 1) over
   `iters` calls each: ms_out[0] = hm_radiative_flux, ms_out[1] = hm_apply_F, ms_out[2] =
   hm_solve_C (per call; ONE launch of the persistent stream engine at world 1, one launch per
   segment plus the allgathers between them when sharded); ms_out[3] = sharded only: the flux
   segments with their allgathers skipped (compute-only time for the communication share; the
   results of those calls are not valid), else 0; ms_out[4..5] = 0.  launches_out[0..2] = kernel
   launches per call (1, or the segment count when sharded); launches_out[3] = passes of the flux
   program, [4] = its work units, [5] = its grid size. */
hm_status hm_profile_flux(hm_ctx* ctx, const hm_hmat* F, const hm_hlu* LU, const double* T,
                          double* q, int32_t iters, double* ms_out, int64_t* launches_out,
                          void* stream);

/* Per-pass timeline of one hm_radiative_flux call (device pointers, nrhs = 1), from %globaltimer
   stamps inside the engine: t_begin_us[p] = first input gather of pass p, t_end_us[p] = last task
   retirement, both relative to the earliest pass start; pass_bytes[p] = factor payload bytes of
   pass p.  Arrays have max_passes entries; *n_passes receives the program's pass count. */
hm_status hm_trace_flux(hm_ctx* ctx, const hm_hmat* F, const hm_hlu* LU, const double* T, double* q,
                        int32_t max_passes, int32_t* n_passes, double* t_begin_us, double* t_end_us,
                        int64_t* pass_bytes, void* stream);

void hm_destroy_geom(hm_geom* geom);
void hm_destroy_hmat(hm_hmat* F);
void hm_destroy_hlu(hm_hlu* LU);

#ifdef __cplusplus
}
#endif
#endif /* HM_H_ */
