/* =====================================================================================
 *  f3m.h -- C ABI of the B200-native F^3M kernel matrix-vector product (sm_100a)
 * =====================================================================================
 *  Problem (Sec. 1 "Notations"; Sec. 2):
 *      v = k(X, Y) . b,   X in R^{nx x D},  Y in R^{ny x D},  b in R^{ny},
 *      k(x, y) = exp(-||x - y||^2 / (2 gamma^2))           (Sec. 5)
 *  approximated by F^3M (App. F Algorithm 1): hierarchical binning
 *  (Sec. 4.1-4.2), far/smooth interpolation with Chebyshev-Lagrange nodes (Sec. 3, 4.3:
 *  S2M = L_Y b, M2L = K v1, L2T = L_X^T v2), exact near/small field
 *  (Sec. 3 Eq. (1), Sec. 4.2).
 *
 *  Conventions (every entry point):
 *   * X, Y: row-major [n x D] contiguous fp32 (a torch [n, D] tensor).  1 <= D <= 7.
 *     Y == NULL selects the k(X, X) case (then ny must equal nx).
 *   * Pointers are DEVICE pointers unless stated otherwise; f3m_matvec also accepts
 *     HOST pointers for X, Y, b, v (auto-detected; staged through device memory on the
 *     given stream -- the "e2e" path).  The library never retains caller pointers
 *     past return and never frees them.
 *   * All device work is enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default).
 *     Calls synchronise that stream before returning (the plan is data dependent:
 *     box counts are read back to build the interaction lists).
 *   * Workspace: allocated with cudaMallocAsync on `cuda_stream` (stream-ordered pool)
 *     and released before return, unless an f3m_allocator is supplied.
 *   * Errors: every function returns f3m_status.  On failure the output is unspecified
 *     and f3m_last_error() returns a thread-local message (valid until the next call on
 *     that thread).  A resource error names the tree depth it happened at.
 *   * Limits: nx, ny < 2^31 per call (int32 permutations); the node grid P^D <= node_cap.
 * ===================================================================================== */
#ifndef F3M_H_
#define F3M_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define F3M_API __attribute__((visibility("default")))
#else
#define F3M_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  F3M_OK = 0,
  F3M_ERR_INVALID_INPUT = 2,    /* bad shape, non-finite coordinate, bad pointer */
  F3M_ERR_RESOURCE = 3,         /* device allocation failed (message carries the depth) */
  F3M_ERR_INTERNAL = 4,         /* internal consistency check failed (a bug) */
  F3M_ERR_INVALID_SPEC = 5,     /* gamma <= 0, P < 2, eta <= 0, rho < 0, zeta < 1 */
  F3M_ERR_GRID_TOO_LARGE = 6,   /* P^D > node_cap ("a cap at r = 2048") */
  F3M_ERR_CUDA = 7              /* a CUDA runtime error (message has the CUDA string) */
} f3m_status;

typedef enum { F3M_KERNEL_GAUSSIAN = 0 } f3m_kernel_kind;

/* Kernel spec: Gaussian with lengthscale gamma > 0, finite. */
typedef struct {
  int32_t kind;        /* f3m_kernel_kind */
  double lengthscale;  /* gamma */
} f3m_kernel;

/* Ablation flags (Tables 5-6). */
#define F3M_EXACT        1u   /* no division: the exact direct sum (exact mode) */
#define F3M_NO_SMOOTH    2u   /* disable the smoothness criterion (Sec. 4.3) */
#define F3M_NO_ADAPTIVE  4u   /* far pairs always use P nodes (Sec. 4.3 rule off) */
#define F3M_NO_SMALL     8u   /* disable the small field (Sec. 4.2) */
#define F3M_NO_DROP     16u   /* far pairs the adaptive rule would drop use P nodes */
#define F3M_ADMISSIBLE_MAXNORM 32u  /* far iff max_d |c_p - c_q|_d >= 2l instead of the Euclidean
                                       ||c_p - c_q|| >= 2l of PAPER.md:135: at D >= 4
                                       corner-touching boxes are then not far */
#define F3M_KEEP_EMPTY  64u   /* no empty-box removal (the FFM(GPU) ablation of Tables 5-6, PAPER.md:368-427;
                                 Fig. 5): every divided box keeps all 2^D children, empty
                                 ones included; same v, more interactions.  Needs D * T_sort <= 24. */

/* Method parameters (defaults from f3m_default_config, Table 2). */
typedef struct {
  int32_t nodes_per_dim;  /* P >= 2 Chebyshev nodes per dimension; m = P^D ("r" of Sec. 5) */
  int32_t node_cap;       /* P^D <= node_cap; default 2048 */
  double eta;             /* effective-variance limit (Sec. 4.3), > 0; default 0.5 */
  int64_t rho;            /* small-field threshold (Sec. 4.2), >= 0; < 0 -> 2 P^D */
  int64_t zeta;           /* max-box-size threshold of Alg. 1, >= 1; < 1 -> P^D */
  int32_t max_depth;      /* cap on the tree depth; < 0 -> floor(63/D) */
  uint32_t flags;         /* F3M_* ablation flags */
  int32_t sparse_level;   /* 0: the P^D tensor grid; q in [1, 3]: the level-q Smolyak sparse grid
                             (Sec. 4.2 "Sparse grids"; reading R27: combination
                             technique over nested Chebyshev levels, |H| nodes per box, |H| <=
                             node_cap replaces the P^D cap).  P still drives the adaptive rule
                             (far pairs with P_far < P use the largest level with |H| <= 3^D). */
} f3m_config;

#define F3M_MAX_LEVELS 64
/* Per-call statistics (host memory).  Arrays are indexed by depth t = 0..63 (Thm. 2,
 * PAPER.md:275-281): M = surviving child pairs, expanded = 4^D x |I_near(t-1)|,
 * m_far (incl. dropped), m_far_dropped, m_smooth, m_small, m_near, boxes_* = active
 * children, empty_* = removed empty children, pfar = adaptive node count. */
typedef struct {
  int32_t depth_reached, t_star, t_sort, num_sort_passes;
  double E;                        /* enclosing-cube edge */
  int64_t M[F3M_MAX_LEVELS], expanded[F3M_MAX_LEVELS], m_far[F3M_MAX_LEVELS],
          m_far_dropped[F3M_MAX_LEVELS], m_smooth[F3M_MAX_LEVELS], m_small[F3M_MAX_LEVELS],
          m_near[F3M_MAX_LEVELS], boxes_x[F3M_MAX_LEVELS], boxes_y[F3M_MAX_LEVELS],
          empty_x[F3M_MAX_LEVELS], empty_y[F3M_MAX_LEVELS], pfar[F3M_MAX_LEVELS];
  int64_t n_near_flushed;          /* near pairs summed exactly at loop exit */
  int64_t s2m_points, l2t_points;  /* source / target points processed by S2M / L2T (all groups) */
  int64_t near_pairs;              /* point pairs summed exactly (small + near field) */
  int32_t far_groups_local;        /* far (depth, P') groups run by the tile-local kernels */
  int32_t far_groups_sorted;       /* far groups run on the globally sorted points */
  int32_t kernel_launches;         /* number of library kernels launched by the call */
  int32_t m2l_grid_groups;         /* far groups whose M2L ran as Kronecker mode products over a
                                      complete level (same pairs, reading R29) */
  int64_t m2l_grid_fma;            /* fp64 FMAs of those mode products */
  int64_t m2l_grid_pairs;          /* far / smooth box pairs those groups cover */
  float ms_phase[16];              /* optional per-phase times (F3M_TIMING env), see f3m_phase_name */
} f3m_stats;

/* Optional caller allocator (e.g. the PyTorch caching allocator).  alloc returns a
 * device pointer of >= bytes (256-byte aligned) usable on `stream`, or NULL. */
typedef struct {
  void* ctx;
  void* (*alloc)(void* ctx, size_t bytes, void* stream);
  void (*free)(void* ctx, void* ptr, void* stream);
} f3m_allocator;

/* Fill *out with the defaults for dimension D: P = 4, node_cap = 2048, eta = 0.5,
 * rho = 2 P^D, zeta = P^D, max_depth = floor(63/D), flags = 0, sparse_level = 0. */
F3M_API f3m_status f3m_default_config(int32_t D, f3m_config* out);

/* The F^3M KMVM (Alg. 1).  v [nx] is overwritten in X's row order (sigma).
 * b has ny entries.  alloc may be NULL; stats may be NULL. */
F3M_API f3m_status f3m_matvec(const float* X, int64_t nx, const float* Y, int64_t ny, int32_t D,
                      const float* b, float* v, const f3m_kernel* k, const f3m_config* cfg,
                      const f3m_allocator* alloc, void* cuda_stream, f3m_stats* stats);

/* Exact KMVM v = k(X, Y) b by a KeOps-style tiled map-reduce: fp32
 * evaluation with fp64 cross-tile accumulation when fp64 == 0 (v is float*), full fp64
 * evaluation and accumulation when fp64 != 0 (v is double*).  Device pointers. */
F3M_API f3m_status f3m_direct(const float* X, int64_t nx, const float* Y, int64_t ny, int32_t D,
                      const float* b, void* v, int32_t fp64, const f3m_kernel* k, void* cuda_stream);

/* ---- Plan API: the same algorithm split at its data-dependent points, for sharding
 * targets across ranks (App. G's k(X, X) split).  Rank g owns
 * the row slice Xlocal of X (= Y) as its targets and its S2M sources.  The caller runs the
 * collectives between the calls (torch.distributed / NCCL):
 *   1. f3m_plan_bbox       -> all_reduce MIN of the minima, MAX of the maxima   (Sec. 3 cube)
 *   2. f3m_plan_leaves     -> all_gather of every rank's sparse (key, count) leaf list
 *      f3m_plan_set_leaves <- the concatenation: every rank builds the identical tree (Alg. 1,
 *                             empty-box removal, zeta / rho decisions from the GLOBAL counts)
 *   3. f3m_plan_s2m        -> all_reduce SUM of the fp64 node charges (v1 = L_Y b is linear)
 *   4. f3m_plan_evaluate   <- M2L (replicated), L2T + near field on the local targets.
 * The near / small field (Sec. 4.2, Alg. 1 last line) needs the sources of every rank: pass
 * the replicated full source set Yfull [ny x D] / bfull [ny] (device); they are sorted only
 * when the tree has near / small pairs, and may be NULL when the caller knows it has none
 * (then such a tree returns F3M_ERR_INVALID_INPUT).  Deviation from SURVEY 8(b): blocal is
 * given at create, not at f3m_plan_s2m, because the counting sort of stage 2 is fused with the
 * speculative leaf-level S2M (one pass over X and b instead of two).
 * All pointers are device pointers; the library keeps Xlocal, blocal, Yfull, bfull
 * referenced until f3m_plan_destroy. */
typedef struct f3m_plan f3m_plan;

/* Ylocal: NULL or Xlocal (the sharded flow is the k(X, X) case; ny_local must then equal
 * nx_local).  alloc may be NULL (stream-ordered cudaMallocAsync); it is copied. */
F3M_API f3m_status f3m_plan_create(const float* Xlocal, int64_t nx_local, const float* Ylocal, int64_t ny_local,
                                   const float* blocal, const float* Yfull, const float* bfull, int64_t ny, int32_t D,
                                   const f3m_kernel* k, const f3m_config* cfg, const f3m_allocator* alloc,
                                   void* cuda_stream, f3m_plan** out);
/* Local per-dimension [min_0..min_{D-1}, max_0..max_{D-1}] as fp64 (host array of 2D);
 * non-finite coordinates return F3M_ERR_INVALID_INPUT. */
F3M_API f3m_status f3m_plan_bbox(f3m_plan* p, double* minmax_host);
/* Set the GLOBAL bbox (host [2D]); computes the keys, sorts the local points and returns this
 * rank's non-empty leaves at depth T_sort as a sparse list: keys (uint64, ascending) and point
 * counts (int64), *len entries, library-owned device arrays valid until the next call. */
F3M_API f3m_status f3m_plan_leaves(f3m_plan* p, const double* global_minmax_host, uint64_t** keys_dev,
                                   int64_t** counts_dev, int64_t* len);
/* The concatenation of every rank's leaf lists (device or host arrays, any order; equal keys
 * are summed): builds the global leaf table and the interaction lists. */
F3M_API f3m_status f3m_plan_set_leaves(f3m_plan* p, const uint64_t* keys, const int64_t* counts, int64_t len);
/* S2M on the local points; returns the LOCAL charges (fp64, device, *len values) to
 * SUM-all-reduce in place. */
F3M_API f3m_status f3m_plan_s2m(f3m_plan* p, double** charges_dev, int64_t* len);
/* M2L on the (global) charges, L2T + near field on the local targets; writes v [nx_local] in
 * the local row order (device). */
F3M_API f3m_status f3m_plan_evaluate(f3m_plan* p, float* v, f3m_stats* stats);
F3M_API void f3m_plan_destroy(f3m_plan* p);

/* ---- Operator API: plan reuse across right-hand sides (the KRR / CG use of
 * Sec. 5, applies the same k(X, X) to many b).  Everything that does not
 * depend on b -- the cube, keys, the counting sort's histogram and per-tile orders, the box
 * tables and the interaction lists (Alg. 1) -- is built once; each apply runs S2M (from the
 * stored tile orders, no re-ranking), M2L and L2T only.  Configurations outside the
 * single-pass tile-local path (D T_sort > 8, a near/small field, sorted far levels, k(X, Y))
 * keep no state: every apply then runs the whole method (f3m_matvec) -- same result either
 * way.  EXCEPTION to the conventions above: X (and Y) are referenced, not copied; they must
 * stay valid and unchanged on the device until f3m_op_destroy.  Device pointers only. */
typedef struct f3m_op f3m_op;
F3M_API f3m_status f3m_op_create(const float* X, int64_t nx, const float* Y, int64_t ny, int32_t D,
                                 const f3m_kernel* k, const f3m_config* cfg, void* cuda_stream, f3m_op** out);
/* v [nx] = F^3M(k(X, Y)) b for b [ny] (device); stream NULL -> the creation stream. */
F3M_API f3m_status f3m_op_apply(f3m_op* op, const float* b, float* v, void* cuda_stream, f3m_stats* stats);
/* nrhs right-hand sides: column r of B (b_r = B + r ldb, ny entries) gives column r of V
 * (v_r = V + r ldv, nx entries); each column reuses the plan (device pointers). */
F3M_API f3m_status f3m_op_apply_batch(f3m_op* op, const float* B, int64_t ldb, int32_t nrhs, float* V, int64_t ldv,
                                      void* cuda_stream, f3m_stats* stats);
/* 1 when applies reuse the stored plan (tile-local path), 0 when each apply recomputes it. */
F3M_API int32_t f3m_op_reuses_plan(const f3m_op* op);
F3M_API void f3m_op_destroy(f3m_op* op);

/* ---- Introspection (parity tests): after f3m_matvec_debug the library keeps the last
 * call's sorted permutation and keys; copy them out (host arrays, int64 / uint64). */
F3M_API f3m_status f3m_debug_last_perm(int32_t side, int64_t* perm_host, int64_t n);
F3M_API f3m_status f3m_debug_last_keys(int32_t side, uint64_t* keys_sorted_host, int64_t n);
/* Number of classified pairs at depth t in the last call, and their (key_p, key_q, tag)
 * with tag 0 near, 1 far, 2 far dropped, 3 smooth, 4 small (host arrays). */
F3M_API int64_t f3m_debug_num_pairs(int32_t t);
F3M_API f3m_status f3m_debug_pairs(int32_t t, uint64_t* kp, uint64_t* kq, int32_t* tag);
/* Charges (stage 1) / locals (stage 2) of charge set i of the last call (host, fp64):
 * info = [t, P, nsrc, ntgt, m, q] (m nodes per box; q > 0: sparse-grid level, P = 2^q + 1). */
F3M_API int32_t f3m_debug_num_charge_sets(void);
F3M_API f3m_status f3m_debug_charge_info(int32_t i, int64_t* info);
F3M_API f3m_status f3m_debug_charges(int32_t i, uint64_t* src_key, double* W, uint64_t* tgt_key, double* U);
/* Enable (1) / disable (0) keeping debug state (costs extra device->host copies).  Level 2
 * (full-size tests) keeps the pair lists, the charges and pi of X only, as int32. */
F3M_API void f3m_debug_enable(int32_t on);
/* pi of X (sorted position -> original row) of the last level-2 call; n must equal nx. */
F3M_API f3m_status f3m_debug_last_perm32(int32_t* perm_host, int64_t n);

F3M_API const char* f3m_last_error(void);
F3M_API const char* f3m_version(void);
F3M_API const char* f3m_phase_name(int32_t i);

#ifdef __cplusplus
}
#endif
#endif /* F3M_H_ */
