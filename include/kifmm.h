/*
 * kifmm.h — C ABI of the B200-native KIFMM evaluate library (libkifmm_b200.so).
 *
 * The reference (arxiv 2303.08394 / PyExaFMM, restated as SPEC.md) has no
 * plugin or FFI surface of its own; its embedded-library contract is
 * "construct config, call run", where `run`
 * builds the tree and lists on the host and then executes the evaluate
 * sequence "zero state -> upward pass -> downward pass -> permute back"
 * over immutable tree/lists/operator cache.
 *
 * This header exports:
 *   1. the host-side modules the evaluate consumes (morton SPEC.md:24-126,
 *      kernel SPEC.md:282-346, surface SPEC.md:348-400, tree SPEC.md:128-203,
 *      interaction_lists SPEC.md:205-280, operators/precompute SPEC.md:413-428),
 *      implemented in C++ (the reference's intended language, CMakeLists.txt:2-5);
 *   2. the GPU evaluate boundary (kifmm_gpu_*), which replaces the evaluate
 *      section of `run` with hand-written sm_100a kernels.
 *
 * Rules at the boundary: C linkage only; no C++ types or exceptions cross it;
 * every failure returns a kifmm_status and sets a thread-local message readable
 * through kifmm_last_error().  Status codes map 1:1 onto the reference error
 * taxonomy of proj/src/common.hpp:19-49.
 */
#ifndef KIFMM_H_
#define KIFMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */

typedef enum kifmm_status {
  KIFMM_OK = 0,
  KIFMM_E_INVALID_ARGUMENT = 1, /* common.hpp:21 InvalidArgument            */
  KIFMM_E_IO = 2,               /* common.hpp:27 IoError                    */
  KIFMM_E_NUMERICAL = 3,        /* common.hpp:33 NumericalError             */
  KIFMM_E_CUDA = 4,             /* device error (new; DeviceError on C++ side) */
  KIFMM_E_NCCL = 5,             /* collective error (new)                   */
  KIFMM_E_OUT_OF_MEMORY = 6,    /* device allocation failed (new)           */
  KIFMM_E_CACHE_MISMATCH = 7,   /* common.hpp:40 CacheMismatch              */
  KIFMM_E_CORRUPT_ARCHIVE = 8,  /* common.hpp:46 CorruptArchive             */
  KIFMM_E_INTERNAL = 9
} kifmm_status;

/* Thread-local message of the last failing call on this thread. */
const char* kifmm_last_error(void);
/* Library version string. */
const char* kifmm_version(void);

/* ------------------------------------------------------------------ morton
 * SPEC.md:24-126.  Key layout (pinned per SPEC.md:125): level in
 * bits 0..3; bits 4..48 hold the bit-interleaved anchor scaled to the
 * MAX_LEVEL grid (x -> bit 3i, y -> 3i+1, z -> 3i+2).  Raw order at a fixed
 * level is Z-order; across levels raw order is spatial Z-order with ancestors
 * first (resolves SURVEY Appendix C3). */
#define KIFMM_MAX_LEVEL 15

kifmm_status kifmm_morton_encode(const uint32_t anchor[3], int32_t level, uint64_t* out);
kifmm_status kifmm_morton_decode(uint64_t key, uint32_t anchor[3], int32_t* level);
kifmm_status kifmm_morton_parent(uint64_t key, uint64_t* out);
kifmm_status kifmm_morton_children(uint64_t key, uint64_t out[8]);
/* same-level neighbours (corners included), ascending raw. Returns count. */
int32_t kifmm_morton_neighbors(uint64_t key, uint64_t out[26]);
/* closed cubes touch and neither contains the other. */
int32_t kifmm_morton_is_adjacent(uint64_t a, uint64_t b);
/* SPEC.md:94 */
void kifmm_morton_node_bounds(uint64_t key, const double origin[3], double side,
                              double center[3], double* half_side);

/* ------------------------------------------------------------------ kernel
 * laplace = 1/(4 pi |x-y|), exactly 0 at |x-y| = 0. */
double kifmm_laplace(const double x[3], const double y[3]);
/* out[j*m + i] = laplace(sources_i, targets_j); sources m x 3, targets k x 3. */
void kifmm_kernel_matrix(const double* sources, int64_t m, const double* targets, int64_t k,
                         double* out);

/* ----------------------------------------------------------------- surface
 * boundary points of the p^3 grid on [-1,1]^3, lexicographic. */
int32_t kifmm_surface_count(int32_t p); /* 6(p-1)^2+2, or -1 for p < 2 */
kifmm_status kifmm_surface_grid(int32_t p, double* out /* n x 3 */);

/* -------------------------------------------------------------------- tree
 * adaptive n_crit octree, 2:1 balance, U/V/W/X lists. */
typedef struct kifmm_tree kifmm_tree;

typedef struct kifmm_tree_view {
  int64_t n_particles;
  int32_t depth;            /* deepest level holding a node */
  int32_t n_overfull;       /* leaves at MAX_LEVEL holding > n_crit (SPEC.md:153 warning) */
  int64_t n_leaves;
  int64_t n_nodes;
  double origin[3];         /* Domain */
  double side;
  const double* positions;        /* N x 3, reordered (leaf-contiguous) */
  const int64_t* original_index;  /* N: reordered slot -> input index */
  const uint64_t* node_key;       /* n_nodes, level-major, ascending raw within a level */
  const int64_t* level_ptr;       /* depth + 2: nodes of level l are [level_ptr[l], level_ptr[l+1]) */
  const int64_t* node_parent;     /* n_nodes, -1 for the root */
  const int64_t* node_children;   /* n_nodes x 8, octant order, -1 absent */
  const int64_t* node_leaf;       /* n_nodes -> leaf index or -1 */
  const int64_t* leaf_node;       /* n_leaves -> node index; leaves in ascending raw key */
  const int64_t* leaf_ptr;        /* n_leaves + 1 particle offsets */
  /* Interaction lists in CSR; members in ascending raw key. */
  const int64_t* u_ptr;  const int64_t* u_idx;  /* per leaf; members are leaf indices  */
  const int64_t* v_ptr;  const int64_t* v_idx;  /* per node; members are node indices  */
  const int32_t* v_tv;                          /* per V entry: transfer-vector id 0..315 */
  const int64_t* w_ptr;  const int64_t* w_idx;  /* per leaf; members are node indices  */
  const int64_t* x_ptr;  const int64_t* x_idx;  /* per NODE; members leaf indices */
} kifmm_tree_view;

/* positions: n x 3 row-major (input order).  domain: {origin[3], side} or NULL
 * for the tight bounding cube with a 1e-10 relative margin.
 * balance: 1 = 2:1 balance, 0 = skip (test hook). threads: 0 = all. */
kifmm_status kifmm_tree_build(const double* positions, int64_t n, int32_t n_crit,
                              const double* domain, int32_t balance, int32_t threads,
                              kifmm_tree** out);
kifmm_status kifmm_tree_get_view(const kifmm_tree* tree, kifmm_tree_view* view);
void kifmm_tree_destroy(kifmm_tree* tree);

/* Transfer vector table: id -> (dx,dy,dz), the 316 offsets of [-3,3]^3 with
 * Chebyshev norm >= 2 in lexicographic (dx slowest) order. */
int32_t kifmm_transfer_vectors(int32_t out[316 * 3]);

/* Contiguous Z-order leaf ranges per rank for multi-GPU, balanced
 * by estimated cost and aligned to level-`cut_level` boxes (0 = auto, see
 * kifmm_halo_plan). leaf_begin has world_size + 1 entries. */
kifmm_status kifmm_partition_leaves(const kifmm_tree_view* tree, int32_t n_e, int32_t gradient,
                                    int32_t world_size, int32_t cut_level, int64_t* leaf_begin);

/* Halo-exchange tables of the multi-GPU evaluate, built on the host (no device needed)
 * and used by kifmm_gpu_plan_create for world_size > 1.  Rank r owns leaves
 * [leaf_begin[r], leaf_begin[r+1]) (ranges aligned to level-cut_level boxes; cut_level 0 = auto: the
 * coarsest level >= 2 that balances the estimated cost within 5 %) and computes the multipoles of the
 * nodes with up_owner == r, i.e. whose leaves all lie in its range; the few nodes spanning ranks
 * (up_owner == -1) are recomputed by every rank from their children.  After the upward pass each rank r contributes the
 * rows export_idx[export_ptr[r] .. export_ptr[r+1]) -- the multipoles it owns that another rank reads
 * (V lists of its targets, W lists of its leaves, children of the redundant top nodes) -- to an
 * all-gather of world_size slots of max_export rows each. */
typedef struct kifmm_halo kifmm_halo;
typedef struct kifmm_halo_view {
  int32_t world_size, cut_level;
  int64_t n_nodes;
  const int64_t* leaf_begin;  /* world_size + 1 */
  const int32_t* up_owner;    /* n_nodes */
  const int64_t* export_ptr;  /* world_size + 1 */
  const int64_t* export_idx;  /* export_ptr[world_size] node indices, ascending within a rank */
  int64_t max_export;         /* rows per all-gather slot */
} kifmm_halo_view;
kifmm_status kifmm_halo_plan(const kifmm_tree_view* tree, int32_t n_e, int32_t gradient, int32_t world_size,
                             int32_t cut_level, kifmm_halo** out);
kifmm_status kifmm_halo_get_view(const kifmm_halo* halo, kifmm_halo_view* view);
void kifmm_halo_destroy(kifmm_halo* halo);

/* --------------------------------------------------------------- operators
 * SPEC.md:413-428, design 501-504.  Pseudo-inverses are stored FACTORED
 * (U_k, sigma_k, V_k): pinv = V diag(1/sigma) U^T, never densified. */
typedef struct kifmm_operators kifmm_operators;

typedef struct kifmm_operator_view {
  int32_t p, n_e, n_c;
  int32_t reference_level;   /* 2 */
  double alpha_inner, alpha_outer, svd_cutoff;
  double domain_side;
  double ref_half_side;      /* half side of a reference-level node = side / 2^(ref+1) */
  const double* surface;     /* n_e x 3 unit grid */
  int32_t uc2e_rank;
  const double* uc2e_u;      /* n_c x k */
  const double* uc2e_s;      /* k */
  const double* uc2e_v;      /* n_e x k */
  int32_t dc2e_rank;
  const double* dc2e_u;
  const double* dc2e_s;
  const double* dc2e_v;
  const double* m2m;         /* 8 x n_e x n_e: parent_i += m2m[o][i][j] child_j */
  const double* l2l;         /* 8 x n_e x n_e: child_i  += l2l[o][i][j] parent_j */
  int32_t n_m2l;             /* 316 */
  const double* m2l;         /* n_m2l x n_c x n_e kernel matrices K_t at the reference level */
  uint64_t fingerprint;      /* over (p, alphas, cutoff, side, kernel) SPEC.md:414 */
} kifmm_operator_view;

kifmm_status kifmm_precompute(int32_t p, double alpha_inner, double alpha_outer,
                              double svd_cutoff, double domain_side, int32_t threads,
                              kifmm_operators** out);
kifmm_status kifmm_operators_get_view(const kifmm_operators* ops, kifmm_operator_view* view);
void kifmm_operators_destroy(kifmm_operators* ops);
/* Persistence: manifest + 64-byte aligned LE f64 payload. */
kifmm_status kifmm_operators_save(const kifmm_operators* ops, const char* path);
kifmm_status kifmm_operators_load(const char* path, uint64_t expected_fingerprint,
                                  kifmm_operators** out);
/* Symmetric one-sided Jacobi SVD used by precompute (exported for tests):
 * a is m x n row-major (m >= n); u m x n, s n (descending), v n x n. */
kifmm_status kifmm_svd(const double* a, int32_t m, int32_t n, double* u, double* s, double* v);

/* --------------------------------------------------------------------- GPU
 * The evaluate boundary.  A plan owns all device state: the
 * uploaded tree/lists/operators, expansion buffers, streams, the optional
 * NCCL communicator and the captured CUDA graph.  Not thread-safe: one caller
 * at a time per plan; distinct plans may run concurrently. */
typedef struct kifmm_gpu_plan kifmm_gpu_plan;

typedef struct kifmm_gpu_options {
  int32_t precision;      /* 32 or 64 */
  int32_t gradient;       /* 1: also produce grad(phi) (extension, SPEC.md:581 non-goal) */
  int32_t device;         /* CUDA ordinal */
  int32_t rank;           /* multi-GPU: this process's rank (one process per GPU) */
  int32_t world_size;     /* 1 = single GPU */
  int32_t cut_level;      /* partition alignment level for world_size > 1 (0 = auto, kifmm_halo_plan) */
  const void* nccl_unique_id; /* 128 bytes from kifmm_gpu_nccl_unique_id() on rank 0 */
  int32_t m2l_backend;    /* 0 auto, 1 SIMT (fp32) / DMMA (fp64), 2 tcgen05 (fp32 only; n_e padded to 64,
                             128, 160 or 224, i.e. p = 4..7 -- the fp32 default there; at p = 7 the M2L
                             alone, solves / M2M / L2L stay on the SIMT GEMM): kind::f16
                             3-term fp16 split by default -- reported as 2 -- or kind::tf32 3xTF32 with
                             KIFMM_TC_KIND=tf32 (p = 6 only) -- reported as 3; 4 tcgen05 kind::i8 (fp64 only, n_e
                             padded to 160 or 224, i.e. p = 6, 7): Ozaki scheme, 8 int8 digit slices per
                             operand, exact int32 accumulation -- the fp64 default where supported */
  int32_t use_graph;      /* capture the evaluate in a CUDA graph */
  int32_t exchange;       /* world_size > 1: 0 = NCCL all-gather inside the evaluate (one process per GPU);
                             1 = host: the caller moves the halo rows between kifmm_gpu_evaluate_upward and
                             kifmm_gpu_evaluate_downward (no NCCL; e.g. ranks emulated by one process) */
} kifmm_gpu_options;

typedef struct kifmm_gpu_timings {
  float total_ms;      /* whole evaluate on the device (events) */
  float upload_ms;     /* H2D charges (+ permutation) */
  float p2m_ms;        /* P2M check + solve */
  float m2m_ms;
  float exchange_ms;   /* NCCL all-gather of multipoles */
  float p2l_ms;
  float m2l_ms;
  float down_solve_ms;
  float l2l_ms;
  float leaf_ms;       /* near field + L2P + M2P */
  float download_ms;   /* D2H potentials (+ permutation) */
  float upward_ms;     /* device time of the last kifmm_gpu_evaluate_upward (without its host copies) */
  float downward_ms;   /* device time of the last kifmm_gpu_evaluate_downward (without its host copies) */
} kifmm_gpu_timings;

typedef struct kifmm_gpu_plan_info {
  int64_t n_particles, n_leaves, n_nodes;
  int64_t owned_leaf_begin, owned_leaf_end;
  int64_t owned_particle_begin, owned_particle_end;
  int64_t near_pairs;       /* sum over owned leaves of n_t * sum_{s in U} n_s */
  int64_t l2p_pairs, m2p_pairs, p2m_pairs, p2l_pairs;
  int64_t m2l_pairs;        /* V-list entries evaluated by this rank */
  int64_t m2l_padded_pairs; /* tile-slots actually computed (incl. zero rows) */
  int32_t n_e, n_c, ne_pad;
  int32_t m2l_backend;      /* backend actually used */
  int64_t device_bytes;     /* device memory held by the plan */
  int32_t kernel_launches;  /* kernels launched per evaluate */
  int64_t halo_rows_max;    /* world_size > 1: rows per all-gather slot (kifmm_halo_view.max_export) */
  int64_t halo_rows_mine;   /* rows this rank exports */
  /* call structure (SPEC acceptance #8): tree levels each level-by-level operator covers -- M2M at the
   * parent levels >= 2 (the multipoles of levels 0-1 feed no operator), M2L at every target level >= 2 in
   * ONE batched launch, L2L at the child levels >= 3 -- and the leaves / nodes each per-target operator
   * is applied to (each exactly once) */
  int32_t m2m_levels, m2l_levels, l2l_levels, m2l_launch_levels;
  int64_t p2m_leaves, near_leaves, l2p_leaves, m2p_leaves, p2l_nodes;
} kifmm_gpu_plan_info;

kifmm_status kifmm_gpu_plan_create(const kifmm_gpu_options* options, const kifmm_tree_view* tree,
                                   const kifmm_operator_view* ops, kifmm_gpu_plan** out);
/* Host buffers.  input_order = 1: charges/potential/gradient are in the caller's
 * input order and the (un)permutation runs on the device; 0: reordered order.
 * charges/potential are fp32 or fp64 per options.precision; gradient is N x 3 or NULL.
 * With world_size > 1 every rank passes the full charge vector and receives the potentials of its
 * own particles: with input_order = 1 the other ranks' entries are written as 0 (sum the ranks'
 * outputs, or take each rank's owned slice, to assemble the result); with input_order = 0 only this
 * rank's contiguous reordered range [owned_particle_begin, owned_particle_end) is written and the rest
 * of the caller's buffer is left untouched. */
kifmm_status kifmm_gpu_evaluate(kifmm_gpu_plan* plan, const void* charges, void* potential,
                                void* gradient, int32_t input_order, kifmm_gpu_timings* timings);
/* n_rhs independent charge vectors through one plan (host buffers, as kifmm_gpu_evaluate;
 * pinned buffers let the copies overlap): H2D of vector k+1 and D2H of the results of k-1 run
 * under the evaluate of k on separate streams.  gradients may be NULL (or hold NULL entries)
 * when no gradient is wanted.  Synchronous: returns when every result is in host memory.
 * No reference counterpart (the reference's `run` takes one charge vector). */
kifmm_status kifmm_gpu_evaluate_many(kifmm_gpu_plan* plan, int32_t n_rhs, const void* const* charges,
                                     void* const* potentials, void* const* gradients, int32_t input_order);
/* Device buffers on the plan's device; runs on `stream` (cudaStream_t or NULL
 * for the plan's stream) and does not synchronise. */
kifmm_status kifmm_gpu_evaluate_device(kifmm_gpu_plan* plan, const void* d_charges,
                                       void* d_potential, void* d_gradient, int32_t input_order,
                                       void* stream);
/* Host-exchange halves of a multi-rank evaluate (options.exchange = 1).  upward: charges
 * (host, full vector, input_order as in kifmm_gpu_evaluate) -> P2M + M2M of the rank's subtrees; writes
 * the rank's export rows to export_rows (host, halo_rows_max x ne_pad values of the plan precision, rows
 * in kifmm_halo_view export order, the tail unwritten).  downward: gathered (host, world_size slots laid
 * out like export_rows, slot r = rank r's export_rows) -> import + redundant top M2M + downward pass +
 * leaves; writes potential / gradient like kifmm_gpu_evaluate with the input_order of the upward call.
 * Each call is synchronous; the two must alternate. */
kifmm_status kifmm_gpu_evaluate_upward(kifmm_gpu_plan* plan, const void* charges, int32_t input_order,
                                       void* export_rows);
kifmm_status kifmm_gpu_evaluate_downward(kifmm_gpu_plan* plan, const void* gathered, void* potential,
                                         void* gradient);
kifmm_status kifmm_gpu_plan_get_info(const kifmm_gpu_plan* plan, kifmm_gpu_plan_info* info);
/* Per-phase device timings (CUDA events on the plan stream) of the last kifmm_gpu_evaluate call that
 * passed a timings struct (a serialized, instrumented run; evaluate_device / evaluate_many are never
 * instrumented and do not update them). */
kifmm_status kifmm_gpu_last_timings(kifmm_gpu_plan* plan, kifmm_gpu_timings* timings);
void kifmm_gpu_plan_destroy(kifmm_gpu_plan* plan);

/* 128-byte NCCL unique id for kifmm_gpu_options.nccl_unique_id (call on rank 0). */
kifmm_status kifmm_gpu_nccl_unique_id(void* out128);

/* Direct summation on the device (verification kernel K10):
 * potentials (and gradients) at `m` target particles (indices into positions)
 * from all n sources; self-pairs contribute 0.  Host buffers. */
kifmm_status kifmm_gpu_direct(int32_t precision, int32_t device, const void* positions,
                              const void* charges, int64_t n, const int64_t* targets, int64_t m,
                              void* potential, void* gradient);

/* FFMA / DFMA throughput probe on `device` (FLOP/s) used as the SIMT roofline denominator. */
kifmm_status kifmm_gpu_fma_peak(int32_t device, int32_t precision, double* flops_per_second);

#ifdef __cplusplus
}
#endif

#endif /* KIFMM_H_ */
