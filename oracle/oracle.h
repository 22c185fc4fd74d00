/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * fp64 CPU restatement of the reference's evaluate path plus
 * brute-force restatements of the tree and the interaction
 * lists.  It is the parity checker for the GPU library and
 * the timed CPU baseline ("kind": "port") in bench.py.  The product library
 * (paper_2303_08394_b200) never links, imports or calls anything in oracle/.
 *
 * Parity status: the reference ships no runnable FMM, so this
 * oracle is pinned by the SPEC's known-answer tests and by direct summation
 * (tests/golden), not by reference outputs.
 */
#ifndef KIFMM_ORACLE_H_
#define KIFMM_ORACLE_H_

#include <stdint.h>

#include "kifmm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_timings {
  double p2m_ms, m2m_ms, m2l_ms, p2l_ms, l2l_ms, near_ms, l2p_ms, m2p_ms, total_ms;
  /* call structure (SPEC acceptance #8): level invocations of the level-by-level operators and
     per-target applications of the leaf / node operators */
  int64_t m2m_levels, m2l_levels, l2l_levels;
  int64_t p2m_calls, near_calls, l2p_calls, m2p_calls, p2l_calls;
} oracle_timings;

/* Full evaluate over reordered charges.  potential: N (reordered);
 * gradient: N x 3 or NULL.  Only targets of leaves [leaf_begin, leaf_end) are
 * written (pass 0, n_leaves for all); the upward pass is always complete. */
int oracle_evaluate(const kifmm_tree_view* tree, const kifmm_operator_view* ops, const double* charges,
                    double* potential, double* gradient, int32_t threads, int64_t leaf_begin,
                    int64_t leaf_end, oracle_timings* timings);

/* Partitioned evaluate, split at the exchange point:
 *  upward_local: P2M + M2M for nodes at level >= cut_level whose leaves all lie
 *                in [leaf_begin, leaf_end) (plus owned leaves coarser than cut);
 *                every other multipole slice is left 0.  multipole: n_nodes x n_e.
 *  upward_top:   M2M for the non-leaf nodes above cut_level from the (gathered)
 *                complete level-cut multipoles.
 *  downward:     M2L/P2L/L2L/L2P/M2P/near field for the owned leaves. */
int oracle_upward_local(const kifmm_tree_view* tree, const kifmm_operator_view* ops, const double* charges,
                        int64_t leaf_begin, int64_t leaf_end, int32_t cut_level, double* multipole,
                        int32_t threads);
int oracle_upward_top(const kifmm_tree_view* tree, const kifmm_operator_view* ops, int32_t cut_level,
                      double* multipole, int32_t threads);
/* M2M of the listed non-leaf nodes, in the given order (children before parents):
 * the multi-rank top of the tree, recomputed by every rank from gathered rows. */
int oracle_m2m_nodes(const kifmm_tree_view* tree, const kifmm_operator_view* ops, int64_t n, const int64_t* nodes,
                     double* multipole);
int oracle_downward(const kifmm_tree_view* tree, const kifmm_operator_view* ops, const double* charges,
                    const double* multipole, int64_t leaf_begin, int64_t leaf_end, double* potential,
                    double* gradient, int32_t threads, oracle_timings* timings);

/* Direct summation at m targets (indices into positions, or
 * NULL for all n) from all n sources; self-pairs contribute 0. */
void oracle_direct(const double* positions, const double* charges, int64_t n, const int64_t* targets,
                   int64_t m, double* potential, double* gradient, int32_t threads);

/* Brute-force lists from the definitions (X on all nodes) for the target leaves
 * leaf_targets (U, W lists) and target nodes node_targets (V with transfer-vector ids, X), every target
 * checked against every candidate of the tree, in the CSR layout of kifmm_tree_view (one row per
 * target, in the order given; members in ascending raw key).  Arrays are malloc'ed; release them
 * with oracle_csr_free. */
typedef struct oracle_csr {
  int64_t *u_ptr, *u_idx, *v_ptr, *v_idx;
  int32_t* v_tv;
  int64_t *w_ptr, *w_idx, *x_ptr, *x_idx;
  int64_t n_u, n_v, n_w, n_x; /* total members */
} oracle_csr;
int oracle_lists_subset(const kifmm_tree_view* tree, int64_t n_leaf_targets, const int64_t* leaf_targets,
                        int64_t n_node_targets, const int64_t* node_targets, int32_t threads, oracle_csr* out);
void oracle_csr_free(oracle_csr* c);

/* Brute-force recursive split + pairwise balance.
 * Writes the sorted leaf keys (capacity cap) and returns their count (or -1). */
int64_t oracle_tree_leaves(const double* positions, int64_t n, int32_t n_crit, const double domain[4],
                           int32_t balance, uint64_t* leaves, int64_t cap);

/* OpenMP threads the oracle uses with threads = 0 (resolve_threads(0), parallel.hpp:22-26). */
int32_t oracle_max_threads(void);

/* Relative L2 error ||a-b|| / ||b||; -1 when ||b|| = 0. */
double oracle_relative_error(const double* a, const double* b, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
