// TEST INFRASTRUCTURE ONLY -- see oracle.h.
//
// fp64 CPU restatement of the KIFMM evaluate as SPEC.md defines it.  Each step
// cites the SPEC line it follows.  Written independently of the product
// library (it only shares the plain-data view structs of include/kifmm.h).
// Parallel loops follow the ownership rule of proj/src/parallel.hpp:28-43 (one
// owner per output slice, no shared accumulators), so results do not depend on
// the thread count; the schedule is dynamic (chunks of 8) rather than
// parallel.hpp's static one because leaf costs are uneven -- the schedule only
// decides which thread computes a slice, never the arithmetic order inside it.
#include "oracle.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <tuple>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <vector>

namespace {

constexpr int MAXL = 15;
constexpr double INV4PI = 1.0 / (4.0 * 3.14159265358979323846);

// ---- key restatement (layout documented in include/kifmm.h)
int lev(uint64_t k) { return int(k & 15u); }
uint32_t compact(uint64_t x) {
  uint32_t r = 0;
  for (int i = 0; i < 21; ++i) r |= uint32_t((x >> (3 * i)) & 1u) << i;
  return r;
}
void anchor(uint64_t k, int64_t a[3]) {
  const uint64_t c = k >> 4;
  const int sh = MAXL - lev(k);
  a[0] = compact(c) >> sh;
  a[1] = compact(c >> 1) >> sh;
  a[2] = compact(c >> 2) >> sh;
}
uint64_t spread(uint32_t v) {
  uint64_t r = 0;
  for (int i = 0; i < 21; ++i) r |= uint64_t((v >> i) & 1u) << (3 * i);
  return r;
}
uint64_t mkkey(int64_t x, int64_t y, int64_t z, int l) {
  const int sh = MAXL - l;
  return ((spread(uint32_t(x << sh)) | (spread(uint32_t(y << sh)) << 1) | (spread(uint32_t(z << sh)) << 2)) << 4) |
         uint64_t(l);
}
uint64_t parent_key(uint64_t k) {
  int64_t a[3];
  anchor(k, a);
  return mkkey(a[0] >> 1, a[1] >> 1, a[2] >> 1, lev(k) - 1);
}
// closed cubes share a point, neither contains the other.
bool adjacent(uint64_t x, uint64_t y) {
  int64_t ax[3], ay[3];
  anchor(x, ax);
  anchor(y, ay);
  const int64_t wx = int64_t(1) << (MAXL - lev(x)), wy = int64_t(1) << (MAXL - lev(y));
  bool xin = true, yin = true;
  for (int d = 0; d < 3; ++d) {
    const int64_t xl = ax[d] * wx, xh = xl + wx, yl = ay[d] * wy, yh = yl + wy;
    if (xl > yh || yl > xh) return false;
    if (!(xl >= yl && xh <= yh)) xin = false;
    if (!(yl >= xl && yh <= xh)) yin = false;
  }
  return !(xin || yin);
}
// center = origin + (anchor + 1/2) side / 2^l, half_side = side / 2^(l+1)
void bounds(const kifmm_tree_view* t, uint64_t k, double c[3], double* h) {
  int64_t a[3];
  anchor(k, a);
  const double w = t->side / double(int64_t(1) << lev(k));
  for (int d = 0; d < 3; ++d) c[d] = t->origin[d] + (double(a[d]) + 0.5) * w;
  *h = t->side / double(int64_t(1) << (lev(k) + 1));
}

// SPEC.md:294-302
inline double lap(double x0, double x1, double x2, double y0, double y1, double y2) {
  const double dx = x0 - y0, dy = x1 - y1, dz = x2 - y2;
  const double r2 = dx * dx + dy * dy + dz * dz;
  return r2 == 0.0 ? 0.0 : INV4PI / std::sqrt(r2);
}
// potential (+ gradient w.r.t. the target) of source q at s, evaluated at t
inline void lap_grad(const double* t, const double* s, double q, double& phi, double* g) {
  const double dx = t[0] - s[0], dy = t[1] - s[1], dz = t[2] - s[2];
  const double r2 = dx * dx + dy * dy + dz * dz;
  if (r2 == 0.0) return;
  const double rinv = 1.0 / std::sqrt(r2);
  const double p = q * INV4PI * rinv;
  phi += p;
  if (g) {
    const double f = p * rinv * rinv;
    g[0] -= f * dx;
    g[1] -= f * dy;
    g[2] -= f * dz;
  }
}

// surface point j of node (c, h) at scaling alpha
inline void surf(const kifmm_operator_view* o, const double c[3], double h, double alpha, int j, double out[3]) {
  for (int d = 0; d < 3; ++d) out[d] = c[d] + alpha * h * o->surface[3 * j + d];
}

// pinv application, factored: out = scale * V diag(1/s) U^T in
void apply_pinv(int nc, int ne, int k, const double* U, const double* S, const double* V, const double* in,
                double scale, double* out) {
  std::vector<double> tmp(k);
  for (int a = 0; a < k; ++a) {
    double acc = 0;
    for (int i = 0; i < nc; ++i) acc += U[size_t(i) * k + a] * in[i];
    tmp[a] = acc / S[a];
  }
  for (int i = 0; i < ne; ++i) {
    double acc = 0;
    for (int a = 0; a < k; ++a) acc += V[size_t(i) * k + a] * tmp[a];
    out[i] = scale * acc;
  }
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

template <class F>
void pfor(int64_t n, int threads, F&& f) {
  if (threads <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
  for (int64_t i = 0; i < n; ++i) f(i);
}

int resolve(int threads) { return threads <= 0 ? omp_get_max_threads() : threads; }

// ---- upward pass ---------------------------------------------------------

// check = p2p(leaf particles -> up-check surface);
// M += scale(l) uc2e_inv check, scale(l) = 2^(2-l) (kernel homogeneity)
void p2m_leaf(const kifmm_tree_view* t, const kifmm_operator_view* o, const double* q, int64_t leaf, double* M) {
  const int ne = o->n_e, nc = o->n_c;
  const int64_t node = t->leaf_node[leaf];
  const uint64_t k = t->node_key[node];
  double c[3], h;
  bounds(t, k, c, &h);
  std::vector<double> check(nc, 0.0);
  for (int j = 0; j < nc; ++j) {
    double y[3];
    surf(o, c, h, o->alpha_outer, j, y);
    double acc = 0;
    for (int64_t i = t->leaf_ptr[leaf]; i < t->leaf_ptr[leaf + 1]; ++i) {
      const double* x = &t->positions[3 * i];
      acc += q[i] * lap(x[0], x[1], x[2], y[0], y[1], y[2]);
    }
    check[j] = acc;
  }
  const double scale = std::ldexp(1.0, o->reference_level - lev(k));
  apply_pinv(nc, ne, o->uc2e_rank, o->uc2e_u, o->uc2e_s, o->uc2e_v, check.data(), scale, &M[size_t(node) * ne]);
}

// parent += sum_o m2m[o] child_o
void m2m_node(const kifmm_tree_view* t, const kifmm_operator_view* o, int64_t node, double* M) {
  const int ne = o->n_e;
  double* out = &M[size_t(node) * ne];
  for (int i = 0; i < ne; ++i) out[i] = 0.0;
  for (int oc = 0; oc < 8; ++oc) {
    const int64_t ch = t->node_children[8 * node + oc];
    if (ch < 0) continue;
    const double* mat = &o->m2m[size_t(oc) * ne * ne];
    const double* in = &M[size_t(ch) * ne];
    for (int i = 0; i < ne; ++i) {
      double acc = 0;
      for (int j = 0; j < ne; ++j) acc += mat[size_t(i) * ne + j] * in[j];
      out[i] += acc;
    }
  }
}

// leaf descendant range of a node (leaves are in ascending raw key = spatial order)
void node_leaf_range(const kifmm_tree_view* t, int64_t node, int64_t& lo, int64_t& hi) {
  int64_t a = node, b = node;
  while (t->node_leaf[a] < 0)
    for (int oc = 0; oc < 8; ++oc)
      if (t->node_children[8 * a + oc] >= 0) {
        a = t->node_children[8 * a + oc];
        break;
      }
  while (t->node_leaf[b] < 0)
    for (int oc = 7; oc >= 0; --oc)
      if (t->node_children[8 * b + oc] >= 0) {
        b = t->node_children[8 * b + oc];
        break;
      }
  lo = t->node_leaf[a];
  hi = t->node_leaf[b] + 1;
}

}  // namespace

// Brute-force lists straight from the definitions (X on all nodes), for a
// chosen set of target leaves (U, W) and target nodes (V, X).  Every target is checked against EVERY
// candidate of the tree (no spatial pruning); geometry is integer intervals on the level-15 grid.
namespace {
struct Box {
  int64_t lo[3], w;  // cube [lo, lo + w] per axis on the MAX_LEVEL grid
  int l;
};
Box box_of(uint64_t k) {
  Box b;
  int64_t a[3];
  anchor(k, a);
  b.l = lev(k);
  b.w = int64_t(1) << (MAXL - b.l);
  for (int d = 0; d < 3; ++d) b.lo[d] = a[d] * b.w;
  return b;
}
Box parent_box(const Box& b) {
  Box p;
  p.l = b.l - 1;
  p.w = 2 * b.w;
  for (int d = 0; d < 3; ++d) p.lo[d] = b.lo[d] - b.lo[d] % p.w;
  return p;
}
// closed cubes share a point and neither contains the other
bool adj(const Box& x, const Box& y) {
  bool xin = true, yin = true;
  for (int d = 0; d < 3; ++d) {
    const int64_t xl = x.lo[d], xh = xl + x.w, yl = y.lo[d], yh = yl + y.w;
    if (xl > yh || yl > xh) return false;
    if (!(xl >= yl && xh <= yh)) xin = false;
    if (!(yl >= xl && yh <= xh)) yin = false;
  }
  return !(xin || yin);
}
int tv_id(int dx, int dy, int dz) {  // rank among [-3,3]^3 offsets with Chebyshev norm >= 2, lexicographic
  int id = 0;
  for (int x = -3; x <= 3; ++x)
    for (int y = -3; y <= 3; ++y)
      for (int z = -3; z <= 3; ++z) {
        if (std::max(std::abs(x), std::max(std::abs(y), std::abs(z))) < 2) continue;
        if (std::make_tuple(x, y, z) < std::make_tuple(dx, dy, dz)) ++id;
      }
  return id;
}
template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<size_t>(1, v.size())));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}
}  // namespace

extern "C" {

int oracle_upward_local(const kifmm_tree_view* t, const kifmm_operator_view* o, const double* q, int64_t lb,
                        int64_t le, int32_t cut, double* M, int32_t threads) {
  threads = resolve(threads);
  const int ne = o->n_e;
  std::memset(M, 0, sizeof(double) * size_t(t->n_nodes) * ne);
  pfor(le - lb, threads, [&](int64_t i) { p2m_leaf(t, o, q, lb + i, M); });
  for (int l = t->depth - 1; l >= std::max(cut, 0); --l) {
    const int64_t b = t->level_ptr[l], e = t->level_ptr[l + 1];
    pfor(e - b, threads, [&](int64_t i) {
      const int64_t node = b + i;
      if (t->node_leaf[node] >= 0) return;
      int64_t lo, hi;
      node_leaf_range(t, node, lo, hi);
      if (lo >= lb && hi <= le) m2m_node(t, o, node, M);
    });
  }
  return 0;
}

int oracle_upward_top(const kifmm_tree_view* t, const kifmm_operator_view* o, int32_t cut, double* M,
                      int32_t threads) {
  threads = resolve(threads);
  for (int l = std::min<int>(cut, t->depth) - 1; l >= 0; --l) {
    const int64_t b = t->level_ptr[l], e = t->level_ptr[l + 1];
    pfor(e - b, threads, [&](int64_t i) {
      const int64_t node = b + i;
      if (t->node_leaf[node] < 0) m2m_node(t, o, node, M);
    });
  }
  return 0;
}

int oracle_m2m_nodes(const kifmm_tree_view* t, const kifmm_operator_view* o, int64_t n, const int64_t* nodes,
                     double* M) {
  for (int64_t i = 0; i < n; ++i) m2m_node(t, o, nodes[i], M);  // in the given (bottom-up) order
  return 0;
}

int oracle_downward(const kifmm_tree_view* t, const kifmm_operator_view* o, const double* q, const double* M,
                    int64_t lb, int64_t le, double* phi, double* grad, int32_t threads, oracle_timings* tm) {
  threads = resolve(threads);
  const int ne = o->n_e, nc = o->n_c;
  const int64_t nn = t->n_nodes;
  oracle_timings local{};
  // target nodes: ancestors-or-self of owned leaves at level >= 2
  std::vector<char> active(nn, 0);
  for (int64_t l = lb; l < le; ++l)
    for (int64_t n = t->leaf_node[l]; n >= 0 && !active[n]; n = t->node_parent[n]) active[n] = 1;
  std::vector<double> L(size_t(nn) * ne, 0.0);
  std::vector<double> chk(size_t(nn) * nc, 0.0);

  // SPEC.md:450-458 M2L in check-accumulate form: check_B = sum_{S in V(B)} K_t M_S at the
  // reference level; the level factors of K_l = 2^(l-2) K_2 and dc2e_inv_l = 2^(2-l) dc2e_inv_2
  // cancel, so L_B = dc2e_inv_2 check_B.
  auto t0 = std::chrono::steady_clock::now();
  {
    std::set<int> lv;
    for (int64_t b = 0; b < nn; ++b)
      if (active[b] && lev(t->node_key[b]) >= 2 && t->v_ptr[b] != t->v_ptr[b + 1]) lv.insert(lev(t->node_key[b]));
    local.m2l_levels = int64_t(lv.size());
    for (int64_t b = 0; b < nn; ++b) local.p2l_calls += active[b] && t->x_ptr[b] != t->x_ptr[b + 1];
  }
  pfor(nn, threads, [&](int64_t b) {
    if (!active[b] || lev(t->node_key[b]) < 2) return;
    double* c = &chk[size_t(b) * nc];
    for (int64_t e = t->v_ptr[b]; e < t->v_ptr[b + 1]; ++e) {
      const double* K = &o->m2l[size_t(t->v_tv[e]) * nc * ne];
      const double* ms = &M[size_t(t->v_idx[e]) * ne];
      for (int i = 0; i < nc; ++i) {
        double acc = 0;
        for (int j = 0; j < ne; ++j) acc += K[size_t(i) * ne + j] * ms[j];
        c[i] += acc;
      }
    }
  });
  local.m2l_ms = ms_since(t0);
  // SPEC.md:481-486 P2L: check += scale(l) p2p(X particles -> down-check surface), scale = 2^(2-l)
  t0 = std::chrono::steady_clock::now();
  pfor(nn, threads, [&](int64_t b) {
    if (!active[b] || t->x_ptr[b] == t->x_ptr[b + 1]) return;
    const uint64_t k = t->node_key[b];
    double cb[3], h;
    bounds(t, k, cb, &h);
    const double scale = std::ldexp(1.0, o->reference_level - lev(k));
    double* c = &chk[size_t(b) * nc];
    for (int j = 0; j < nc; ++j) {
      double y[3];
      surf(o, cb, h, o->alpha_inner, j, y);
      double acc = 0;
      for (int64_t e = t->x_ptr[b]; e < t->x_ptr[b + 1]; ++e) {
        const int64_t a = t->x_idx[e];
        for (int64_t i = t->leaf_ptr[a]; i < t->leaf_ptr[a + 1]; ++i) {
          const double* x = &t->positions[3 * i];
          acc += q[i] * lap(x[0], x[1], x[2], y[0], y[1], y[2]);
        }
      }
      c[j] += scale * acc;
    }
  });
  local.p2l_ms = ms_since(t0);
  // downward solve then L2L, level by level ("for l = 2..d")
  t0 = std::chrono::steady_clock::now();
  for (int l = 2; l <= t->depth; ++l) {
    const int64_t b0 = t->level_ptr[l], e0 = t->level_ptr[l + 1];
    if (l - 1 >= 2) ++local.l2l_levels;
    pfor(e0 - b0, threads, [&](int64_t i) {
      const int64_t b = b0 + i;
      if (!active[b]) return;
      double* Lb = &L[size_t(b) * ne];
      apply_pinv(nc, ne, o->dc2e_rank, o->dc2e_u, o->dc2e_s, o->dc2e_v, &chk[size_t(b) * nc], 1.0, Lb);
      const int64_t par = t->node_parent[b];
      if (l - 1 >= 2) {
        const int oc = int((t->node_key[b] >> (4 + 3 * (MAXL - l))) & 7u);
        const double* mat = &o->l2l[size_t(oc) * ne * ne];
        const double* lp = &L[size_t(par) * ne];
        for (int r = 0; r < ne; ++r) {
          double acc = 0;
          for (int j = 0; j < ne; ++j) acc += mat[size_t(r) * ne + j] * lp[j];
          Lb[r] += acc;
        }
      }
    });
  }
  local.l2l_ms = ms_since(t0);

  // leaves: near field, L2P (467-472), M2P (474-479)
  t0 = std::chrono::steady_clock::now();
  for (int64_t a = lb; a < le; ++a) {
    ++local.near_calls;
    local.l2p_calls += lev(t->node_key[t->leaf_node[a]]) >= 2;
    local.m2p_calls += t->w_ptr[a] != t->w_ptr[a + 1];
  }
  pfor(le - lb, threads, [&](int64_t li) {
    const int64_t a = lb + li;
    const int64_t node = t->leaf_node[a];
    const uint64_t k = t->node_key[node];
    double ca[3], ha;
    bounds(t, k, ca, &ha);
    for (int64_t i = t->leaf_ptr[a]; i < t->leaf_ptr[a + 1]; ++i) {
      const double* x = &t->positions[3 * i];
      double p = 0, g[3] = {0, 0, 0};
      double* gp = grad ? g : nullptr;
      for (int64_t e = t->u_ptr[a]; e < t->u_ptr[a + 1]; ++e) {
        const int64_t s = t->u_idx[e];
        for (int64_t j = t->leaf_ptr[s]; j < t->leaf_ptr[s + 1]; ++j) lap_grad(x, &t->positions[3 * j], q[j], p, gp);
      }
      if (lev(k) >= 2) {
        const double* Lb = &L[size_t(node) * ne];
        for (int j = 0; j < ne; ++j) {
          double y[3];
          surf(o, ca, ha, o->alpha_outer, j, y);
          lap_grad(x, y, Lb[j], p, gp);
        }
      }
      for (int64_t e = t->w_ptr[a]; e < t->w_ptr[a + 1]; ++e) {
        const int64_t s = t->w_idx[e];
        double cs[3], hs;
        bounds(t, t->node_key[s], cs, &hs);
        const double* Ms = &M[size_t(s) * ne];
        for (int j = 0; j < ne; ++j) {
          double y[3];
          surf(o, cs, hs, o->alpha_inner, j, y);
          lap_grad(x, y, Ms[j], p, gp);
        }
      }
      phi[i] = p;
      if (grad)
        for (int d = 0; d < 3; ++d) grad[3 * i + d] = g[d];
    }
  });
  local.near_ms = ms_since(t0);
  if (tm) {
    tm->m2l_levels += local.m2l_levels;
    tm->l2l_levels += local.l2l_levels;
    tm->near_calls += local.near_calls;
    tm->l2p_calls += local.l2p_calls;
    tm->m2p_calls += local.m2p_calls;
    tm->p2l_calls += local.p2l_calls;
    tm->m2l_ms += local.m2l_ms;
    tm->p2l_ms += local.p2l_ms;
    tm->l2l_ms += local.l2l_ms;
    tm->near_ms += local.near_ms;
  }
  return 0;
}

int oracle_evaluate(const kifmm_tree_view* t, const kifmm_operator_view* o, const double* q, double* phi,
                    double* grad, int32_t threads, int64_t lb, int64_t le, oracle_timings* tm) {
  threads = resolve(threads);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<double> M(size_t(t->n_nodes) * o->n_e, 0.0);
  oracle_timings local{};
  auto t1 = std::chrono::steady_clock::now();
  pfor(t->n_leaves, threads, [&](int64_t l) { p2m_leaf(t, o, q, l, M.data()); });
  local.p2m_calls = t->n_leaves;
  local.p2m_ms = ms_since(t1);
  t1 = std::chrono::steady_clock::now();
  for (int l = t->depth - 1; l >= 0; --l) {
    ++local.m2m_levels;
    const int64_t b = t->level_ptr[l], e = t->level_ptr[l + 1];
    pfor(e - b, threads, [&](int64_t i) {
      if (t->node_leaf[b + i] < 0) m2m_node(t, o, b + i, M.data());
    });
  }
  local.m2m_ms = ms_since(t1);
  oracle_downward(t, o, q, M.data(), lb, le, phi, grad, threads, &local);
  local.total_ms = ms_since(t0);
  if (tm) *tm = local;
  return 0;
}

void oracle_direct(const double* pos, const double* q, int64_t n, const int64_t* targets, int64_t m, double* phi,
                   double* grad, int32_t threads) {
  threads = resolve(threads);
  if (!targets) m = n;
  pfor(m, threads, [&](int64_t r) {
    const int64_t i = targets ? targets[r] : r;
    double p = 0, g[3] = {0, 0, 0};
    for (int64_t j = 0; j < n; ++j) lap_grad(&pos[3 * i], &pos[3 * j], q[j], p, grad ? g : nullptr);
    phi[r] = p;
    if (grad)
      for (int d = 0; d < 3; ++d) grad[3 * r + d] = g[d];
  });
}

int32_t oracle_max_threads(void) { return resolve(0); }

double oracle_relative_error(const double* a, const double* b, int64_t n) {
  long double num = 0, den = 0;
  for (int64_t i = 0; i < n; ++i) {
    num += (long double)(a[i] - b[i]) * (a[i] - b[i]);
    den += (long double)b[i] * b[i];
  }
  if (den == 0) return -1.0;
  return double(std::sqrt(num / den));
}


int oracle_lists_subset(const kifmm_tree_view* t, int64_t n_lt, const int64_t* leaf_targets, int64_t n_nt,
                        const int64_t* node_targets, int32_t threads, oracle_csr* out) {
  threads = resolve(threads);
  const int64_t nn = t->n_nodes, nl = t->n_leaves;
  std::vector<Box> bx(nn);
  pfor(nn, threads, [&](int64_t n) { bx[n] = box_of(t->node_key[n]); });
  // members in ascending raw key: nodes are level-major, so sort candidates by key
  std::vector<std::vector<int64_t>> U(n_lt), W(n_lt), V(n_nt), X(n_nt);
  std::vector<std::vector<int32_t>> TV(n_nt);
  auto by_key = [&](std::vector<int64_t>& m) {
    std::sort(m.begin(), m.end(), [&](int64_t a, int64_t b) { return t->node_key[a] < t->node_key[b]; });
  };
  pfor(n_lt, threads, [&](int64_t i) {
    const int64_t a = leaf_targets[i];
    const int64_t na = t->leaf_node[a];
    const Box& A = bx[na];
    // U: every leaf adjacent to A, plus A itself
    std::vector<int64_t> u;
    for (int64_t b = 0; b < nl; ++b)
      if (b == a || adj(A, bx[t->leaf_node[b]])) u.push_back(t->leaf_node[b]);
    by_key(u);
    for (auto& x : u) x = t->node_leaf[x];
    U[i] = std::move(u);
    // W: nodes strictly finer than A whose parent is adjacent to A, not adjacent to A
    std::vector<int64_t> w;
    for (int64_t c = 0; c < nn; ++c)
      if (bx[c].l > A.l && adj(parent_box(bx[c]), A) && !adj(bx[c], A)) w.push_back(c);
    by_key(w);
    W[i] = std::move(w);
  });
  pfor(n_nt, threads, [&](int64_t i) {
    const int64_t b = node_targets[i];
    const Box& B = bx[b];
    // V: same-level nodes whose parent is a same-level neighbour of parent(B), not adjacent to B
    if (B.l >= 2) {
      const Box PB = parent_box(B);
      std::vector<int64_t> v;
      for (int64_t c = t->level_ptr[B.l]; c < t->level_ptr[B.l + 1]; ++c) {
        const Box PC = parent_box(bx[c]);
        bool same = true;
        for (int d = 0; d < 3; ++d) same = same && PC.lo[d] == PB.lo[d];
        if (!same && adj(PC, PB) && !adj(bx[c], B)) v.push_back(c);
      }
      by_key(v);
      std::vector<int32_t> tv;
      for (int64_t c : v)
        tv.push_back(tv_id(int((bx[c].lo[0] - B.lo[0]) / B.w), int((bx[c].lo[1] - B.lo[1]) / B.w),
                           int((bx[c].lo[2] - B.lo[2]) / B.w)));
      V[i] = std::move(v);
      TV[i] = std::move(tv);
    }
    // X: leaves A with B in W(A) -- coarser than B, adjacent to parent(B), not adjacent to B
    if (B.l >= 1) {
      const Box PB = parent_box(B);
      std::vector<int64_t> x;
      for (int64_t a = 0; a < nl; ++a) {
        const Box& A = bx[t->leaf_node[a]];
        if (A.l < B.l && adj(PB, A) && !adj(B, A)) x.push_back(a);  // leaves ascend in raw key
      }
      X[i] = std::move(x);
    }
  });
  auto csr = [](const std::vector<std::vector<int64_t>>& L, int64_t** ptr, int64_t** idx, int64_t* total) {
    std::vector<int64_t> p{0}, ix;
    for (const auto& l : L) {
      ix.insert(ix.end(), l.begin(), l.end());
      p.push_back(int64_t(ix.size()));
    }
    *ptr = dup(p);
    *idx = dup(ix);
    *total = int64_t(ix.size());
  };
  csr(U, &out->u_ptr, &out->u_idx, &out->n_u);
  csr(W, &out->w_ptr, &out->w_idx, &out->n_w);
  csr(V, &out->v_ptr, &out->v_idx, &out->n_v);
  csr(X, &out->x_ptr, &out->x_idx, &out->n_x);
  std::vector<int32_t> tvs;
  for (const auto& l : TV) tvs.insert(tvs.end(), l.begin(), l.end());
  out->v_tv = dup(tvs);
  return 0;
}

void oracle_csr_free(oracle_csr* c) {
  for (void* p : {(void*)c->u_ptr, (void*)c->u_idx, (void*)c->v_ptr, (void*)c->v_idx, (void*)c->v_tv,
                  (void*)c->w_ptr, (void*)c->w_idx, (void*)c->x_ptr, (void*)c->x_idx})
    std::free(p);
  std::memset(c, 0, sizeof(*c));
}

int64_t oracle_tree_leaves(const double* pos, int64_t n, int32_t n_crit, const double dom[4], int32_t balance,
                           uint64_t* out, int64_t cap) {
  // fine cells: floor((x - o) 2^15 / side), clamped at the closed upper face
  std::vector<std::array<int64_t, 3>> cell(n);
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      const double v = (pos[3 * i + d] - dom[d]) * (double(1 << MAXL) / dom[3]);
      int64_t c = int64_t(std::floor(v));
      if (c >= (1 << MAXL)) c = (1 << MAXL) - 1;
      if (c < 0) return -1;
      cell[i][d] = c;
    }
  auto inside = [&](uint64_t k, int64_t i) {
    int64_t a[3];
    anchor(k, a);
    const int sh = MAXL - lev(k);
    for (int d = 0; d < 3; ++d)
      if ((cell[i][d] >> sh) != a[d]) return false;
    return true;
  };
  auto count = [&](uint64_t k) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i) c += inside(k, i);
    return c;
  };
  auto split = [&](uint64_t k, std::vector<uint64_t>& dst) {
    int64_t a[3];
    anchor(k, a);
    for (int oc = 0; oc < 8; ++oc) {
      const uint64_t ch = mkkey(2 * a[0] + (oc & 1), 2 * a[1] + ((oc >> 1) & 1), 2 * a[2] + ((oc >> 2) & 1), lev(k) + 1);
      if (count(ch) > 0) dst.push_back(ch);
    }
  };
  // recursive split
  std::vector<uint64_t> leaves, work{mkkey(0, 0, 0, 0)};
  while (!work.empty()) {
    const uint64_t k = work.back();
    work.pop_back();
    if (count(k) <= n_crit || lev(k) == MAXL) {
      leaves.push_back(k);
      continue;
    }
    split(k, work);
  }
  // pairwise balance to a fixed point
  while (balance) {
    std::set<uint64_t> refine;
    for (uint64_t a : leaves)
      for (uint64_t b : leaves)
        if (lev(a) + 1 < lev(b) && adjacent(a, b)) refine.insert(a);
    if (refine.empty()) break;
    std::vector<uint64_t> next;
    for (uint64_t a : leaves) {
      if (refine.count(a))
        split(a, next);
      else
        next.push_back(a);
    }
    leaves.swap(next);
  }
  std::sort(leaves.begin(), leaves.end());
  if (int64_t(leaves.size()) > cap) return -1;
  std::copy(leaves.begin(), leaves.end(), out);
  return int64_t(leaves.size());
}

}  // extern "C"
