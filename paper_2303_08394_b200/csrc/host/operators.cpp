// Surface grids, kernel matrices, truncated-SVD pseudo-inverses (kept factored),
// M2M/L2L composites and M2L kernel matrices, plus
// the on-disk cache archive.
#include "operators.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <exception>
#include <cstdio>
#include <cstring>
#include <tuple>
#include <fstream>
#include <numeric>
#include <sstream>

#include "common.hpp"
#include "parallel.hpp"
#include "tree.hpp"

namespace kifmm {

int surface_count(int p) { return p < 2 ? -1 : 6 * (p - 1) * (p - 1) + 2; }

std::vector<double> surface_grid(int p) {
  if (p < 2) throw InvalidArgument("surface_grid: p must be >= 2");
  std::vector<double> pts;
  pts.reserve(3 * size_t(surface_count(p)));
  // (2i - (p-1)) / (p-1): exact at the faces and symmetric under reflection
  auto coord = [p](int i) { return double(2 * i - (p - 1)) / double(p - 1); };
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k) {
        const bool on = i == 0 || i == p - 1 || j == 0 || j == p - 1 || k == 0 || k == p - 1;
        if (!on) continue;
        pts.push_back(coord(i));
        pts.push_back(coord(j));
        pts.push_back(coord(k));
      }
  return pts;
}

void kernel_matrix(const double* src, int64_t m, const double* tgt, int64_t k, double* out) {
  for (int64_t j = 0; j < k; ++j)
    for (int64_t i = 0; i < m; ++i)
      out[j * m + i] = laplace(src[3 * i], src[3 * i + 1], src[3 * i + 2], tgt[3 * j], tgt[3 * j + 1],
                               tgt[3 * j + 2]);
}

namespace {
// Below this column count a matrix is swept serially in cyclic order (the two precompute SVDs then run side by
// side with the M2L matrices); from it on, in parallel rounds of disjoint pairs.  The order depends on n only,
// never on the thread count, so the operators are reproducible on any host.
constexpr int kJacobiParallelMin = 256;
// One-sided Jacobi state of one matrix (columns of w are rotated until mutually orthogonal; vv accumulates V).
struct JacobiState {
  int m = 0, n = 0;
  std::vector<double> w, vv;  // column-major
  bool done = false;
  JacobiState(const double* a, int m_, int n_) : m(m_), n(n_), w(size_t(m_) * n_), vv(size_t(n_) * n_, 0.0) {
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) w[size_t(j) * m + i] = a[size_t(i) * n + j];
    for (int j = 0; j < n; ++j) vv[size_t(j) * n + j] = 1.0;
  }
  int rotate(int p, int q) {
    const double tol = DBL_EPSILON;
    double* wp = &w[size_t(p) * m];
    double* wq = &w[size_t(q) * m];
    double alpha = 0, beta = 0, gamma = 0;
    for (int i = 0; i < m; ++i) {
      alpha += wp[i] * wp[i];
      beta += wq[i] * wq[i];
      gamma += wp[i] * wq[i];
    }
    if (gamma == 0.0 || std::fabs(gamma) <= tol * std::sqrt(alpha * beta)) return 0;
    const double zeta = (beta - alpha) / (2.0 * gamma);
    const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
    const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
    for (int i = 0; i < m; ++i) {
      const double x = wp[i], y = wq[i];
      wp[i] = c * x - sn * y;
      wq[i] = sn * x + c * y;
    }
    double* vp = &vv[size_t(p) * n];
    double* vq = &vv[size_t(q) * n];
    for (int i = 0; i < n; ++i) {
      const double x = vp[i], y = vq[i];
      vp[i] = c * x - sn * y;
      vq[i] = sn * x + c * y;
    }
    return 1;
  }
  // serial cyclic-by-rows sweeps (all pairs p < q in order) until a sweep makes no rotation
  void cyclic_sweeps() {
    for (int sweep = 0; sweep < 80; ++sweep) {
      int rot = 0;
      for (int p = 0; p < n - 1; ++p)
        for (int q = p + 1; q < n; ++q) rot += rotate(p, q);
      if (rot == 0) break;
    }
    done = true;
  }
  void finish(double* u, double* s, double* v) const {
    std::vector<double> sig(n);
    for (int j = 0; j < n; ++j) {
      double acc = 0;
      for (int i = 0; i < m; ++i) acc += w[size_t(j) * m + i] * w[size_t(j) * m + i];
      sig[j] = std::sqrt(acc);
    }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sig[x] > sig[y]; });
    for (int jj = 0; jj < n; ++jj) {
      const int j = order[jj];
      s[jj] = sig[j];
      const double inv = sig[j] > 0 ? 1.0 / sig[j] : 0.0;
      for (int i = 0; i < m; ++i) u[size_t(i) * n + jj] = w[size_t(j) * m + i] * inv;
      for (int i = 0; i < n; ++i) v[size_t(i) * n + jj] = vv[size_t(j) * n + i];
    }
  }
};

// Round-robin ("tournament") pair order: a sweep is np - 1 rounds of np / 2 disjoint column pairs (np = n
// rounded up to even; the extra column is a bye).  The pairs of a round -- of every matrix of the batch, all
// of the same n -- rotate independently, so one parallel loop per round covers them all and the result does
// not depend on the thread count.  A matrix leaves the batch after its first sweep without a rotation.
void jacobi_sweeps(std::vector<JacobiState*>& mats, int threads) {
  if (mats.empty()) return;
  const int n = mats[0]->n, np = n + (n & 1), half = np / 2, nm = int(mats.size());
  std::vector<int> seat(np);
  std::iota(seat.begin(), seat.end(), 0);
  std::vector<long long> rot(nm);
  for (int sweep = 0; sweep < 80 && n > 1; ++sweep) {
    std::fill(rot.begin(), rot.end(), 0);
    for (int round = 0; round < np - 1; ++round) {
      // seats i and np - 1 - i meet; seat 0 stays, the others move one place per round
      auto meet = [&](int job) -> int {
        JacobiState& st = *mats[job / half];
        if (st.done) return 0;
        const int i = job % half;
        int p = seat[i], q = seat[np - 1 - i];
        if (p >= n || q >= n) return 0;  // bye
        if (p > q) std::swap(p, q);
        return st.rotate(p, q);
      };
      const int jobs = nm * half;
      if (threads > 1 && jobs >= 16) {
#pragma omp parallel for schedule(static) num_threads(threads)
        for (int job = 0; job < jobs; ++job) {
          if (meet(job)) {
#pragma omp atomic
            rot[job / half] += 1;
          }
        }
      } else {
        for (int job = 0; job < jobs; ++job) rot[job / half] += meet(job);
      }
      std::rotate(seat.begin() + 1, seat.end() - 1, seat.end());
    }
    bool all = true;
    for (int k = 0; k < nm; ++k) {
      if (rot[k] == 0) mats[k]->done = true;
      all = all && mats[k]->done;
    }
    if (all) break;
  }
}
}  // namespace

void jacobi_svd(const double* a, int m, int n, double* u, double* s, double* v, int threads) {
  if (m < n || n < 1) throw InvalidArgument("jacobi_svd: need m >= n >= 1");
  JacobiState st(a, m, n);
  if (n < kJacobiParallelMin) {
    st.cyclic_sweeps();
  } else {
    std::vector<JacobiState*> mats{&st};
    jacobi_sweeps(mats, threads);
  }
  st.finish(u, s, v);
}

// The SVDs of two matrices of the same shape in one batch (half as many synchronisations per rotation).
void jacobi_svd_pair(const double* a0, const double* a1, int m, int n, double* u0, double* s0, double* v0, double* u1,
                     double* s1, double* v1, int threads) {
  if (m < n || n < 1) throw InvalidArgument("jacobi_svd: need m >= n >= 1");
  JacobiState x(a0, m, n), y(a1, m, n);
  std::vector<JacobiState*> mats{&x, &y};
  jacobi_sweeps(mats, threads);
  x.finish(u0, s0, v0);
  y.finish(u1, s1, v1);
}

uint64_t operator_fingerprint(int p, double ai, double ao, double cutoff, double side) {
  uint64_t h = 1469598103934665603ULL;
  auto mix = [&](const void* data, size_t len) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < len; ++i) {
      h ^= b[i];
      h *= 1099511628211ULL;
    }
  };
  const char kernel[] = "laplace3d-1/(4pi r)-v1";
  mix(kernel, sizeof(kernel));
  mix(&p, sizeof(p));
  mix(&ai, sizeof(ai));
  mix(&ao, sizeof(ao));
  mix(&cutoff, sizeof(cutoff));
  mix(&side, sizeof(side));
  return h;
}

namespace {

// Truncated SVD of the check<-equivalent kernel matrix; keeps sigma_i >= cutoff*sigma_max.
void truncate_svd(const std::vector<double>& u, const std::vector<double>& s, const std::vector<double>& v, int nc,
                  int ne, double cutoff, int& rank, std::vector<double>& uk, std::vector<double>& sk,
                  std::vector<double>& vk, const char* name) {
  if (!(s[0] > 0.0) || !std::isfinite(s[0]))
    throw NumericalError(std::string("precompute: singular/non-finite ") + name);
  int r = 0;
  while (r < ne && s[r] >= cutoff * s[0]) ++r;
  rank = r;
  uk.assign(size_t(nc) * r, 0.0);
  vk.assign(size_t(ne) * r, 0.0);
  sk.assign(s.begin(), s.begin() + r);
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j < r; ++j) uk[size_t(i) * r + j] = u[size_t(i) * ne + j];
  for (int i = 0; i < ne; ++i)
    for (int j = 0; j < r; ++j) vk[size_t(i) * r + j] = v[size_t(i) * ne + j];
}

// out (ne x ne) = scale * V diag(1/s) (U^T K), K: nc x ne.  Factored application.
void apply_pinv(const std::vector<double>& uk, const std::vector<double>& sk, const std::vector<double>& vk,
                int r, int nc, int ne, const double* kmat, double scale, double* out) {
  std::vector<double> t(size_t(r) * ne, 0.0);
  for (int a = 0; a < r; ++a) {
    for (int c = 0; c < ne; ++c) {
      double acc = 0.0;
      for (int i = 0; i < nc; ++i) acc += uk[size_t(i) * r + a] * kmat[size_t(i) * ne + c];
      t[size_t(a) * ne + c] = acc / sk[a];
    }
  }
  for (int i = 0; i < ne; ++i)
    for (int c = 0; c < ne; ++c) {
      double acc = 0.0;
      for (int a = 0; a < r; ++a) acc += vk[size_t(i) * r + a] * t[size_t(a) * ne + c];
      out[size_t(i) * ne + c] = scale * acc;
    }
}

std::vector<double> scaled(const std::vector<double>& unit, const double c[3], double r) {
  std::vector<double> out(unit.size());
  for (size_t i = 0; i < unit.size() / 3; ++i)
    for (int d = 0; d < 3; ++d) out[3 * i + d] = c[d] + r * unit[3 * i + d];
  return out;
}

}  // namespace

void precompute(Operators& ops, int p, double ai, double ao, double cutoff, double side, int threads) {
  if (p < 2) throw InvalidArgument("precompute: p must be >= 2");
  if (!(ai > 0.0) || !(ao > ai)) throw InvalidArgument("precompute: need 0 < alpha_inner < alpha_outer");
  if (!(cutoff > 0.0) || !(cutoff < 1.0)) throw InvalidArgument("precompute: svd_cutoff must be in (0,1)");
  if (!(side > 0.0)) throw InvalidArgument("precompute: domain side must be > 0");
  threads = resolve_threads(threads);
  ops = Operators{};
  ops.p = p;
  ops.n_e = ops.n_c = surface_count(p);
  ops.alpha_inner = ai;
  ops.alpha_outer = ao;
  ops.svd_cutoff = cutoff;
  ops.domain_side = side;
  ops.reference_level = 2;
  const double h2 = side / 8.0;  // half side at the reference level 2
  ops.ref_half_side = h2;
  ops.surface = surface_grid(p);
  const int ne = ops.n_e, nc = ops.n_c;
  const double zero[3] = {0, 0, 0};

  // upward: check (alpha_out) <- equivalent (alpha_in); downward: check (alpha_in) <- equivalent (alpha_out)
  const auto ue = scaled(ops.surface, zero, ai * h2), uc = scaled(ops.surface, zero, ao * h2);
  const auto de = scaled(ops.surface, zero, ao * h2), dc = scaled(ops.surface, zero, ai * h2);
  std::vector<double> kup(size_t(nc) * ne), kdn(size_t(nc) * ne);
  kernel_matrix(ue.data(), ne, uc.data(), nc, kup.data());
  kernel_matrix(de.data(), ne, dc.data(), nc, kdn.data());
  // M2L kernel matrices K_t: source up-equivalent (alpha_in) at offset t * (2 h2) ->
  // target down-check (alpha_in), both at the reference level.
  const auto& tvs = transfer_vector_table();
  ops.m2l.assign(tvs.size() * size_t(nc) * ne, 0.0);
  auto m2l_matrix = [&](size_t t) {
    const double sc[3] = {2.0 * h2 * tvs[t][0], 2.0 * h2 * tvs[t][1], 2.0 * h2 * tvs[t][2]};
    const auto sue = scaled(ops.surface, sc, ai * h2);
    kernel_matrix(sue.data(), ne, dc.data(), nc, &ops.m2l[t * size_t(nc) * ne]);
  };
  std::vector<double> u0(size_t(nc) * ne), s0(ne), v0(size_t(ne) * ne), u1(u0.size()), s1(ne), v1(v0.size());
  if (ne < kJacobiParallelMin) {
    // small systems (p <= 7): the two serial SVDs (~45 ms each at p = 6) and the 316 M2L matrices are
    // independent jobs of one dynamic loop (jobs 0, 1 = the SVDs); each job owns its outputs
    std::exception_ptr svd_err[2];
    auto first_job = [&](size_t job) {
      if (job >= 2) return m2l_matrix(job - 2);
      try {
        if (job == 0)
          jacobi_svd(kup.data(), nc, ne, u0.data(), s0.data(), v0.data(), 1);
        else
          jacobi_svd(kdn.data(), nc, ne, u1.data(), s1.data(), v1.data(), 1);
      } catch (...) {
        svd_err[job] = std::current_exception();
      }
    };
    const long long n_first = 2 + static_cast<long long>(tvs.size());
    if (threads <= 1) {
      for (long long j = 0; j < n_first; ++j) first_job(size_t(j));
    } else {
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
      for (long long j = 0; j < n_first; ++j) first_job(size_t(j));
    }
    for (auto& e : svd_err)
      if (e) std::rethrow_exception(e);
  } else {
    // large systems (p >= 8): one Jacobi batch of both matrices, parallel over the disjoint column pairs of
    // each round-robin round; then the M2L matrices
    jacobi_svd_pair(kup.data(), kdn.data(), nc, ne, u0.data(), s0.data(), v0.data(), u1.data(), s1.data(), v1.data(),
                    threads);
    parallel_for(tvs.size(), threads, m2l_matrix);
  }
  truncate_svd(u0, s0, v0, nc, ne, cutoff, ops.uc2e_rank, ops.uc2e_u, ops.uc2e_s, ops.uc2e_v, "uc2e");
  truncate_svd(u1, s1, v1, nc, ne, cutoff, ops.dc2e_rank, ops.dc2e_u, ops.dc2e_s, ops.dc2e_v, "dc2e");

  // M2M_o = uc2e_inv(l) K(child ue(l+1) -> parent uc(l)); L2L_o = dc2e_inv(l+1) K(parent de(l) -> child dc(l+1)).
  // Both level-invariant; built with parent at level 2, child at 3.
  ops.m2m.assign(size_t(8) * ne * ne, 0.0);
  ops.l2l.assign(size_t(8) * ne * ne, 0.0);
  parallel_for(16, threads, [&](size_t job) {
    const int o = int(job % 8);
    const double h3 = 0.5 * h2;
    const double cc[3] = {((o & 1) ? 1.0 : -1.0) * h3, ((o & 2) ? 1.0 : -1.0) * h3, ((o & 4) ? 1.0 : -1.0) * h3};
    std::vector<double> k(size_t(nc) * ne);
    if (job < 8) {
      const auto cue = scaled(ops.surface, cc, ai * h3);
      kernel_matrix(cue.data(), ne, uc.data(), nc, k.data());
      apply_pinv(ops.uc2e_u, ops.uc2e_s, ops.uc2e_v, ops.uc2e_rank, nc, ne, k.data(), 1.0,
                 &ops.m2m[size_t(o) * ne * ne]);
    } else {
      const auto cdc = scaled(ops.surface, cc, ai * h3);
      kernel_matrix(de.data(), ne, cdc.data(), nc, k.data());
      // dc2e_inv at level 3 = 2^(2-3) dc2e_inv at level 2 (kernel homogeneity)
      apply_pinv(ops.dc2e_u, ops.dc2e_s, ops.dc2e_v, ops.dc2e_rank, nc, ne, k.data(), 0.5,
                 &ops.l2l[size_t(o) * ne * ne]);
    }
  });

  for (double x : ops.m2m)
    if (!std::isfinite(x)) throw NumericalError("precompute: non-finite m2m");
  for (double x : ops.l2l)
    if (!std::isfinite(x)) throw NumericalError("precompute: non-finite l2l");
  ops.fingerprint = operator_fingerprint(p, ai, ao, cutoff, side);
}

// ------------------------------------------------------------- persistence
// Archive: text manifest padded to a 64-byte multiple, then 64-byte aligned
// little-endian f64 row-major segments.
namespace {
constexpr int kArchiveVersion = 1;
struct Seg {
  std::string name;
  int64_t rows, cols;
  const std::vector<double>* data;
  std::vector<double>* out;
};
std::vector<Seg> segments(Operators& o) {
  const int64_t ne = o.n_e, nc = o.n_c;
  return {{"surface", ne, 3, &o.surface, &o.surface},
          {"uc2e_u", nc, o.uc2e_rank, &o.uc2e_u, &o.uc2e_u},
          {"uc2e_s", 1, o.uc2e_rank, &o.uc2e_s, &o.uc2e_s},
          {"uc2e_v", ne, o.uc2e_rank, &o.uc2e_v, &o.uc2e_v},
          {"dc2e_u", nc, o.dc2e_rank, &o.dc2e_u, &o.dc2e_u},
          {"dc2e_s", 1, o.dc2e_rank, &o.dc2e_s, &o.dc2e_s},
          {"dc2e_v", ne, o.dc2e_rank, &o.dc2e_v, &o.dc2e_v},
          {"m2m", 8 * ne, ne, &o.m2m, &o.m2m},
          {"l2l", 8 * ne, ne, &o.l2l, &o.l2l},
          {"m2l", 316 * nc, ne, &o.m2l, &o.m2l}};
}
int64_t align64(int64_t x) { return (x + 63) / 64 * 64; }
}  // namespace

void save_operators(const Operators& ops_in, const std::string& path) {
  Operators& ops = const_cast<Operators&>(ops_in);
  auto segs = segments(ops);
  std::ostringstream man;
  man.precision(17);
  man << "KIFMM-OPERATOR-CACHE " << kArchiveVersion << "\n";
  man << "fingerprint " << std::hex << ops.fingerprint << std::dec << "\n";
  man << "p " << ops.p << "\nn_e " << ops.n_e << "\nn_c " << ops.n_c << "\n";
  man << "reference_level " << ops.reference_level << "\n";
  man << "alpha_inner " << ops.alpha_inner << "\nalpha_outer " << ops.alpha_outer << "\n";
  man << "svd_cutoff " << ops.svd_cutoff << "\ndomain_side " << ops.domain_side << "\n";
  man << "uc2e_rank " << ops.uc2e_rank << "\ndc2e_rank " << ops.dc2e_rank << "\n";
  int64_t off = 0;
  for (auto& s : segs) {
    man << "matrix " << s.name << " " << s.rows << " " << s.cols << " " << off << "\n";
    off = align64(off + s.rows * s.cols * 8);
  }
  man << "end\n";
  std::string m = man.str();
  const int64_t header = align64(int64_t(m.size()) + 16);
  std::ofstream f(path, std::ios::binary);
  if (!f) throw IoError("save_cache: cannot open " + path);
  char head[16] = {0};
  std::snprintf(head, sizeof(head), "%015lld", static_cast<long long>(header));
  head[15] = '\n';
  f.write(head, 16);
  f.write(m.data(), std::streamsize(m.size()));
  std::string pad(size_t(header - 16 - int64_t(m.size())), '\0');
  f.write(pad.data(), std::streamsize(pad.size()));
  int64_t pos = 0;
  for (auto& s : segs) {
    const int64_t bytes = s.rows * s.cols * 8;
    static_assert(sizeof(double) == 8, "f64");
    // host is little-endian (x86-64 / aarch64); the archive is defined LE
    f.write(reinterpret_cast<const char*>(s.data->data()), std::streamsize(bytes));
    const int64_t next = align64(pos + bytes);
    std::string z(size_t(next - pos - bytes), '\0');
    f.write(z.data(), std::streamsize(z.size()));
    pos = next;
  }
  if (!f) throw IoError("save_cache: write failed for " + path);
}

void load_operators(Operators& ops, const std::string& path, uint64_t expected) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("load_cache: cannot open " + path);
  std::string all((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (all.size() < 16) throw CorruptArchive("load_cache: truncated header in " + path);
  const long long header = std::atoll(all.substr(0, 15).c_str());
  if (header < 16 || size_t(header) > all.size()) throw CorruptArchive("load_cache: bad header size");
  std::istringstream man(all.substr(16, size_t(header) - 16));
  std::string magic;
  int version = -1;
  man >> magic >> version;
  if (magic != "KIFMM-OPERATOR-CACHE") throw CorruptArchive("load_cache: bad magic");
  if (version != kArchiveVersion) throw CacheMismatch("load_cache: foreign format version " + std::to_string(version));
  Operators o;
  std::string key;
  std::vector<std::tuple<std::string, int64_t, int64_t, int64_t>> mats;
  bool ended = false;
  while (man >> key) {
    if (key == "fingerprint") man >> std::hex >> o.fingerprint >> std::dec;
    else if (key == "p") man >> o.p;
    else if (key == "n_e") man >> o.n_e;
    else if (key == "n_c") man >> o.n_c;
    else if (key == "reference_level") man >> o.reference_level;
    else if (key == "alpha_inner") man >> o.alpha_inner;
    else if (key == "alpha_outer") man >> o.alpha_outer;
    else if (key == "svd_cutoff") man >> o.svd_cutoff;
    else if (key == "domain_side") man >> o.domain_side;
    else if (key == "uc2e_rank") man >> o.uc2e_rank;
    else if (key == "dc2e_rank") man >> o.dc2e_rank;
    else if (key == "matrix") {
      std::string name;
      int64_t r, c, off;
      man >> name >> r >> c >> off;
      mats.emplace_back(name, r, c, off);
    } else if (key == "end") {
      ended = true;
      break;
    } else {
      throw CorruptArchive("load_cache: unknown manifest key " + key);
    }
    if (!man) throw CorruptArchive("load_cache: malformed manifest");
  }
  if (!ended) throw CorruptArchive("load_cache: manifest not terminated");
  if (expected != 0 && o.fingerprint != expected) throw CacheMismatch("load_cache: fingerprint mismatch");
  auto segs = segments(o);
  if (mats.size() != segs.size()) throw CorruptArchive("load_cache: wrong matrix catalog");
  for (size_t i = 0; i < segs.size(); ++i) {
    const auto& [name, r, c, off] = mats[i];
    if (name != segs[i].name || r != segs[i].rows || c != segs[i].cols)
      throw CorruptArchive("load_cache: catalog entry mismatch for " + name);
    const size_t begin = size_t(header + off), bytes = size_t(r * c * 8);
    if (off % 64 != 0 || begin + bytes > all.size()) throw CorruptArchive("load_cache: truncated payload (" + name + ")");
    segs[i].out->resize(size_t(r * c));
    std::memcpy(segs[i].out->data(), all.data() + begin, bytes);
  }
  o.ref_half_side = o.domain_side / double(1 << (o.reference_level + 1));
  ops = std::move(o);
}

}  // namespace kifmm
