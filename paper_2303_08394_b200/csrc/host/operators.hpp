// Precomputed KIFMM operators (design 501-504).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace kifmm {

struct Operators {
  int p = 0, n_e = 0, n_c = 0;
  int reference_level = 2;
  double alpha_inner = 1.05, alpha_outer = 2.95, svd_cutoff = 1e-12;
  double domain_side = 1.0, ref_half_side = 0.125;
  std::vector<double> surface;       // n_e x 3
  int uc2e_rank = 0;
  std::vector<double> uc2e_u, uc2e_s, uc2e_v;  // n_c x k, k, n_e x k
  int dc2e_rank = 0;
  std::vector<double> dc2e_u, dc2e_s, dc2e_v;
  std::vector<double> m2m, l2l;      // 8 x n_e x n_e
  std::vector<double> m2l;           // 316 x n_c x n_e
  uint64_t fingerprint = 0;
};

int surface_count(int p);
std::vector<double> surface_grid(int p);
void kernel_matrix(const double* src, int64_t m, const double* tgt, int64_t k, double* out);
// One-sided Jacobi SVD, a: m x n row-major (m >= n). Singular values descending.
// threads > 1: the disjoint column pairs of each round-robin round rotate in parallel (same result for any count)
void jacobi_svd(const double* a, int m, int n, double* u, double* s, double* v, int threads = 1);
uint64_t operator_fingerprint(int p, double ai, double ao, double cutoff, double side);
void precompute(Operators& ops, int p, double alpha_inner, double alpha_outer, double svd_cutoff,
                double domain_side, int threads);
void save_operators(const Operators& ops, const std::string& path);
void load_operators(Operators& ops, const std::string& path, uint64_t expected_fingerprint);

}  // namespace kifmm
