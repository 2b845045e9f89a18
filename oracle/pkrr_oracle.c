/*
 * pkrr_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's partitioned Gaussian KRR path
 * (arxiv 1805.00569 reference implementation, /root/reference/proj) used as the
 * parity checker for the sm_100a path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library; the product path in
 * paper_1805_00569_b200/ never links or calls it.
 *
 * Every function restates one reference function in plain C, on DENSE row-major
 * inputs (the reference stores standardized rows densely, dataset.cpp:183-193, so
 * its sparse merge loops reduce to sequential dense loops in index order).  The
 * floating-point operation order is kept identical so that, built with
 * -ffp-contract=off and no -march, results are bitwise equal to the reference
 * library compiled the same way (pinned by tests/test_oracle.py against
 * oracle/_ref and the fixtures in tests/golden/).
 */
#include "pkrr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* RNG: rng.hpp:14-42, rng.cpp:8-63                                          */
/* ------------------------------------------------------------------------ */

#define MT_N 312
#define MT_M 156

/* std::mt19937_64 seeding (the engine is fully specified by the C++ standard;
 * rng.hpp:21 constructs it from the seed). */
void pko_rng_init(pko_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
  r->cached = 0.0;
  r->has_cached = 0;
}

/* rng.hpp:23 next_u64() = eng_() */
uint64_t pko_rng_next(pko_rng* r) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->mti >= MT_N) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_N - MT_M; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < MT_N - 1; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:26 uniform01: 53 random bits */
double pko_uniform01(pko_rng* r) { return (double)(pko_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.cpp:8-17 below(n): rejection sampling, no draw for n <= 1 */
uint64_t pko_below(pko_rng* r, uint64_t n) {
  if (n <= 1) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = pko_rng_next(r);
  } while (x >= limit);
  return x % n;
}

/* rng.cpp:19-32 normal(): Box-Muller, second value cached */
double pko_normal(pko_rng* r) {
  if (r->has_cached) {
    r->has_cached = 0;
    return r->cached;
  }
  const double u1 = 1.0 - pko_uniform01(r);
  const double u2 = pko_uniform01(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  r->cached = radius * sin(angle);
  r->has_cached = 1;
  return radius * cos(angle);
}

static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.cpp:36-56 sub_seed = splitmix64(splitmix64(seed ^ fnv1a64(tag))) */
uint64_t pko_sub_seed(uint64_t seed, const char* tag) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const unsigned char* p = (const unsigned char*)tag; *p; ++p) {
    h ^= *p;
    h *= 0x100000001b3ULL;
  }
  return splitmix64(splitmix64(seed ^ h));
}

/* rng.cpp:58-63 + rng.hpp:33-38: identity then Fisher-Yates, descending */
void pko_random_permutation(uint64_t n, pko_rng* r, uint64_t* perm) {
  for (uint64_t i = 0; i < n; ++i) perm[i] = i;
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = pko_below(r, i);
    const uint64_t t = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = t;
  }
}

/* ------------------------------------------------------------------------ */
/* dense arithmetic primitives: dataset.cpp:32-61                           */
/* ------------------------------------------------------------------------ */

/* dataset.cpp:49-53 squared_norm: sequential sum of v*v */
double pko_squared_norm(const double* x, int64_t d) {
  double s = 0.0;
  for (int64_t k = 0; k < d; ++k) s += x[k] * x[k];
  return s;
}

/* dataset.cpp:32-47 sparse_dot on dense rows: sequential a_k*b_k */
double pko_dot(const double* a, const double* b, int64_t d) {
  double s = 0.0;
  for (int64_t k = 0; k < d; ++k) s += a[k] * b[k];
  return s;
}

/* dataset.cpp:55-61 squared_distance_to_center */
double pko_sqdist_center(const double* x, double x_sq, const double* c, double c_sq,
                         int64_t d) {
  double dot = 0.0;
  for (int64_t k = 0; k < d; ++k) dot += x[k] * c[k];
  const double dist2 = x_sq + c_sq - 2.0 * dot;
  return dist2 < 0.0 ? 0.0 : dist2;
}

/* clustering.cpp:28-32 center_sq_norm */
static double center_sq_norm(const double* c, int64_t d) {
  double s = 0.0;
  for (int64_t k = 0; k < d; ++k) s += c[k] * c[k];
  return s;
}

/* ------------------------------------------------------------------------ */
/* kernel: kernel.cpp:43-59, 81-141                                         */
/* ------------------------------------------------------------------------ */

/* kernel.cpp:52-56: gaussian branch of kernel_eval_cached (a is the first arg) */
double pko_gauss(const double* a, double a_sq, const double* b, double b_sq, int64_t d,
                 double sigma) {
  double dist2 = a_sq + b_sq - 2.0 * pko_dot(a, b, d);
  if (dist2 < 0.0) dist2 = 0.0;
  return exp(-dist2 / (2.0 * sigma * sigma));
}

/* kernel.cpp:81-119: same-set gram, norms first, i<=j computed and mirrored */
void pko_gram_sym(const double* X, int64_t m, int64_t d, double sigma, double* K) {
  double* nrm = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  for (int64_t i = 0; i < m; ++i) nrm[i] = pko_squared_norm(X + i * d, d);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = i; j < m; ++j) {
      const double v = pko_gauss(X + i * d, nrm[i], X + j * d, nrm[j], d, sigma);
      K[i * m + j] = v;
      K[j * m + i] = v;
    }
  free(nrm);
}

/* kernel.cpp:120-129: rectangular gram, K(i,j) = k(A_i, B_j) */
void pko_gram_cross(const double* A, int64_t na, const double* B, int64_t nb, int64_t d,
                    double sigma, double* K) {
  double* an = (double*)malloc(sizeof(double) * (size_t)(na > 0 ? na : 1));
  double* bn = (double*)malloc(sizeof(double) * (size_t)(nb > 0 ? nb : 1));
  for (int64_t i = 0; i < na; ++i) an[i] = pko_squared_norm(A + i * d, d);
  for (int64_t j = 0; j < nb; ++j) bn[j] = pko_squared_norm(B + j * d, d);
  for (int64_t i = 0; i < na; ++i)
    for (int64_t j = 0; j < nb; ++j)
      K[i * nb + j] = pko_gauss(A + i * d, an[i], B + j * d, bn[j], d, sigma);
  free(an);
  free(bn);
}

/* kernel.cpp:134-141 assemble_system: copy K, diag += lambda*mult */
void pko_assemble(const double* K, int64_t m, double lambda, int64_t mult, double* A) {
  memcpy(A, K, sizeof(double) * (size_t)(m * m));
  const double shift = lambda * (double)mult;
  for (int64_t i = 0; i < m; ++i) A[i * m + i] += shift;
}

/* ------------------------------------------------------------------------ */
/* solver: solver.cpp:13-125                                                */
/* ------------------------------------------------------------------------ */

/* solver.cpp:13-44: unblocked right-looking Cholesky in place.
 * Returns 0, or PKO_NPD with *pivot = first column j with !(A_jj > 0). */
int pko_cholesky(double* A, int64_t m, int64_t* pivot, double* pivot_value) {
  double* col = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  for (int64_t j = 0; j < m; ++j) {
    const double p = A[j * m + j];
    if (!(p > 0.0)) {
      if (pivot) *pivot = j;
      if (pivot_value) *pivot_value = p;
      free(col);
      return PKO_NPD;
    }
    const double diag = sqrt(p);
    A[j * m + j] = diag;
    for (int64_t i = j + 1; i < m; ++i) {
      A[i * m + j] /= diag;
      col[i] = A[i * m + j];
    }
    for (int64_t i = j + 1; i < m; ++i) {
      double* row = A + i * m;
      const double lij = col[i];
      for (int64_t k = j + 1; k <= i; ++k) row[k] -= lij * col[k];
    }
    for (int64_t k = j + 1; k < m; ++k) A[j * m + k] = 0.0;
  }
  free(col);
  return 0;
}

/* solver.cpp:46-72: forward row-wise, backward column-strided */
void pko_solve_spd(const double* L, int64_t m, const double* b, double* x) {
  for (int64_t i = 0; i < m; ++i) {
    double sum = b[i];
    const double* row = L + i * m;
    for (int64_t k = 0; k < i; ++k) sum -= row[k] * x[k];
    x[i] = sum / row[i];
  }
  for (int64_t ii = m; ii-- > 0;) {
    double sum = x[ii];
    for (int64_t k = ii + 1; k < m; ++k) sum -= L[k * m + ii] * x[k];
    x[ii] = sum / L[ii * m + ii];
  }
}

/* strategies.cpp:310-320 (grid slice residual): sqrt(res_sq / y_sq) */
double pko_residual_slice(const double* K, int64_t m, double shift, const double* alpha,
                          const double* y) {
  double res_sq = 0.0, y_sq = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double acc = shift * alpha[i] - y[i];
    const double* row = K + i * m;
    for (int64_t j = 0; j < m; ++j) acc += row[j] * alpha[j];
    res_sq += acc * acc;
    y_sq += y[i] * y[i];
  }
  return y_sq > 0.0 ? sqrt(res_sq / y_sq) : sqrt(res_sq);
}

/* solver.cpp:89-125 train_krr (residual formula sqrt(res)/sqrt(y), :119) */
int pko_train_krr(const double* X, const double* y, int64_t m, int64_t d, double sigma,
                  double lambda, double* alpha, double* residual, int64_t* pivot) {
  if (m <= 0 || !(lambda > 0.0)) return PKO_INVALID;
  double* K = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* A = (double*)malloc(sizeof(double) * (size_t)(m * m));
  pko_gram_sym(X, m, d, sigma, K);
  pko_assemble(K, m, lambda, m, A);
  int st = pko_cholesky(A, m, pivot, NULL);
  if (st == 0) {
    pko_solve_spd(A, m, y, alpha);
    const double shift = lambda * (double)m;
    double res_sq = 0.0, y_sq = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = shift * alpha[i] - y[i];
      const double* row = K + i * m;
      for (int64_t j = 0; j < m; ++j) acc += row[j] * alpha[j];
      res_sq += acc * acc;
      y_sq += y[i] * y[i];
    }
    if (residual) *residual = y_sq > 0.0 ? sqrt(res_sq) / sqrt(y_sq) : sqrt(res_sq);
  }
  free(K);
  free(A);
  return st;
}

/* solver.cpp:74-87 KrrModel::predict: sum += alpha_i * k(s_i, x) */
double pko_predict(const double* S, const double* s_sq, const double* alpha, int64_t m,
                   int64_t d, double sigma, const double* x) {
  const double x_sq = pko_squared_norm(x, d);
  double sum = 0.0;
  for (int64_t i = 0; i < m; ++i)
    sum += alpha[i] * pko_gauss(S + i * d, s_sq[i], x, x_sq, d, sigma);
  return sum;
}

/* ------------------------------------------------------------------------ */
/* clustering: clustering.cpp:34-197                                        */
/* ------------------------------------------------------------------------ */

/* clustering.cpp:34-49 recompute_means: row-order sums, then * (1/size) */
static void recompute_means(const double* X, int64_t n, int64_t d, int k,
                            const int32_t* membership, double* centers, int64_t* sizes) {
  memset(centers, 0, sizeof(double) * (size_t)(k * d));
  for (int j = 0; j < k; ++j) sizes[j] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int j = membership[i];
    ++sizes[j];
    const double* r = X + i * d;
    double* c = centers + (int64_t)j * d;
    for (int64_t t = 0; t < d; ++t) c[t] += r[t];
  }
  for (int j = 0; j < k; ++j) {
    if (sizes[j] == 0) continue;
    const double inv = 1.0 / (double)sizes[j];
    double* c = centers + (int64_t)j * d;
    for (int64_t t = 0; t < d; ++t) c[t] *= inv;
  }
}

/* clustering.cpp:53-138 kmeans (Lloyd; uniform distinct-sample init) */
int pko_kmeans(const double* X, int64_t n, int64_t d, int k, uint64_t seed, double threshold,
               int max_iters, int32_t* membership, double* centers, int64_t* sizes,
               int* iterations, double* wcss) {
  if (k < 1 || (int64_t)k > n) return PKO_INVALID;
  for (int64_t i = 0; i < n; ++i) membership[i] = -1;
  for (int j = 0; j < k; ++j) sizes[j] = 0;

  pko_rng rng;
  pko_rng_init(&rng, seed);
  uint64_t* perm = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  pko_random_permutation((uint64_t)n, &rng, perm);
  for (int j = 0; j < k; ++j) memcpy(centers + (int64_t)j * d, X + perm[j] * d, sizeof(double) * (size_t)d);
  free(perm);

  double* x_norms = (double*)malloc(sizeof(double) * (size_t)n);
  double* best = (double*)malloc(sizeof(double) * (size_t)n);
  double* c_norms = (double*)malloc(sizeof(double) * (size_t)k);
  int64_t* sz = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  for (int64_t i = 0; i < n; ++i) x_norms[i] = pko_squared_norm(X + i * d, d);

  int iter = 0;
  for (; iter < max_iters; ++iter) {
    for (int j = 0; j < k; ++j) c_norms[j] = center_sq_norm(centers + (int64_t)j * d, d);
    int64_t changed = 0;
    for (int64_t i = 0; i < n; ++i) {
      double min_d = INFINITY;
      int min_j = 0;
      for (int j = 0; j < k; ++j) {
        const double dist =
            pko_sqdist_center(X + i * d, x_norms[i], centers + (int64_t)j * d, c_norms[j], d);
        if (dist < min_d) {
          min_d = dist;
          min_j = j;
        }
      }
      if (membership[i] != min_j) {
        membership[i] = min_j;
        ++changed;
      }
      best[i] = min_d;
    }
    /* clustering.cpp:98-117 empty-cluster reseed */
    for (int j = 0; j < k; ++j) sz[j] = 0;
    for (int64_t i = 0; i < n; ++i) ++sz[membership[i]];
    for (int j = 0; j < k; ++j) {
      if (sz[j] != 0) continue;
      double far_d = -1.0;
      int64_t far_i = 0;
      for (int64_t i = 0; i < n; ++i) {
        if (sz[membership[i]] <= 1) continue;
        if (best[i] > far_d) {
          far_d = best[i];
          far_i = i;
        }
      }
      --sz[membership[far_i]];
      membership[far_i] = j;
      sz[j] = 1;
      best[far_i] = 0.0;
      ++changed;
    }
    recompute_means(X, n, d, k, membership, centers, sizes);
    if (wcss) {
      double w = 0.0;
      for (int j = 0; j < k; ++j) c_norms[j] = center_sq_norm(centers + (int64_t)j * d, d);
      for (int64_t i = 0; i < n; ++i) {
        const int j = membership[i];
        w += pko_sqdist_center(X + i * d, x_norms[i], centers + (int64_t)j * d, c_norms[j], d);
      }
      wcss[iter] = w;
    }
    if ((double)changed / (double)n <= threshold) {
      ++iter;
      break;
    }
  }
  if (iterations) *iterations = iter;
  free(x_norms);
  free(best);
  free(c_norms);
  free(sz);
  return 0;
}

/* clustering.cpp:140-180 kbalance: kmeans warm start + capacity scan */
int pko_kbalance(const double* X, int64_t n, int64_t d, int k, uint64_t seed, double threshold,
                 int max_iters, int recompute, int32_t* membership, double* centers,
                 int64_t* sizes) {
  if (k < 1 || (int64_t)k > n) return PKO_INVALID;
  int st = pko_kmeans(X, n, d, k, seed, threshold, max_iters, membership, centers, sizes, NULL,
                      NULL);
  if (st) return st;
  const int64_t base = n / k, extra = n % k;
  for (int64_t i = 0; i < n; ++i) membership[i] = -1;
  for (int j = 0; j < k; ++j) sizes[j] = 0;
  int64_t grown = 0;
  double* x_norms = (double*)malloc(sizeof(double) * (size_t)n);
  double* c_norms = (double*)malloc(sizeof(double) * (size_t)k);
  for (int64_t i = 0; i < n; ++i) x_norms[i] = pko_squared_norm(X + i * d, d);
  for (int j = 0; j < k; ++j) c_norms[j] = center_sq_norm(centers + (int64_t)j * d, d);
  for (int64_t i = 0; i < n; ++i) {
    double min_d = INFINITY;
    int min_j = -1;
    for (int j = 0; j < k; ++j) {
      const int open = sizes[j] < base || (sizes[j] == base && grown < extra);
      if (!open) continue;
      const double dist =
          pko_sqdist_center(X + i * d, x_norms[i], centers + (int64_t)j * d, c_norms[j], d);
      if (dist < min_d) {
        min_d = dist;
        min_j = j;
      }
    }
    if (min_j < 0) {
      free(x_norms);
      free(c_norms);
      return PKO_LOGIC;
    }
    if (sizes[min_j] == base) ++grown;
    ++sizes[min_j];
    membership[i] = min_j;
  }
  free(x_norms);
  free(c_norms);
  if (recompute) recompute_means(X, n, d, k, membership, centers, sizes);
  return 0;
}

/* clustering.cpp:182-195 nearest_center (center norms recomputed per call) */
int pko_nearest_center(const double* centers, int k, int64_t d, const double* x) {
  const double x_sq = pko_squared_norm(x, d);
  double min_d = INFINITY;
  int min_j = 0;
  for (int j = 0; j < k; ++j) {
    const double* c = centers + (int64_t)j * d;
    const double dist = pko_sqdist_center(x, x_sq, c, center_sq_norm(c, d), d);
    if (dist < min_d) {
      min_d = dist;
      min_j = j;
    }
  }
  return min_j;
}

/* strategies.cpp:168-177 mse: sequential sum / n */
double pko_mse(const double* pred, const double* truth, int64_t n) {
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double diff = pred[i] - truth[i];
    sum += diff * diff;
  }
  return sum / (double)n;
}

/* ------------------------------------------------------------------------ */
/* strategies: make_partition (strategies.cpp:64-102), grid_search (:343-507) */
/* ------------------------------------------------------------------------ */

static int partitioner_for(int kind) {
  switch (kind) {
    case PKO_EXACT: return 0;            /* whole */
    case PKO_DC: return 1;               /* random */
    case PKO_KK: case PKO_KK2: case PKO_KK3: return 2;  /* kmeans */
    default: return 3;                   /* kbalance */
  }
}

static int predictor_for(int kind) {
  switch (kind) {
    case PKO_EXACT: return 0;                             /* whole */
    case PKO_DC: case PKO_KK: case PKO_BK: return 1;      /* average */
    case PKO_KK2: case PKO_BK2: return 2;                 /* nearest */
    default: return 3;                                    /* oracle */
  }
}

/* Writes part_of[i] (part id per train row), order[] = the parts' rows
 * concatenated part by part in their within-part order (row order for
 * whole/kmeans/kbalance, shuffle order for random: strategies.cpp:82-89,97-99)
 * and, for center-based partitioners, centers[p*d].  Returns the effective p. */
int64_t pko_make_partition(int kind, const double* X, int64_t n, int64_t d, int64_t p,
                           uint64_t seed, int32_t* part_of, int64_t* order, double* centers) {
  const int pk = partitioner_for(kind);
  if (pk == 0) {
    for (int64_t i = 0; i < n; ++i) {
      part_of[i] = 0;
      order[i] = i;
    }
    return 1;
  }
  if (p < 1 || p > n) return -PKO_INVALID;
  if (pk == 1) {
    pko_rng rng;
    pko_rng_init(&rng, seed);
    uint64_t* perm = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
    pko_random_permutation((uint64_t)n, &rng, perm);
    const int64_t base = n / p, extra = n % p;
    int64_t at = 0;
    for (int64_t t = 0; t < p; ++t) {
      const int64_t size = base + (t < extra ? 1 : 0);
      for (int64_t q = 0; q < size; ++q) {
        part_of[perm[at + q]] = (int32_t)t;
        order[at + q] = (int64_t)perm[at + q];
      }
      at += size;
    }
    free(perm);
    return p;
  }
  int64_t* sizes = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  /* make_partition always uses default KMeansParams (strategies.cpp:93-96) */
  int st = pk == 2 ? pko_kmeans(X, n, d, (int)p, seed, 0.01, 100, part_of, centers, sizes, NULL, NULL)
                   : pko_kbalance(X, n, d, (int)p, seed, 0.01, 100, 1, part_of, centers, sizes);
  free(sizes);
  if (st) return -st;
  int64_t at = 0;
  for (int64_t t = 0; t < p; ++t)
    for (int64_t i = 0; i < n; ++i)
      if (part_of[i] == t) order[at++] = i;
  return p;
}

/* grid_search with the partition supplied (part_of/centers, p parts).
 * Outputs per cell (lambda-major, li*ns+si): mse, failed, max residual;
 * returns best index (first strict min over non-failed) or -1. */
int64_t pko_grid_search_parts(int kind, const double* Xtr, const double* ytr, int64_t n,
                              int64_t d, const double* Xte, const double* yte, int64_t t,
                              int64_t p, const int32_t* part_of, const int64_t* order,
                              const double* centers,
                              const double* lambdas, int64_t nl, const double* sigmas,
                              int64_t ns, double* cell_mse, uint8_t* cell_failed,
                              double* cell_residual, double* best_pred) {
  const int pred_kind = predictor_for(kind);
  /* parts in train row order (strategies.cpp:97-99) */
  int64_t* psize = (int64_t*)calloc((size_t)p, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) psize[part_of[i]]++;
  int64_t** rows = (int64_t**)malloc(sizeof(int64_t*) * (size_t)p);
  int64_t* fill = (int64_t*)calloc((size_t)p, sizeof(int64_t));
  for (int64_t q = 0; q < p; ++q) rows[q] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(psize[q] + 1));
  for (int64_t q = 0; q < n; ++q) {
    const int64_t i = order[q];
    rows[part_of[i]][fill[part_of[i]]++] = i;
  }
  /* targets (strategies.cpp:370-381) */
  int64_t* tsize = (int64_t*)calloc((size_t)p, sizeof(int64_t));
  int64_t** targets = (int64_t**)malloc(sizeof(int64_t*) * (size_t)p);
  if (pred_kind == 2) {
    int32_t* route = (int32_t*)malloc(sizeof(int32_t) * (size_t)t);
    for (int64_t j = 0; j < t; ++j) {
      route[j] = pko_nearest_center(centers, (int)p, d, Xte + j * d);
      tsize[route[j]]++;
    }
    for (int64_t q = 0; q < p; ++q) targets[q] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(tsize[q] + 1));
    memset(fill, 0, sizeof(int64_t) * (size_t)p);
    for (int64_t j = 0; j < t; ++j) targets[route[j]][fill[route[j]]++] = j;
    free(route);
  } else {
    for (int64_t q = 0; q < p; ++q) {
      tsize[q] = t;
      targets[q] = (int64_t*)malloc(sizeof(int64_t) * (size_t)t);
      for (int64_t j = 0; j < t; ++j) targets[q][j] = j;
    }
  }
  const int64_t ncell = nl * ns;
  for (int64_t c = 0; c < ncell; ++c) {
    cell_mse[c] = NAN;
    cell_failed[c] = 0;
    cell_residual[c] = 0.0;
  }
  /* predictions per (part, lambda) for the current sigma */
  double** preds = (double**)malloc(sizeof(double*) * (size_t)(p * nl));
  uint8_t* slice_failed = (uint8_t*)malloc((size_t)(p * nl));
  double* pred = (double*)malloc(sizeof(double) * (size_t)t);
  int64_t best = -1;
  double* best_cell_pred = (double*)malloc(sizeof(double) * (size_t)t);
  double* all_pred = (double*)malloc(sizeof(double) * (size_t)(ncell * t));
  for (int64_t si = 0; si < ns; ++si) {
    const double sigma = sigmas[si];
    for (int64_t q = 0; q < p; ++q) {
      const int64_t m = psize[q], tt = tsize[q];
      double* Xp = (double*)malloc(sizeof(double) * (size_t)(m * d));
      double* yp = (double*)malloc(sizeof(double) * (size_t)m);
      for (int64_t i = 0; i < m; ++i) {
        memcpy(Xp + i * d, Xtr + rows[q][i] * d, sizeof(double) * (size_t)d);
        yp[i] = ytr[rows[q][i]];
      }
      double* K = (double*)malloc(sizeof(double) * (size_t)(m * m));
      pko_gram_sym(Xp, m, d, sigma, K);
      /* cross(j,i) = k(part_i, test_j)  (strategies.cpp:284-294) */
      double* pn = (double*)malloc(sizeof(double) * (size_t)m);
      double* tn = (double*)malloc(sizeof(double) * (size_t)(tt + 1));
      for (int64_t i = 0; i < m; ++i) pn[i] = pko_squared_norm(Xp + i * d, d);
      for (int64_t j = 0; j < tt; ++j) tn[j] = pko_squared_norm(Xte + targets[q][j] * d, d);
      double* cross = (double*)malloc(sizeof(double) * (size_t)(tt * m + 1));
      for (int64_t j = 0; j < tt; ++j)
        for (int64_t i = 0; i < m; ++i)
          cross[j * m + i] = pko_gauss(Xp + i * d, pn[i], Xte + targets[q][j] * d, tn[j], d, sigma);
      double* A = (double*)malloc(sizeof(double) * (size_t)(m * m));
      double* alpha = (double*)malloc(sizeof(double) * (size_t)m);
      for (int64_t li = 0; li < nl; ++li) {
        double* pr = (double*)malloc(sizeof(double) * (size_t)(tt + 1));
        preds[q * nl + li] = pr;
        pko_assemble(K, m, lambdas[li], m, A);
        int64_t piv = 0;
        if (pko_cholesky(A, m, &piv, NULL) != 0) {
          slice_failed[q * nl + li] = 1;
          continue;
        }
        slice_failed[q * nl + li] = 0;
        pko_solve_spd(A, m, yp, alpha);
        const double res = pko_residual_slice(K, m, lambdas[li] * (double)m, alpha, yp);
        const int64_t c = li * ns + si;
        if (res > cell_residual[c]) cell_residual[c] = res;
        for (int64_t j = 0; j < tt; ++j) {
          const double* row = cross + j * m;
          double acc = 0.0;
          for (int64_t i = 0; i < m; ++i) acc += row[i] * alpha[i];
          pr[j] = acc;
        }
      }
      free(Xp); free(yp); free(K); free(pn); free(tn); free(cross); free(A); free(alpha);
    }
    for (int64_t li = 0; li < nl; ++li) {
      const int64_t c = li * ns + si;
      for (int64_t q = 0; q < p; ++q)
        if (slice_failed[q * nl + li]) cell_failed[c] = 1;
      if (!cell_failed[c]) {
        /* combine in fixed partition order (strategies.cpp:458-495) */
        if (pred_kind == 0) {
          memcpy(pred, preds[li], sizeof(double) * (size_t)t);
        } else if (pred_kind == 1) {
          for (int64_t j = 0; j < t; ++j) pred[j] = 0.0;
          for (int64_t q = 0; q < p; ++q)
            for (int64_t j = 0; j < t; ++j) pred[j] += preds[q * nl + li][j];
          const double inv_p = 1.0 / (double)p;
          for (int64_t j = 0; j < t; ++j) pred[j] *= inv_p;
        } else if (pred_kind == 2) {
          for (int64_t q = 0; q < p; ++q)
            for (int64_t j = 0; j < tsize[q]; ++j) pred[targets[q][j]] = preds[q * nl + li][j];
        } else {
          for (int64_t j = 0; j < t; ++j) {
            double bp = 0.0, be = INFINITY;
            for (int64_t q = 0; q < p; ++q) {
              const double v = preds[q * nl + li][j];
              const double err = (v - yte[j]) * (v - yte[j]);
              if (err < be) {
                be = err;
                bp = v;
              }
            }
            pred[j] = bp;
          }
        }
        cell_mse[c] = pko_mse(pred, yte, t);
        memcpy(all_pred + c * t, pred, sizeof(double) * (size_t)t);
      }
      for (int64_t q = 0; q < p; ++q) free(preds[q * nl + li]);
    }
  }
  for (int64_t c = 0; c < ncell; ++c) {
    if (cell_failed[c]) continue;
    if (best < 0 || cell_mse[c] < cell_mse[best]) best = c;
  }
  if (best >= 0 && best_pred) memcpy(best_pred, all_pred + best * t, sizeof(double) * (size_t)t);
  for (int64_t q = 0; q < p; ++q) {
    free(rows[q]);
    free(targets[q]);
  }
  free(rows); free(targets); free(psize); free(tsize); free(fill); free(preds);
  free(slice_failed); free(pred); free(best_cell_pred); free(all_pred);
  return best;
}

/* strategies.cpp:343-507 grid_search: partition once, then the cell loop. */
int64_t pko_grid_search(int kind, const double* Xtr, const double* ytr, int64_t n, int64_t d,
                        const double* Xte, const double* yte, int64_t t, int64_t p,
                        const double* lambdas, int64_t nl, const double* sigmas, int64_t ns,
                        uint64_t seed, double* cell_mse, uint8_t* cell_failed,
                        double* cell_residual, int32_t* part_of, double* centers,
                        double* best_pred) {
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  const int64_t pe = pko_make_partition(kind, Xtr, n, d, p, seed, part_of, order, centers);
  if (pe < 0) {
    free(order);
    return -2;
  }
  const int64_t best = pko_grid_search_parts(kind, Xtr, ytr, n, d, Xte, yte, t, pe, part_of, order,
                                             centers, lambdas, nl, sigmas, ns, cell_mse, cell_failed,
                                             cell_residual, best_pred);
  free(order);
  return best;
}

/* ------------------------------------------------------------------------ */
/* data preparation                                                         */
/* ------------------------------------------------------------------------ */

/* dataset.cpp:199-232 standardize + apply_feature_stats :178-197, dense rows:
   row-order sums over the stored entries, divisor n, variance clamped at 0 */
void pko_standardize(const double* Xtr, int64_t n, int64_t d, const double* Xte, int64_t t,
                     double* Xtr_out, double* Xte_out, double* mean, double* stddev) {
  double* sum = (double*)calloc((size_t)d, sizeof(double));
  double* sq = (double*)calloc((size_t)d, sizeof(double));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < d; ++j) {
      const double v = Xtr[i * d + j];
      sum[j] += v;
      sq[j] += v * v;
    }
  const double inv_n = 1.0 / (double)n;
  for (int64_t j = 0; j < d; ++j) {
    mean[j] = sum[j] * inv_n;
    double var = sq[j] * inv_n - mean[j] * mean[j];
    if (var < 0.0) var = 0.0;
    stddev[j] = sqrt(var);
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < d; ++j)
      Xtr_out[i * d + j] = stddev[j] == 0.0 ? 0.0 : (Xtr[i * d + j] - mean[j]) / stddev[j];
  for (int64_t i = 0; i < t; ++i)
    for (int64_t j = 0; j < d; ++j)
      Xte_out[i * d + j] = stddev[j] == 0.0 ? 0.0 : (Xte[i * d + j] - mean[j]) / stddev[j];
  free(sum);
  free(sq);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* strategies.cpp:204-234 auto_sigma_grid */
void pko_auto_sigma_grid(const double* X, int64_t n, int64_t d, uint64_t seed, double* grid9) {
  const int64_t count = n < 512 ? n : 512;
  pko_rng rng;
  pko_rng_init(&rng, pko_sub_seed(seed, "sigma-grid"));
  uint64_t* perm = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
  pko_random_permutation((uint64_t)n, &rng, perm);
  double* norms = (double*)malloc(sizeof(double) * (size_t)(count > 0 ? count : 1));
  for (int64_t i = 0; i < count; ++i) norms[i] = pko_squared_norm(X + perm[i] * d, d);
  const int64_t np = count * (count - 1) / 2;
  double* dists = (double*)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1));
  int64_t e = 0;
  for (int64_t i = 0; i < count; ++i)
    for (int64_t j = i + 1; j < count; ++j) {
      double d2 = norms[i] + norms[j] - 2.0 * pko_dot(X + perm[i] * d, X + perm[j] * d, d);
      if (d2 < 0.0) d2 = 0.0;
      dists[e++] = sqrt(d2);
    }
  double g = 1.0;
  if (np > 0) {
    qsort(dists, (size_t)np, sizeof(double), cmp_double);
    const double median = dists[(np - 1) / 2];
    if (median > 0.0) g = median;
  }
  for (int k = -4; k <= 4; ++k) grid9[k + 4] = g * ldexp(1.0, k);
  free(perm);
  free(norms);
  free(dists);
}
