/* pkrr_oracle.h -- TEST INFRASTRUCTURE ONLY (see pkrr_oracle.c header). */
#ifndef PKRR_ORACLE_H
#define PKRR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PKO_OK = 0, PKO_INVALID = 1, PKO_NPD = 2, PKO_LOGIC = 4 };
/* StrategyKind order of strategies.hpp:21 */
enum { PKO_EXACT = 0, PKO_DC, PKO_KK, PKO_KK2, PKO_KK3, PKO_BK, PKO_BK2, PKO_BK3 };

typedef struct {
  uint64_t mt[312];
  int mti;
  double cached;
  int has_cached;
} pko_rng;

void pko_rng_init(pko_rng* r, uint64_t seed);
uint64_t pko_rng_next(pko_rng* r);
double pko_uniform01(pko_rng* r);
uint64_t pko_below(pko_rng* r, uint64_t n);
double pko_normal(pko_rng* r);
uint64_t pko_sub_seed(uint64_t seed, const char* tag);
void pko_random_permutation(uint64_t n, pko_rng* r, uint64_t* perm);

double pko_squared_norm(const double* x, int64_t d);
double pko_dot(const double* a, const double* b, int64_t d);
double pko_sqdist_center(const double* x, double x_sq, const double* c, double c_sq, int64_t d);
double pko_gauss(const double* a, double a_sq, const double* b, double b_sq, int64_t d,
                 double sigma);
void pko_gram_sym(const double* X, int64_t m, int64_t d, double sigma, double* K);
void pko_gram_cross(const double* A, int64_t na, const double* B, int64_t nb, int64_t d,
                    double sigma, double* K);
void pko_assemble(const double* K, int64_t m, double lambda, int64_t mult, double* A);
int pko_cholesky(double* A, int64_t m, int64_t* pivot, double* pivot_value);
void pko_solve_spd(const double* L, int64_t m, const double* b, double* x);
double pko_residual_slice(const double* K, int64_t m, double shift, const double* alpha,
                          const double* y);
int pko_train_krr(const double* X, const double* y, int64_t m, int64_t d, double sigma,
                  double lambda, double* alpha, double* residual, int64_t* pivot);
double pko_predict(const double* S, const double* s_sq, const double* alpha, int64_t m,
                   int64_t d, double sigma, const double* x);
int pko_kmeans(const double* X, int64_t n, int64_t d, int k, uint64_t seed, double threshold,
               int max_iters, int32_t* membership, double* centers, int64_t* sizes,
               int* iterations, double* wcss);
int pko_kbalance(const double* X, int64_t n, int64_t d, int k, uint64_t seed, double threshold,
                 int max_iters, int recompute, int32_t* membership, double* centers,
                 int64_t* sizes);
int pko_nearest_center(const double* centers, int k, int64_t d, const double* x);
double pko_mse(const double* pred, const double* truth, int64_t n);
int64_t pko_make_partition(int kind, const double* X, int64_t n, int64_t d, int64_t p,
                           uint64_t seed, int32_t* part_of, int64_t* order, double* centers);
int64_t pko_grid_search_parts(int kind, const double* Xtr, const double* ytr, int64_t n,
                              int64_t d, const double* Xte, const double* yte, int64_t t,
                              int64_t p, const int32_t* part_of, const int64_t* order,
                              const double* centers,
                              const double* lambdas, int64_t nl, const double* sigmas,
                              int64_t ns, double* cell_mse, uint8_t* cell_failed,
                              double* cell_residual, double* best_pred);
int64_t pko_grid_search(int kind, const double* Xtr, const double* ytr, int64_t n, int64_t d,
                        const double* Xte, const double* yte, int64_t t, int64_t p,
                        const double* lambdas, int64_t nl, const double* sigmas, int64_t ns,
                        uint64_t seed, double* cell_mse, uint8_t* cell_failed,
                        double* cell_residual, int32_t* part_of, double* centers,
                        double* best_pred);

/* data preparation: dataset.cpp:199-232, strategies.cpp:204-234 */
void pko_standardize(const double* Xtr, int64_t n, int64_t d, const double* Xte, int64_t t,
                     double* Xtr_out, double* Xte_out, double* mean, double* stddev);
void pko_auto_sigma_grid(const double* X, int64_t n, int64_t d, uint64_t seed, double* grid9);

#ifdef __cplusplus
}
#endif
#endif
