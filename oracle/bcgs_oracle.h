/* TEST INFRASTRUCTURE — NOT THE PRODUCT.
 *
 * CPU restatement ("oracle") of the reference's BCGS QR hot path
 * (/root/reference/proj/src/{bcgs,intraorth,tsqr_tree,dense_kernels,exact_sum,
 * dist_block,matrix_gen,metrics,variant,cost_model}.cpp), written from scratch in C.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it, and only as the checker.  The product path
 * (paper_2507_21791_b200/) never links, loads or calls it.
 *
 * Pinning: tests/test_oracle_pin.py checks this restatement BITWISE against the
 * reference library itself (oracle/_ref/libblockgs_ref.so built by oracle/Makefile from
 * /root/reference) and against committed golden fixtures in tests/golden/.
 *
 * All matrices are column-major with leading dimension = rows.
 * Variant ids follow blockgs::VariantId order (variant.hpp:8-15):
 *   0 BCGS (not supported here: out of scope), 1 BCGSI+, 2 BCGSPIPI+,
 *   3 BCGSI+P-1S, 4 BCGSI+P-2S, 5 BCGSI+1S.
 * Error codes (same as include/bgs_gpu.h):
 *   0 ok, 1 Dimension, 2 NotSpd, 3 Singular, 4 RankDeficient, 5 NonFinite,
 *   6 Collective, 7 Config, 8 other.
 */
#ifndef BCGS_ORACLE_H
#define BCGS_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  long sync_count;
  long words_reduced;
  int n_events;
  char labels[64 * 1024]; /* '\n'-joined event labels, issue order */
  int pivot;              /* NotSpd: 1-based pivot */
  char msg[1024];         /* error text (reference wording) */
} or_stats;

int or_gen_matrix(long n, long m, long s, double kappa, unsigned long long seed, int dist,
                  double* x);
int or_factor(int variant, const double* x, long n, long m, long s, int procs, double* q,
              double* r, or_stats* st);
void or_gram(const double* a, long n, long ma, const double* b, long mb, double* out);
int or_householder(const double* x, long rows, long cols, double* q, double* r);
double or_loo(const double* q, long n, long m);
double or_residual(const double* x, const double* q, const double* r, long n, long m);
double or_variant_flops(int variant, long n, long m, long s);
long or_expected_syncs(int variant, long q);
int or_chol(const double* a, long n, double* g, int* pivot);

#ifdef __cplusplus
}
#endif
#endif
