/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for C = A*B of block-sparse
 * matrices (arXiv 1501.07800, Rubensson & Rudberg).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, header or table with the CUDA
 * path in paper_1501_07800_b200/.
 *
 * What it computes (the plain definition the method reaches exactly, up to
 * rounding order; SURVEY.md §8(c) "Definition"):
 *   pattern  S_C = { (I,J) : exists K with (I,K) in S_A and (K,J) in S_B }
 *            (zero submatrices are skipped at every level and nothing else is
 *            dropped: §3.2 "sparsity is dynamically
 *            exploited ... by skipping operations on zero submatrices";
 *            DESIGN.md reading C-1 "structural pattern")
 *   values   C(I,J) = sum over K ascending of A(I,K) * B(K,J)
 *            (the leaf product is a sum of outer products over the inner block
 *            index, PAPER.md P:381-388 Fig. fig:block-sparse-mmul; summation
 *            order "ascending global k" is DESIGN.md reading C-5).
 *
 * Algorithm: block-CSR Gustavson with a dense marker over block columns.
 * Each block product is the textbook triple loop c[i][j] += a[i][k]*b[k][j].
 * Compile with -ffp-contract=off so every multiply and add is rounded
 * separately.  Threads (pthreads) split block rows; each output block is
 * produced by exactly one thread, so results do not depend on the thread
 * count.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- symbolic */

/* Count C blocks per block row: c_cnt[I] = |{J : exists K, A(I,K), B(K,J)}|.
 * marker: caller-free scratch.  Returns total number of C blocks. */
/* Norm screening (the optional last three arguments of oracle_symbolic and
 * oracle_numeric): the block product A(I,K) B(K,J) is taken iff
 * na2[p] * nb2[q] >= tau2, with na2/nb2 the squared Frobenius norms of the
 * blocks (oracle_block_norm2) — the definition of the screened product C~. */
static int keep_product(const double* na2, const double* nb2, double tau2, int64_t p, int64_t q) {
  return !na2 || na2[p] * nb2[q] >= tau2;
}

int64_t oracle_symbolic(int32_t nbr, const int64_t* a_ptr, const int32_t* a_col,
                        int32_t nbk, const int64_t* b_ptr, const int32_t* b_col,
                        int32_t nbc, int64_t* c_cnt, const double* na2, const double* nb2,
                        double tau2) {
  (void)nbk;
  int32_t* marker = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nbc > 0 ? nbc : 1));
  for (int32_t j = 0; j < nbc; ++j) marker[j] = -1;
  int64_t total = 0;
  for (int32_t I = 0; I < nbr; ++I) {
    int64_t cnt = 0;
    for (int64_t p = a_ptr[I]; p < a_ptr[I + 1]; ++p) {
      int32_t K = a_col[p];
      for (int64_t q = b_ptr[K]; q < b_ptr[K + 1]; ++q) {
        if (!keep_product(na2, nb2, tau2, p, q)) continue;
        int32_t J = b_col[q];
        if (marker[J] != I) { marker[J] = I; ++cnt; }
      }
    }
    c_cnt[I] = cnt;
    total += cnt;
  }
  free(marker);
  return total;
}

static int cmp_i32(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  return (a > b) - (a < b);
}

/* ----------------------------------------------------------------- numeric */

typedef struct {
  const double *na2, *nb2;
  double tau2;
  int32_t nbr, nbc, bs;
  const int64_t *a_ptr, *b_ptr, *c_ptr;
  const int32_t *a_col, *b_col;
  const double *a_val, *b_val;
  int32_t* c_col;
  double* c_val;
  int32_t row_lo, row_hi, nthreads, tid;
} job_t;

/* One block row I of C: columns (sorted ascending) and values. */
static void row_product(const job_t* jb, int32_t I, int32_t* pos_of) {
  const int32_t bs = jb->bs;
  const int64_t bb = (int64_t)bs * bs;
  int64_t c0 = jb->c_ptr[I], nc = 0;
  int32_t* ccol = jb->c_col + c0;
  /* 1. the set of output block columns of this row */
  for (int64_t p = jb->a_ptr[I]; p < jb->a_ptr[I + 1]; ++p) {
    int32_t K = jb->a_col[p];
    for (int64_t q = jb->b_ptr[K]; q < jb->b_ptr[K + 1]; ++q) {
      if (!keep_product(jb->na2, jb->nb2, jb->tau2, p, q)) continue;
      int32_t J = jb->b_col[q];
      if (pos_of[J] != -2 - I) { pos_of[J] = -2 - I; ccol[nc++] = J; }
    }
  }
  qsort(ccol, (size_t)nc, sizeof(int32_t), cmp_i32);
  for (int64_t t = 0; t < nc; ++t) pos_of[ccol[t]] = (int32_t)t;
  double* cv = jb->c_val + c0 * bb;
  memset(cv, 0, sizeof(double) * (size_t)(nc * bb));
  /* 2. accumulate A(I,K)*B(K,J) for K ascending (a_col is sorted) */
  for (int64_t p = jb->a_ptr[I]; p < jb->a_ptr[I + 1]; ++p) {
    int32_t K = jb->a_col[p];
    const double* a = jb->a_val + p * bb;
    for (int64_t q = jb->b_ptr[K]; q < jb->b_ptr[K + 1]; ++q) {
      if (!keep_product(jb->na2, jb->nb2, jb->tau2, p, q)) continue;
      int32_t J = jb->b_col[q];
      const double* b = jb->b_val + q * bb;
      double* c = cv + (int64_t)pos_of[J] * bb;
      for (int32_t i = 0; i < bs; ++i)
        for (int32_t k = 0; k < bs; ++k) {
          double aik = a[i * bs + k];
          for (int32_t j = 0; j < bs; ++j) c[i * bs + j] += aik * b[k * bs + j];
        }
    }
  }
  /* reset markers of this row so the next row starts clean */
  for (int64_t t = 0; t < nc; ++t) pos_of[ccol[t]] = -1;
}

static void* worker(void* arg) {
  job_t* jb = (job_t*)arg;
  int32_t* pos_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(jb->nbc > 0 ? jb->nbc : 1));
  for (int32_t j = 0; j < jb->nbc; ++j) pos_of[j] = -1;
  for (int32_t I = jb->row_lo + jb->tid; I < jb->row_hi; I += jb->nthreads)
    row_product(jb, I, pos_of);
  free(pos_of);
  return NULL;
}

/* Numeric product for block rows [row_lo, row_hi).
 * c_ptr: exclusive prefix of oracle_symbolic's counts (length nbr+1);
 * c_col / c_val are written at c_ptr[I] for the rows in range.
 * nthreads <= 0 means 1. */
void oracle_numeric(int32_t nbr, int32_t bs,
                    const int64_t* a_ptr, const int32_t* a_col, const double* a_val,
                    const int64_t* b_ptr, const int32_t* b_col, const double* b_val,
                    int32_t nbc, const int64_t* c_ptr, int32_t* c_col, double* c_val,
                    int32_t row_lo, int32_t row_hi, int32_t nthreads, const double* na2,
                    const double* nb2, double tau2) {
  if (nthreads <= 0) nthreads = 1;
  if (row_lo < 0) row_lo = 0;
  if (row_hi > nbr) row_hi = nbr;
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)nthreads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int32_t t = 0; t < nthreads; ++t) {
    job_t j = {na2, nb2, tau2, nbr, nbc, bs, a_ptr, b_ptr, c_ptr, a_col, b_col, a_val, b_val,
               c_col, c_val, row_lo, row_hi, nthreads, t};
    jobs[t] = j;
  }
  if (nthreads == 1) {
    worker(&jobs[0]);
  } else {
    for (int32_t t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &jobs[t]);
    for (int32_t t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  free(th);
  free(jobs);
}

/* Squared Frobenius norm of each bs x bs block: row-major, one rounding per
 * multiply and per add (compiled with -ffp-contract=off). */
void oracle_block_norm2(int64_t nb, int32_t bs, const double* vals, double* out) {
  const int64_t bb = (int64_t)bs * bs;
  for (int64_t t = 0; t < nb; ++t) {
    double s = 0.0;
    for (int64_t e = 0; e < bb; ++e) {
      double v = vals[t * bb + e];
      s += v * v;
    }
    out[t] = s;
  }
}

/* -------------------------------------------------- dense brute force (i) */

/* C = A*B for dense row-major n x n matrices, textbook i-j-k triple loop with
 * k ascending.  Tiny n only. */
void oracle_dense(int32_t n, const double* A, const double* B, double* C) {
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int32_t k = 0; k < n; ++k) s += A[(int64_t)i * n + k] * B[(int64_t)k * n + j];
      C[(int64_t)i * n + j] = s;
    }
}
