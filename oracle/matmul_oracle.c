/*
 * oracle/matmul_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement of the matrix application that the reference tunes
 * (/root/reference/proj/fixtures/matmul.c:7-35), with a runtime matrix size and
 * heap arrays instead of the fixture's compile-time `#define N 256` (matmul.c:3)
 * and static arrays (matmul.c:5).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's library.
 * The product (paper_1806_01430_b200/csrc) never links or calls it.
 *
 * Parity pin: oracle/ref_fixture_harness.c compiles the reference fixture itself
 * (unmodified, from where it lies) and tests/test_oracle.py checks that this
 * restatement reproduces its a, b, bt, c arrays bit for bit at the fixture size
 * N=256 (golden hashes committed in tests/golden/fixture_n256.json).
 *
 * Arithmetic contract (must match `gcc -O2` on baseline x86-64, which has no FMA
 * and therefore never contracts a*b+c): every nest keeps the fixture's loop
 * order; the matmul inner loop runs k ascending with a separate multiply and
 * add.  Build with -O2 -ffp-contract=off (see oracle/Makefile).
 *
 * The float flavour is the same program with every `double` replaced by `float`
 * (the reference ships only the double program; BASELINE.json asks for FP32 too).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define MMO_API __attribute__((visibility("default")))

/* nest ids, in program order (matmul.c line of the outer `for`) */
enum { MMO_INIT_A = 0 /* :8 */, MMO_INIT_B = 1 /* :12 */, MMO_ZERO_C = 2 /* :16 */,
       MMO_TRANSPOSE = 3 /* :21 */, MMO_MATMUL = 4 /* :25 */, MMO_TRACE = 5 /* :31 */ };

/* ---- one row-range of each nest, both precisions ------------------------------- */

#define DEFINE_NESTS(T, SFX)                                                              \
  /* matmul.c:8-10  a[i][j] = (T)(i + j) / N */                                           \
  static void init_a_##SFX(T* a, int n, int r0, int r1) {                                 \
    for (int i = r0; i < r1; i++)                                                         \
      for (int j = 0; j < n; j++) a[(size_t)i * n + j] = (T)(i + j) / n;                  \
  }                                                                                       \
  /* matmul.c:12-14 b[i][j] = (T)(i - j) / N */                                           \
  static void init_b_##SFX(T* b, int n, int r0, int r1) {                                 \
    for (int i = r0; i < r1; i++)                                                         \
      for (int j = 0; j < n; j++) b[(size_t)i * n + j] = (T)(i - j) / n;                  \
  }                                                                                       \
  /* matmul.c:16-18 c[i][j] = 0.0 */                                                      \
  static void zero_c_##SFX(T* c, int n, int r0, int r1) {                                 \
    for (int i = r0; i < r1; i++)                                                         \
      for (int j = 0; j < n; j++) c[(size_t)i * n + j] = (T)0.0;                          \
  }                                                                                       \
  /* matmul.c:21-23 bt[i][j] = b[j][i] */                                                 \
  static void transpose_##SFX(T* bt, const T* b, int n, int r0, int r1) {                 \
    for (int i = r0; i < r1; i++)                                                         \
      for (int j = 0; j < n; j++) bt[(size_t)i * n + j] = b[(size_t)j * n + i];           \
  }                                                                                       \
  /* matmul.c:25-28 c[i][j] += a[i][k] * bt[j][k], k ascending, mul then add */           \
  static void matmul_##SFX(T* c, const T* a, const T* bt, int n, int r0, int r1) {        \
    for (int i = r0; i < r1; i++)                                                         \
      for (int j = 0; j < n; j++)                                                         \
        for (int k = 0; k < n; k++)                                                       \
          c[(size_t)i * n + j] += a[(size_t)i * n + k] * bt[(size_t)j * n + k];           \
  }                                                                                       \
  /* matmul.c:30-32 sum += c[i][i] ; always accumulated in the array's type... */        \
  static double trace_##SFX(const T* c, int n) {                                          \
    T sum = (T)0.0;                                                                       \
    for (int i = 0; i < n; i++) sum += c[(size_t)i * n + i];                              \
    return (double)sum;                                                                   \
  }

DEFINE_NESTS(double, f64)
DEFINE_NESTS(float, f32)

/* ---- row-parallel driver (same per-element arithmetic, so same bits) ----------- */

typedef struct {
  int nest, dtype, n, r0, r1;
  void *a, *b, *c, *bt;
} mmo_job;

static void run_rows(const mmo_job* j) {
  if (j->dtype == 0) {
    switch (j->nest) {
      case MMO_INIT_A: init_a_f64(j->a, j->n, j->r0, j->r1); break;
      case MMO_INIT_B: init_b_f64(j->b, j->n, j->r0, j->r1); break;
      case MMO_ZERO_C: zero_c_f64(j->c, j->n, j->r0, j->r1); break;
      case MMO_TRANSPOSE: transpose_f64(j->bt, j->b, j->n, j->r0, j->r1); break;
      case MMO_MATMUL: matmul_f64(j->c, j->a, j->bt, j->n, j->r0, j->r1); break;
    }
  } else {
    switch (j->nest) {
      case MMO_INIT_A: init_a_f32(j->a, j->n, j->r0, j->r1); break;
      case MMO_INIT_B: init_b_f32(j->b, j->n, j->r0, j->r1); break;
      case MMO_ZERO_C: zero_c_f32(j->c, j->n, j->r0, j->r1); break;
      case MMO_TRANSPOSE: transpose_f32(j->bt, j->b, j->n, j->r0, j->r1); break;
      case MMO_MATMUL: matmul_f32(j->c, j->a, j->bt, j->n, j->r0, j->r1); break;
    }
  }
}

static void* thread_main(void* p) {
  run_rows((const mmo_job*)p);
  return NULL;
}

/*
 * Run rows [r0, r1) of one of the five matrix nests with `threads` workers
 * (contiguous row blocks).  dtype: 0 = double, 1 = float.  Returns 0, or -1 on
 * bad arguments.  The trace nest is sequential: use mmo_trace.
 */
MMO_API int mmo_run_nest(int nest, int dtype, int n, int r0, int r1, int threads, void* a,
                         void* b, void* c, void* bt) {
  if (nest < MMO_INIT_A || nest > MMO_MATMUL || n <= 0 || r0 < 0 || r1 > n || r0 > r1) return -1;
  if (dtype != 0 && dtype != 1) return -1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  const int rows = r1 - r0;
  if (threads > rows) threads = rows > 0 ? rows : 1;
  mmo_job jobs[256];
  pthread_t tid[256];
  for (int t = 0; t < threads; t++) {
    jobs[t] = (mmo_job){nest, dtype, n, r0 + (int)((long long)rows * t / threads),
                        r0 + (int)((long long)rows * (t + 1) / threads), a, b, c, bt};
  }
  if (threads == 1) {
    run_rows(&jobs[0]);
    return 0;
  }
  for (int t = 0; t < threads; t++) pthread_create(&tid[t], NULL, thread_main, &jobs[t]);
  for (int t = 0; t < threads; t++) pthread_join(tid[t], NULL);
  return 0;
}

MMO_API double mmo_trace(int dtype, int n, const void* c) {
  return dtype == 0 ? trace_f64((const double*)c, n) : trace_f32((const float*)c, n);
}

/* Whole program, matmul.c:8-32, returning the value its printf would print. */
MMO_API double mmo_app(int dtype, int n, int threads, void* a, void* b, void* c, void* bt) {
  for (int nest = MMO_INIT_A; nest <= MMO_MATMUL; nest++)
    mmo_run_nest(nest, dtype, n, 0, n, threads, a, b, c, bt);
  return mmo_trace(dtype, n, c);
}

/* ---- known answers that do not need the O(N^3) loop ---------------------------- */

/*
 * Exact value of c[i][j] = sum_k (i+k)(k-j)/N^2 = (S2 + (i-j) S1 - N i j) / N^2
 * (SURVEY appendix A).  For N a power of two every operand, product and partial
 * sum of the loop is a dyadic rational that fits a double exactly (up to
 * N = 2^17), so the loop result equals this for any summation order.  Computed
 * in 128-bit integers, then one exact division by a power of two; for other N
 * the division is correctly rounded to nearest (long double intermediate is
 * avoided: we return the nearest double of the exact rational via __int128).
 */
MMO_API double mmo_closed_form(int n, int i, int j) {
  const __int128 N = n;
  const __int128 S1 = N * (N - 1) / 2;
  const __int128 S2 = (N - 1) * N * (2 * N - 1) / 6;
  const __int128 num = S2 + (__int128)(i - j) * S1 - N * (__int128)i * (__int128)j;
  /* |num| < 2^53 for n <= 2^17, so the conversion is exact */
  return (double)(long long)num / ((double)n * (double)n);
}

/* Fill c (double) from the closed form; rows [r0, r1). */
MMO_API void mmo_closed_form_fill(int n, int r0, int r1, double* c) {
  for (int i = r0; i < r1; i++)
    for (int j = 0; j < n; j++) c[(size_t)i * n + j] = mmo_closed_form(n, i, j);
}

/* FNV-1a-64 over a byte range (used for the golden hashes of whole arrays). */
MMO_API uint64_t mmo_fnv1a64(const void* data, size_t bytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < bytes; i++) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

/* ---- timing leg for bench.py (cpu_baseline / --impl reference) ----------------- */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/*
 * Time the program on the host.  The five cheap nests run in full; the matmul
 * nest runs only rows [0, matmul_rows) so the call stays bounded (the caller
 * scales: every row of the nest costs the same 2N^2 flop).  seconds[0..5] get the
 * per-nest wall times (seconds[4] is for the sampled rows only).  Returns the
 * trace of the (partially computed) c, or NAN when allocation fails.
 */
MMO_API double mmo_time_app(int dtype, int n, int threads, int matmul_rows, double seconds[6]) {
  const size_t esz = dtype == 0 ? sizeof(double) : sizeof(float);
  const size_t bytes = (size_t)n * n * esz;
  void* a = malloc(bytes);
  void* b = malloc(bytes);
  void* c = malloc(bytes);
  void* bt = malloc(bytes);
  double tr = NAN;
  if (a && b && c && bt) {
    if (matmul_rows > n) matmul_rows = n;
    for (int nest = MMO_INIT_A; nest <= MMO_MATMUL; nest++) {
      const int r1 = nest == MMO_MATMUL ? matmul_rows : n;
      const double t0 = now_s();
      mmo_run_nest(nest, dtype, n, 0, r1, threads, a, b, c, bt);
      seconds[nest] = now_s() - t0;
    }
    const double t0 = now_s();
    tr = mmo_trace(dtype, n, c);
    seconds[MMO_TRACE] = now_s() - t0;
  }
  free(a);
  free(b);
  free(c);
  free(bt);
  return tr;
}
