/*
 * oracle/ref_fixture_harness.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Compiles the reference workload itself -- /root/reference/proj/fixtures/matmul.c,
 * unmodified and included from where it lies (oracle/Makefile passes
 * -I/root/reference/proj) -- into oracle/_ref/libmatmul_fixture.so and exposes the
 * arrays the program leaves behind, so the restatement in matmul_oracle.c can be
 * pinned bit for bit against the real reference at its shipped size (N = 256,
 * matmul.c:3).  The fixture's `main` is renamed by macro; its static arrays
 * (matmul.c:5) are visible here because this is the same translation unit.
 */
#define main acctune_fixture_main
#include "fixtures/matmul.c"
#undef main

#define FX_API __attribute__((visibility("default")))

FX_API int fixture_n(void) { return N; }
/* runs matmul.c:7-35 (prints "checksum ..." on stdout, like the program) */
FX_API int fixture_run(void) { return acctune_fixture_main(); }
FX_API const double* fixture_a(void) { return &a[0][0]; }
FX_API const double* fixture_b(void) { return &b[0][0]; }
FX_API const double* fixture_c(void) { return &c[0][0]; }
FX_API const double* fixture_bt(void) { return &bt[0][0]; }
