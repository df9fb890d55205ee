/*
 * oracle.c -- sequential CPU oracle for the task-stream hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
 * paper_1304_0878_b200/, include/, the CUDA library) may include, link or call
 * this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant with the CUDA path.
 *
 * What it computes (section 3, 293-296 and the
 * conclusion, lines 1082-1084): an annotated StarPU program compiled without
 * the plug-in "still leads a valid sequential program".  Running every task
 * call synchronously, one after the other in submission (program) order,
 * therefore DEFINES the result any schedule must reproduce.
 * states it as "byte-identical to executing all tasks in submission order on
 * a single CPU worker".
 *
 * Task bodies (each on the element range [off, off+len) of the (sub)handle
 * it names; n = the handle's NX):
 *   SCAL(f; x:RW)        for i<n: x[i] = x[i] * f
 *   AXPY(a; x:R, y:RW)   for i<n: y[i] = (a * x[i]) + y[i] BASELINE.json configs[2];
 *                        two roundings, no contraction (reading R14)
 *   COPY(x:R, y:W)       for i<n: y[i] = x[i]               BASELINE.json configs[2]
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (never -ffast-math/-Ofast,
 * which link crtfastmath.o and set FTZ/DAZ).  IEEE-754 binary32, round to
 * nearest even, subnormals preserved (readings R12, R14 in DESIGN.md).
 */
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#include "oracle.h"

#if defined(__FAST_MATH__)
#error "the oracle must not be built with -ffast-math"
#endif

/* SCAL: "for (unsigned i = 0; i < n; i++) val[i] *= *factor;" */
static void scal(float *x, int64_t n, float f) {
  for (int64_t i = 0; i < n; i++) x[i] = x[i] * f;
}

/* AXPY: y[i] = (a*x[i]) + y[i].  The product is rounded to binary32 before
 * the add (separate statements; -ffp-contract=off forbids FMA contraction). */
static void axpy(float a, const float *x, float *y, int64_t n) {
  for (int64_t i = 0; i < n; i++) {
    float p = a * x[i];
    y[i] = p + y[i];
  }
}

/* COPY: y[i] = x[i] in increasing index order (write-only destination). */
static void copy(const float *x, float *y, int64_t n) {
  for (int64_t i = 0; i < n; i++) y[i] = x[i];
}

int oracle_run(int64_t ntasks, const int32_t *codelet, const float *scalar,
               const int32_t *buf0, const int64_t *off0, const int64_t *len0,
               const int32_t *buf1, const int64_t *off1, const int64_t *len1,
               float *const *bufs) {
  /* Tasks one by one in submission order. */
  for (int64_t t = 0; t < ntasks; t++) {
    switch (codelet[t]) {
      case ORACLE_SCAL:
        scal(bufs[buf0[t]] + off0[t], len0[t], scalar[t]);
        break;
      case ORACLE_AXPY:
        if (len0[t] != len1[t]) return -1;
        axpy(scalar[t], bufs[buf0[t]] + off0[t], bufs[buf1[t]] + off1[t], len0[t]);
        break;
      case ORACLE_COPY:
        if (len0[t] != len1[t]) return -1;
        copy(bufs[buf0[t]] + off0[t], bufs[buf1[t]] + off1[t], len0[t]);
        break;
      default:
        return -1;
    }
  }
  return 0;
}

/* OpenMP variant, for the bench's CPU baseline on all host cores (SURVEY.md
 * 8(d) "Report an OpenMP variant beside it"): tasks still one by one in
 * submission order; inside a task the element range is split among
 * nthreads threads.  Every element of a task is computed by the same single
 * IEEE operation(s) as in oracle_run, and no element depends on another, so
 * the result is byte-identical (pinned in tests/test_oracle.py). */
int oracle_run_omp(int64_t ntasks, const int32_t *codelet, const float *scalar,
                   const int32_t *buf0, const int64_t *off0, const int64_t *len0,
                   const int32_t *buf1, const int64_t *off1, const int64_t *len1,
                   float *const *bufs, int nthreads) {
  for (int64_t t = 0; t < ntasks; t++) {
    if (codelet[t] != ORACLE_SCAL && len0[t] != len1[t]) return -1;
    if (codelet[t] < ORACLE_SCAL || codelet[t] > ORACLE_COPY) return -1;
  }
  for (int64_t t = 0; t < ntasks; t++) {
    float *x = bufs[buf0[t]] + off0[t];
    const int64_t n = len0[t];
    const float f = scalar[t];
    float *y = codelet[t] == ORACLE_SCAL ? x : bufs[buf1[t]] + off1[t];
    switch (codelet[t]) {
      case ORACLE_SCAL:
#pragma omp parallel for num_threads(nthreads) schedule(static) if (n >= 65536)
        for (int64_t i = 0; i < n; i++) x[i] = x[i] * f;
        break;
      case ORACLE_AXPY:
        /* aliasing (x == y, reading R6) stays element-wise: element i is
         * read and written by one thread; partially overlapping ranges run
         * in index order */
        if (x != y && ((x < y && x + n > y) || (y < x && y + n > x))) {
          for (int64_t i = 0; i < n; i++) {
            float p = f * x[i];
            y[i] = p + y[i];
          }
          break;
        }
#pragma omp parallel for num_threads(nthreads) schedule(static) if (n >= 65536)
        for (int64_t i = 0; i < n; i++) {
          float p = f * x[i];
          y[i] = p + y[i];
        }
        break;
      default:
        if (x == y) break;
        if ((x < y && x + n > y) || (y < x && y + n > x)) {   /* overlapping ranges: in order */
          for (int64_t i = 0; i < n; i++) y[i] = x[i];
          break;
        }
#pragma omp parallel for num_threads(nthreads) schedule(static) if (n >= 65536)
        for (int64_t i = 0; i < n; i++) y[i] = x[i];
        break;
    }
  }
  return 0;
}

/* Element-major evaluation of a stream of SCAL tasks that all cover the same
 * element range: element i goes through f_1, ..., f_k in submission order.
 * Equal to task-major order because each SCAL is element-wise (element i of
 * the output depends only on element i of the input and the factors in
 * order); pinned against oracle_run in tests/test_oracle.py.  Used to check
 * 4 GiB outputs in bounded CPU time. */
void oracle_scal_chain(float *x, int64_t n, const float *factors, int64_t k) {
  for (int64_t i = 0; i < n; i++) {
    float v = x[i];
    for (int64_t j = 0; j < k; j++) v = v * factors[j];
    x[i] = v;
  }
}

/* Build-time sanity: float multiply semantics as compiled into this object. */
int oracle_flt_eval_method(void) {
#ifdef __FLT_EVAL_METHOD__
  return __FLT_EVAL_METHOD__;
#else
  return -99;
#endif
}
