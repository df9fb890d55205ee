/* oracle.h -- sequential CPU oracle (TEST INFRASTRUCTURE ONLY; see oracle.c).
 * Not included by, and sharing nothing with, the CUDA product path. */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

/* Codelet ids of the oracle's own program model (oracle/oracle.py). */
#define ORACLE_SCAL 1
#define ORACLE_AXPY 2
#define ORACLE_COPY 3

/* Execute ntasks tasks in submission order.  Operand 0 / 1 of task t is the
 * element range [off, off+len) of host buffer bufs[buf].  SCAL uses operand 0
 * only (x:RW); AXPY and COPY read operand 0 (x:R) and write operand 1.
 * Returns 0, or -1 on an unknown codelet or operand length mismatch. */
int oracle_run(int64_t ntasks, const int32_t *codelet, const float *scalar,
               const int32_t *buf0, const int64_t *off0, const int64_t *len0,
               const int32_t *buf1, const int64_t *off1, const int64_t *len1,
               float *const *bufs);

/* The same, element-parallel inside each task on nthreads OpenMP threads
 * (tasks in submission order; byte-identical result).  Timing only. */
int oracle_run_omp(int64_t ntasks, const int32_t *codelet, const float *scalar,
                   const int32_t *buf0, const int64_t *off0, const int64_t *len0,
                   const int32_t *buf1, const int64_t *off1, const int64_t *len1,
                   float *const *bufs, int nthreads);

/* Element-major chain of k SCALs over x[0..n) (same result as task-major). */
void oracle_scal_chain(float *x, int64_t n, const float *factors, int64_t k);

int oracle_flt_eval_method(void);
#endif
