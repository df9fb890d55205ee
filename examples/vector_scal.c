/*
 * The paper's running example (section 2) written against
 * the btask C ABI: register a vector, insert a vector_scal task with factor
 * 3.14, wait for all tasks, unregister -- then a partitioned chain of
 * scalings, the shape of BASELINE.json configs[1].
 *
 *   gcc -O2 -I include examples/vector_scal.c -L paper_1304_0878_b200 -lbtask \
 *       -Wl,-rpath,$PWD/paper_1304_0878_b200 -o vector_scal && ./vector_scal
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "btask.h"

#define NX 1024

#define CHECK(call)                                                              \
  do {                                                                           \
    int err_ = (call);                                                           \
    if (err_ != 0) {                                                             \
      fprintf(stderr, "%s: %s (%s)\n", #call, bt_strerror(err_), bt_last_error(rt)); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main(void) {
  bt_runtime *rt = NULL;
  bt_config cfg;
  bt_config_init(&cfg);
  int err = bt_init(&cfg, &rt);
  if (err) {
    fprintf(stderr, "bt_init: %s\n", bt_strerror(err));
    return 1;
  }

  /* starpu_vector_data_register (&vector_handle, 0, vector, NX, sizeof (vector[0])); */
  static float vector[NX];
  for (int i = 0; i < NX; i++) vector[i] = (float)(i + 1);
  bt_handle vector_handle;
  CHECK(bt_vector_data_register(rt, &vector_handle, 0, vector, NX, sizeof(vector[0])));

  /* float factor = 3.14;
   * starpu_insert_task (&scale_vector_codelet, STARPU_VALUE, &factor, sizeof factor,
   *                     STARPU_RW, vector_handle, 0); */
  float factor = 3.14f;
  int mode = BT_RW;
  CHECK(bt_insert_task(rt, BT_CL_SCAL, &factor, sizeof factor, &vector_handle, &mode, 1));

  /* starpu_task_wait_for_all (); starpu_data_unregister (vector_handle); */
  CHECK(bt_task_wait_for_all(rt));
  CHECK(bt_data_unregister(rt, vector_handle));
  printf("vector[0..3] = %.7g %.7g %.7g %.7g, vector[1023] = %.9g\n", vector[0], vector[1], vector[2], vector[3],
         vector[NX - 1]);

  /* an unregistered pointer: the generated task body's error */
  bt_handle h;
  if (bt_data_lookup(rt, vector, &h) == 0) return 1;
  printf("lookup after unregister: %s\n", bt_last_error(rt));

  /* a partitioned chain: 16 sweeps of vector_scal over 64 tiles */
  float *big = NULL;
  CHECK(bt_malloc((void **)&big, 64 * 1024 * sizeof(float)));
  for (int i = 0; i < 64 * 1024; i++) big[i] = 1.0f;
  bt_handle hb, tiles[64];
  CHECK(bt_vector_data_register(rt, &hb, 0, big, 64 * 1024, sizeof(float)));
  CHECK(bt_data_partition(rt, hb, 64));
  CHECK(bt_data_get_children(rt, hb, tiles, 64));
  for (int s = 0; s < 16; s++)
    for (int t = 0; t < 64; t++) CHECK(bt_insert_task(rt, BT_CL_SCAL, &factor, sizeof factor, &tiles[t], &mode, 1));
  CHECK(bt_task_wait_for_all(rt));
  bt_stats st;
  bt_stats_get(rt, &st);
  CHECK(bt_data_unpartition(rt, hb));
  CHECK(bt_data_unregister(rt, hb));
  printf("chain: big[0] = %.9g after 16 scalings; %llu tasks in %llu items (%llu fused)\n", big[0],
         (unsigned long long)st.tasks_submitted, (unsigned long long)st.items, (unsigned long long)st.fused_tasks);
  CHECK(bt_free(big));
  CHECK(bt_shutdown(rt));
  return 0;
}
