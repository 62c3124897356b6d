/* gen_internal.h — host-side generator context shared by the C host part and
 * the CUDA twin of the generator (both in gen/). Input infrastructure only. */
#ifndef ASSE_GEN_INTERNAL_H
#define ASSE_GEN_INTERNAL_H
#include <stddef.h>
#include "asse_gen.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gen_ctx {
  gen_desc host;        /* descriptor with host table pointers */
  gen_desc dev;         /* descriptor with device table pointers (after upload) */
  int uploaded;
  int preset;
  uint64_t* cdf;
  uint32_t* n_a;
  uint64_t* plant_off;
  uint32_t* victim_on;
  size_t cdf_n, n_a_n, plant_n, victim_n;
  /* device copies */
  void* d_cdf;
  void* d_n_a;
  void* d_plant_off;
  void* d_victim_on;
} gen_ctx;

#ifdef __cplusplus
}
#endif
#endif
