// knng_partition.cu -- K8 balanced k-medoids (Alg. 4).  (filled in below)
#include "../../include/knng.h"
extern "C" int partition_kmedoids(knng_graph *, int32_t, double, int32_t, uint64_t, uint8_t *, int32_t *, int64_t *,
                                  const int32_t *) {
  return KNNG_ERR_INVALID_ARG;
}
