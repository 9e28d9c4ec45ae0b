// nd_individual.cu — multi-slot individual apps (k-hop) — placeholder until
// the engine lands.
#include "nd_internal.h"

extern "C" int nd_run_individual(const nd_graph*, int, const double*, int64_t, const int64_t*,
                                 int64_t, int64_t, int64_t, const int64_t*, int64_t, uint64_t,
                                 int64_t, int, void*, nd_result**) {
  nd_set_last_error("nd_run_individual: not built yet", __FILE__, __LINE__);
  return ND_ERR_ARG;
}
