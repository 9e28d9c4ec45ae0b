// nd_collective.cu — collective apps — placeholder until the engine lands.
#include "nd_internal.h"

extern "C" int nd_run_collective(const nd_graph*, int, int64_t, int64_t, int, int64_t, int64_t,
                                 int64_t, int64_t, int64_t, int64_t, const int64_t*,
                                 const int64_t*, uint64_t, int64_t, void*, nd_result**) {
  nd_set_last_error("nd_run_collective: not built yet", __FILE__, __LINE__);
  return ND_ERR_ARG;
}
