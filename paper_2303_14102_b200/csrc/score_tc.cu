// score_tc.cu -- K3: tcgen05 scoring (placeholder until the tensor-core kernel lands).
#include "score_common.cuh"

namespace fsil {

bool tc_supported(const fsil_context*) { return false; }
int64_t tc_tiles(const fsil_context* c, int* tile_rows) {
  *tile_rows = 128;
  return (c->n + 127) / 128;
}
void score_tc(fsil_context*, const ScoreParams&) {
  fail(FSIL_ERR_INVALID_ARGUMENT, "tcgen05 scoring path not built");
}

}  // namespace fsil
