// Graph build (K1-K5): placeholder until the GPU builder lands.
#include "common.cuh"

using namespace ra;

extern "C" ra_status ra_graph_build(ra_ctx* ctx, ra_kv* keys, const float* train_q, uint64_t nq,
                                    uint32_t q_dim, int on_device, const ra_build_params* params,
                                    ra_build_stats* stats, ra_graph** out) {
  return guard([&] { runtime("graph build not implemented yet"); });
}
