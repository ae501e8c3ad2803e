// Shared device state of the drop-in TUs (attnindex_*_gpu.cpp): the
// per-thread ra_ctx, the reference's exception mapping, and the HBM copy of
// each key set keyed by VectorSet identity, so every graph and engine over
// the same shared_ptr<const VectorSet> (the GQA heads of one KV group,
// types.hpp:54-61) uses ONE upload.
#pragma once

#include <memory>

#include "attnindex/types.hpp"
#include "ra_capi.h"

namespace attnindex {
class OODGraph;

namespace gpu {

// ra_status -> std::invalid_argument (RA_ERR_INVALID_ARGUMENT) or
// std::runtime_error, with ra_last_error()'s text (the reference's messages)
[[noreturn]] void rethrow(ra_status st);
inline void check(ra_status st) {
  if (st != RA_OK) rethrow(st);
}

// one context (stream + scratch) per calling thread, device 0
ra_ctx* thread_ctx();

// The group's device copy of `keys` (a retained reference the caller
// releases). Entries whose VectorSet has expired are freed on every call.
ra_kv* keys_kv(const std::shared_ptr<const VectorSet>& keys);

// keys_kv with `values` attached (uploaded on first use). Returns nullptr
// when that key set already carries a different value set.
ra_kv* kv_with_values(const std::shared_ptr<const VectorSet>& keys,
                      const std::shared_ptr<const VectorSet>& values);

// The device graph of an OODGraph built or loaded through the drop-in
// (attnindex_oodgraph_gpu.cpp), uploaded on first use for any other live
// OODGraph; not retained (valid while the object lives).
ra_graph* device_graph(const OODGraph& g);

}  // namespace gpu
}  // namespace attnindex
