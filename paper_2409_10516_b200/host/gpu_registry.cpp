// See gpu_registry.hpp.
#include "gpu_registry.hpp"

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace attnindex::gpu {

void rethrow(ra_status st) {
  const std::string msg = ra_last_error();
  if (st == RA_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

ra_ctx* thread_ctx() {
  thread_local struct Holder {
    ra_ctx* c = nullptr;
    ~Holder() {
      if (c) ra_ctx_destroy(c);
    }
  } h;
  if (!h.c) check(ra_ctx_create(0, &h.c));
  return h.c;
}

namespace {
struct KvEntry {
  std::weak_ptr<const VectorSet> keys, values;
  const VectorSet* values_id = nullptr;
  ra_kv* kv = nullptr;  // the registry's reference
};
std::mutex g_mu;
std::map<const VectorSet*, KvEntry> g_kv;

// drop entries whose key set died (graphs / engines keep their own refs)
void purge_locked() {
  for (auto it = g_kv.begin(); it != g_kv.end();) {
    if (it->second.keys.expired()) {
      ra_kv_release(it->second.kv);
      it = g_kv.erase(it);
    } else {
      ++it;
    }
  }
}

ra_kv* lookup_locked(const std::shared_ptr<const VectorSet>& keys) {
  purge_locked();
  auto it = g_kv.find(keys.get());
  if (it != g_kv.end() && it->second.keys.lock() == keys) return it->second.kv;
  if (it != g_kv.end()) {  // a dead set at a reused address
    ra_kv_release(it->second.kv);
    g_kv.erase(it);
  }
  ra_kv* kv = nullptr;
  check(ra_kv_create(thread_ctx(), keys->n ? keys->data.data() : nullptr, nullptr, keys->n,
                     keys->d, 0, &kv));
  g_kv[keys.get()] = KvEntry{keys, {}, nullptr, kv};
  return kv;
}
}  // namespace

ra_kv* keys_kv(const std::shared_ptr<const VectorSet>& keys) {
  std::lock_guard<std::mutex> lk(g_mu);
  ra_kv* kv = lookup_locked(keys);
  ra_kv_retain(kv);
  return kv;
}

ra_kv* kv_with_values(const std::shared_ptr<const VectorSet>& keys,
                      const std::shared_ptr<const VectorSet>& values) {
  std::lock_guard<std::mutex> lk(g_mu);
  ra_kv* kv = lookup_locked(keys);
  KvEntry& e = g_kv[keys.get()];
  if (!ra_kv_has_values(kv)) {
    if (values->n != keys->n) throw std::invalid_argument("keys and values must have equal n");
    check(ra_kv_attach_values(thread_ctx(), kv, values->n ? values->data.data() : nullptr,
                              values->n, 0));
    e.values = values;
    e.values_id = values.get();
  } else if (e.values_id != values.get() || e.values.lock() != values) {
    return nullptr;
  }
  ra_kv_retain(kv);
  return kv;
}

}  // namespace attnindex::gpu
