// C-ABI entry points (include/autoplan_b200.h): argument checks, handle
// lifetime and the thread-local error string.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <new>
#include <string>

#include "engine.h"

namespace apb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int current_sm_count(int* sms) {
  static std::atomic<int> cache[64];
  int dev = 0;
  AP_CUDA_CHECK(cudaGetDevice(&dev));
  const bool cached = dev >= 0 && dev < 64;
  int v = cached ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (v <= 0) {
    AP_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    if (cached) cache[dev].store(v, std::memory_order_relaxed);
  }
  *sms = v;
  return AP_OK;
}

int cuda_fail(cudaError_t err, const char* what) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "CUDA error %s (%d) in %s", cudaGetErrorString(err), (int)err, what);
  g_last_error = buf;
  return AP_ERR_CUDA;
}

static void release_graph(GraphTables* t) {
  t->d_slot_class.release();
  t->d_forced_words.release();
  if (t->d_scratch) cudaFree(t->d_scratch);
  t->d_scratch = nullptr;
  t->scratch_words = 0;
  t->d_imp_offset.release();
  t->d_imp_target.release();
  t->d_program.release();
  t->d_forced_list.release();
  t->d_slot_base.release();
  t->d_slot_owner.release();
  t->d_slot_desc.release();
  t->d_slot_desc_t.release();
  t->d_slot_cls8.release();
  t->d_imp_bits.release();
  t->d_forced_bits.release();
}

static void release_decision(DecisionTables* t) {
  t->d_dec_class.release();
  t->d_dec_flags.release();
  t->d_first_same.release();
  t->d_slots.release();
  t->d_dec_desc.release();
  t->d_dec_masks.release();
  t->d_dec_cls8.release();
  t->d_class_ncand.release();
  t->d_ncand_planes.release();
}

}  // namespace apb

extern "C" {

const char* ap_last_error(void) { return apb::g_last_error.c_str(); }

const char* ap_version(void) { return "autoplan_b200 0.1.0 sm_100a"; }

int ap_graph_create(const ap_graph_desc* desc, ap_graph_t* out) {
  if (!out) {
    apb::set_error("ap_graph_create: null output handle");
    return AP_ERR_INVALID;
  }
  *out = nullptr;
  ap_graph* g = new (std::nothrow) ap_graph();
  if (!g) {
    apb::set_error("ap_graph_create: out of host memory");
    return AP_ERR_INVALID;
  }
  const int rc = apb::build_graph(desc, &g->t);
  if (rc != AP_OK) {
    apb::release_graph(&g->t);
    delete g;
    return rc;
  }
  *out = g;
  return AP_OK;
}

int ap_graph_destroy(ap_graph_t g) {
  if (!g) return AP_OK;
  apb::release_graph(&g->t);
  delete g;
  return AP_OK;
}

int ap_graph_get_info(ap_graph_t g, ap_graph_info* info) {
  if (!g || !info) {
    apb::set_error("ap_graph_get_info: null argument");
    return AP_ERR_INVALID;
  }
  info->num_slots = g->t.num_slots;
  info->num_classes = g->t.num_classes;
  info->num_links = g->t.num_links;
  info->num_implications = (int64_t)g->t.imp_target.size();
  int32_t forced = 0;
  for (uint8_t f : g->t.slot_forced) forced += f;
  info->num_forced = forced;
  return AP_OK;
}

int ap_graph_export(ap_graph_t g, int32_t* class_of_slot, uint8_t* class_forced, int32_t* imp_offset,
                    int32_t* imp_target) {
  if (!g) {
    apb::set_error("ap_graph_export: null handle");
    return AP_ERR_INVALID;
  }
  const apb::GraphTables& t = g->t;
  if (class_of_slot)
    for (int64_t s = 0; s < t.num_slots; ++s) class_of_slot[s] = t.class_of_slot[s];
  if (class_forced)
    for (int32_t c = 0; c < t.num_classes; ++c) class_forced[c] = t.class_forced[c];
  if (imp_offset)
    for (int32_t c = 0; c <= t.num_classes; ++c) imp_offset[c] = t.imp_offset[c];
  if (imp_target)
    for (size_t k = 0; k < t.imp_target.size(); ++k) imp_target[k] = t.imp_target[k];
  return AP_OK;
}

int ap_decision_create(ap_graph_t g, const int64_t* slots, const uint8_t* is_candidate, int32_t n,
                       ap_decision_t* out) {
  if (!g || !out) {
    apb::set_error("ap_decision_create: null argument");
    return AP_ERR_INVALID;
  }
  *out = nullptr;
  ap_decision* d = new (std::nothrow) ap_decision();
  if (!d) {
    apb::set_error("ap_decision_create: out of host memory");
    return AP_ERR_INVALID;
  }
  const int rc = apb::build_decision(&g->t, slots, is_candidate, n, &d->t);
  if (rc != AP_OK) {
    apb::release_decision(&d->t);
    delete d;
    return rc;
  }
  *out = d;
  return AP_OK;
}

int ap_decision_destroy(ap_decision_t d) {
  if (!d) return AP_OK;
  apb::release_decision(&d->t);
  delete d;
  return AP_OK;
}

int ap_propagate_batch(ap_graph_t g, ap_decision_t d, const int8_t* seeds_dev, int64_t batch, int64_t seed_stride,
                       int8_t* slots_dev, int64_t slots_stride, int8_t* cand_dev, int64_t cand_stride,
                       uint8_t* outcome_dev, int32_t* counts_dev, void* stream) {
  if (!g || !d) {
    apb::set_error("ap_propagate_batch: null handle");
    return AP_ERR_INVALID;
  }
  int rc = apb::ensure_graph_on_device(&g->t);
  if (rc == AP_OK) rc = apb::ensure_decision_on_device(&d->t);
  if (rc != AP_OK) return rc;
  // descriptor-driven fast kernel when the graph / strides allow it, else the
  // generic kernel (AP_PROPAGATE_GENERIC=1 forces the generic one, for tests)
  const char* force = std::getenv("AP_PROPAGATE_GENERIC");
  if (!(force && force[0] == '1') && batch > 0) {
    rc = apb::launch_propagate_fast(&g->t, &d->t, seeds_dev, batch, seed_stride, slots_dev, slots_stride, cand_dev,
                                    cand_stride, outcome_dev, counts_dev, static_cast<cudaStream_t>(stream));
    if (rc != AP_ERR_UNSUPPORTED) return rc;
  }
  return apb::launch_propagate(&g->t, &d->t, seeds_dev, batch, seed_stride, slots_dev, slots_stride, cand_dev,
                               cand_stride, outcome_dev, counts_dev, static_cast<cudaStream_t>(stream));
}

int ap_propagate_batch_packed(ap_graph_t g, ap_decision_t d, const int8_t* seeds_dev, int64_t batch,
                              int64_t seed_stride, uint8_t* packed_dev, int64_t packed_stride, int8_t* cand_dev,
                              int64_t cand_stride, uint8_t* outcome_dev, int32_t* counts_dev, void* stream) {
  if (!g || !d) {
    apb::set_error("ap_propagate_batch_packed: null handle");
    return AP_ERR_INVALID;
  }
  const int64_t S = g->t.num_slots, need = 4 * ((S + 15) / 16);
  if (batch < 0 || packed_stride < need || packed_stride % 4 || (batch > 0 && (!packed_dev || !seeds_dev)) ||
      (reinterpret_cast<uintptr_t>(packed_dev) & 3)) {
    apb::set_error("ap_propagate_batch_packed: bad arguments (packed rows 4-byte aligned, stride >= 4*ceil(S/16))");
    return AP_ERR_INVALID;
  }
  int rc = apb::ensure_graph_on_device(&g->t);
  if (rc == AP_OK) rc = apb::ensure_decision_on_device(&d->t);
  if (rc != AP_OK || batch == 0) return rc;
  auto st = static_cast<cudaStream_t>(stream);
  const char* force = std::getenv("AP_PROPAGATE_GENERIC");
  if (!(force && force[0] == '1')) {
    rc = apb::launch_propagate_fast(&g->t, &d->t, seeds_dev, batch, seed_stride, nullptr, 0, cand_dev, cand_stride,
                                    outcome_dev, counts_dev, st, packed_dev, packed_stride);
    if (rc != AP_ERR_UNSUPPORTED) return rc;
  }
  // generic kernel into int8 rows (stream-ordered scratch, chunks of <= 64 Mi bytes), then pack
  const int64_t stride = std::max<int64_t>(16, (S + 15) / 16 * 16);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, (64ll << 20) / stride));
  int8_t* scratch = nullptr;
  AP_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&scratch), chunk * stride, st));
  for (int64_t lo = 0; lo < batch && rc == AP_OK; lo += chunk) {
    const int64_t n = std::min(chunk, batch - lo);
    rc = apb::launch_propagate(&g->t, &d->t, seeds_dev + lo * seed_stride, n, seed_stride, scratch, stride,
                               cand_dev ? cand_dev + lo * cand_stride : nullptr, cand_stride, outcome_dev + lo,
                               counts_dev ? counts_dev + 4 * lo : nullptr, st);
    if (rc == AP_OK) rc = ap_pack_slots2(scratch, n, stride, S, packed_dev + lo * packed_stride, packed_stride, stream);
  }
  cudaFreeAsync(scratch, st);
  return rc;
}

int ap_propagate_trace(ap_graph_t g, ap_decision_t d, const int8_t* seeds_host, const int8_t* init_state_host,
                       int8_t* slots_host, int32_t* outcome_host, int32_t* conflict_site_out, void* stream) {
  if (!g || !d || !slots_host || !outcome_host || !conflict_site_out || (d->t.n && !seeds_host)) {
    apb::set_error("ap_propagate_trace: null argument");
    return AP_ERR_INVALID;
  }
  int rc = apb::ensure_graph_on_device(&g->t);
  if (rc == AP_OK) rc = apb::ensure_decision_on_device(&d->t);
  if (rc != AP_OK) return rc;
  return apb::run_trace(&g->t, &d->t, seeds_host, init_state_host, slots_host, outcome_host, conflict_site_out,
                        static_cast<cudaStream_t>(stream));
}

}  // extern "C"
