// C ABI: cluster lifecycle, step, parameters (see include/hpsim_b200.h).
#include <cstring>
#include <memory>
#include <string>

#include "cluster.hpp"
#include "comm.hpp"
#include "errors.hpp"
#include "hpsim_b200.h"

namespace hp {
extern thread_local std::string g_last_error;

template <class F>
int guarded_c(F&& f) {
  try {
    f();
    g_last_error.clear();
    return HP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HP_ERR_CUDA;
  }
}
}  // namespace hp

struct hp_cluster {
  std::unique_ptr<hp::ClusterBase> impl;
  int workers = 0;
};

using namespace hp;

namespace {
// Every entry point that takes a cluster rejects a null handle (UsageError).
const hp_cluster& need(const hp_cluster* c, const char* fn) {
  if (!c || !c->impl) usage_error(std::string(fn) + ": null cluster");
  return *c;
}
hp_cluster& need(hp_cluster* c, const char* fn) {
  if (!c || !c->impl) usage_error(std::string(fn) + ": null cluster");
  return *c;
}
}  // namespace

extern "C" {

HP_API int hp_cluster_create(const hp_model_spec* spec, const hp_cluster_config* cfg, hp_cluster** out) {
  return guarded_c([&] {
    if (!spec || !cfg || !out) usage_error("hp_cluster_create: null argument");
    auto c = std::make_unique<hp_cluster>();
    c->impl = make_cluster(spec, cfg);
    c->workers = cfg->workers;
    *out = c.release();
  });
}

HP_API void hp_cluster_destroy(hp_cluster* c) { delete c; }

HP_API int hp_nccl_unique_id(unsigned char out[128]) {
  return guarded_c([&] { nccl_unique_id(out); });
}

HP_API int hp_cluster_run_step(hp_cluster* c, const float* const* batches, const float* const* targets,
                               int mem_kind, const hp_hyper* hp_, double lr, hp_step_metrics* out) {
  return guarded_c([&] {
    need(c, "run_step");
    if (!hp_ || !out) usage_error("run_step: null argument");
    c->impl->run_step(batches, targets, mem_kind, *hp_, lr, out);
  });
}

HP_API int hp_cluster_prefetch(hp_cluster* c, const float* const* batches, const float* const* targets) {
  return guarded_c([&] {
    if (!c) usage_error("prefetch: null cluster");
    c->impl->prefetch(batches, targets);
  });
}

HP_API int hp_cluster_trace(const hp_cluster* c, hp_trace_event* out, int cap) {
  int n = -1;
  const int rc = guarded_c([&] {
    const auto& t = need(c, "hp_cluster_trace").impl->trace;
    if (cap > 0 && !out) usage_error("hp_cluster_trace: null output");
    for (int i = 0; i < static_cast<int>(t.size()) && i < cap; ++i) out[i] = t[i];
    n = static_cast<int>(t.size());
  });
  return rc == HP_OK ? n : -1;
}

HP_API int hp_cluster_worker_bytes(const hp_cluster* c, int worker, int64_t sent[4], int64_t received[4]) {
  return guarded_c([&] {
    need(c, "hp_cluster_worker_bytes");
    if (!sent || !received) usage_error("hp_cluster_worker_bytes: null output");
    if (worker < 0 || worker >= c->workers) usage_error("worker index out of range");
    for (int i = 0; i < 4; ++i) {
      sent[i] = c->impl->sent[worker][i];
      received[i] = c->impl->received[worker][i];
    }
  });
}

HP_API int64_t hp_cluster_param_size(const hp_cluster* c, int worker, int which, int layer) {
  int64_t n = -1;
  guarded_c([&] { n = need(c, "hp_cluster_param_size").impl->param_size(worker, which, layer); });
  return n;
}

HP_API int hp_cluster_read_param(hp_cluster* c, int worker, int which, int layer, float* dst, int64_t n) {
  return guarded_c([&] {
    need(c, "hp_cluster_read_param");
    if (!dst && n > 0) usage_error("hp_cluster_read_param: null destination");
    c->impl->read_param(worker, which, layer, dst, n);
  });
}

HP_API int64_t hp_cluster_debug_decisions(hp_cluster* c, int worker, int kind, int layer, void* dst, int64_t n) {
  int64_t r = -1;
  const int rc = guarded_c([&] {
    need(c, "hp_cluster_debug_decisions");
    r = c->impl->read_decisions(worker, kind, layer, dst, n);
  });
  return rc == 0 ? r : -1;
}

HP_API int hp_cluster_write_param(hp_cluster* c, int worker, int which, int layer, const float* src,
                                  int64_t n) {
  return guarded_c([&] {
    need(c, "hp_cluster_write_param");
    if (!src && n > 0) usage_error("hp_cluster_write_param: null source");
    c->impl->write_param(worker, which, layer, src, n);
  });
}

HP_API int hp_cluster_gather_model(hp_cluster* c, float* const* conv_k, float* const* conv_b,
                                   float* const* fc_w, float* const* fc_b) {
  return guarded_c([&] {
    need(c, "hp_cluster_gather_model");
    if (!conv_k || !conv_b || !fc_w || !fc_b) usage_error("hp_cluster_gather_model: null output array");
    c->impl->gather_model(conv_k, conv_b, fc_w, fc_b);
  });
}

HP_API int hp_cluster_set_skip_sync_broadcast(hp_cluster* c, int v) {
  return guarded_c([&] { need(c, "hp_cluster_set_skip_sync_broadcast").impl->skip_sync_broadcast = v != 0; });
}

HP_API double hp_cluster_last_step_ms(const hp_cluster* c) { return c && c->impl ? c->impl->last_ms : -1.0; }
HP_API int64_t hp_cluster_last_step_launches(const hp_cluster* c) {
  return c && c->impl ? c->impl->last_launches : -1;
}

HP_API int hp_step_accounting(const hp_model_spec* spec, const hp_cluster_config* cfg, int steps,
                              int64_t bytes_sent[4], hp_trace_event* trace, int cap, int* n_events,
                              int64_t* worker_sent, int64_t* worker_received) {
  return guarded_c([&] {
    if (!spec || !cfg) usage_error("hp_step_accounting: null argument");
    if (cfg->workers < 1) config_error("cluster.workers: must be >= 1");
    if (cfg->per_worker_batch < 1) config_error("cluster.per_worker_batch: must be >= 1");
    if (cfg->scheme == HP_SCHEME_C && cfg->per_worker_batch % cfg->workers != 0)
      config_error("cluster.per_worker_batch: scheme C scatters b/K examples per worker per turn; " +
                   std::to_string(cfg->per_worker_batch) + " is not divisible by " +
                   std::to_string(cfg->workers));
    Geometry g = make_geometry(spec, cfg->workers, cfg->per_worker_batch);
    std::vector<std::array<int64_t, 4>> sent(cfg->workers, {0, 0, 0, 0}), recv(cfg->workers, {0, 0, 0, 0});
    std::vector<hp_trace_event> tr;
    for (int i = 0; i < 4; ++i) bytes_sent[i] = 0;
    for (int s = 0; s < steps; ++s)
      step_accounting(g, cfg->workers, cfg->per_worker_batch, cfg->scheme, sent, recv, tr, bytes_sent);
    *n_events = static_cast<int>(tr.size());
    for (int i = 0; i < static_cast<int>(tr.size()) && i < cap; ++i) trace[i] = tr[i];
    for (int w = 0; w < cfg->workers; ++w)
      for (int i = 0; i < 4; ++i) {
        worker_sent[w * 4 + i] = sent[w][i];
        worker_received[w * 4 + i] = recv[w][i];
      }
  });
}

HP_API void* hp_cluster_stream(const hp_cluster* c) { return c && c->impl ? c->impl->stream() : nullptr; }

HP_API void hp_cluster_last_step_io(const hp_cluster* c, int64_t* h2d, int64_t* d2h) {
  const bool ok = c && c->impl;
  if (h2d) *h2d = ok ? c->impl->io_h2d : -1;
  if (d2h) *d2h = ok ? c->impl->io_d2h : -1;
}

HP_API double hp_cluster_last_gemm_flops(const hp_cluster* c) {
  return c && c->impl ? c->impl->last_gemm_flops : -1.0;
}

HP_API int hp_cluster_set_graphs(hp_cluster* c, int on) {
  return guarded_c([&] { need(c, "hp_cluster_set_graphs").impl->use_graphs = on != 0; });
}

HP_API int hp_cluster_set_debug_capture(hp_cluster* c, int on) {
  return guarded_c([&] { need(c, "hp_cluster_set_debug_capture").impl->capture_fc = on != 0; });
}

HP_API int hp_cluster_set_fuse_fc_sgd(hp_cluster* c, int on) {
  return guarded_c([&] { need(c, "hp_cluster_set_fuse_fc_sgd").impl->fuse_fc_sgd = on != 0; });
}

HP_API int hp_cluster_set_shift_conv(hp_cluster* c, int on) {
  return guarded_c([&] {
    need(c, "hp_cluster_set_shift_conv").impl->use_shift = on != 0;
    c->impl->rebuild_plans();
  });
}

HP_API int hp_cluster_set_profile(hp_cluster* c, int on) {
  return guarded_c([&] { need(c, "hp_cluster_set_profile").impl->profile = on != 0; });
}

HP_API int hp_cluster_debug_marker_graph(hp_cluster* c, const float* const* batches, const float* const* targets,
                                         int mem_kind, const hp_hyper* hp_, double lr, int32_t* tags,
                                         uint8_t* reach, int cap, int* n_markers) {
  return guarded_c([&] {
    need(c, "hp_cluster_debug_marker_graph");
    if (!hp_ || !n_markers) usage_error("hp_cluster_debug_marker_graph: null argument");
    std::vector<int> t;
    std::vector<uint8_t> r;
    c->impl->marker_graph(batches, targets, mem_kind, *hp_, lr, t, r);
    *n_markers = static_cast<int>(t.size());
    if (static_cast<int>(t.size()) > cap) usage_error("hp_cluster_debug_marker_graph: cap too small");
    for (size_t i = 0; i < t.size(); ++i) tags[i] = t[i];
    std::memcpy(reach, r.data(), r.size());
  });
}

HP_API int hp_cluster_gemm_profile(const hp_cluster* c, hp_gemm_prof* out, int cap) {
  if (!c || !c->impl) return -1;
  const auto& p = c->impl->prof;
  for (int i = 0; i < static_cast<int>(p.size()) && i < cap; ++i) {
    std::memset(out[i].tag, 0, sizeof out[i].tag);
    std::strncpy(out[i].tag, p[i].tag, sizeof out[i].tag - 1);
    out[i].layer = p[i].layer;
    out[i].flops = p[i].flops;
    out[i].ms = p[i].ms;
  }
  return static_cast<int>(p.size());
}

}  // extern "C"
