// ref_shim.cpp — C ABI around the UNMODIFIED reference (hpsim) so tests and
// the CPU baseline can drive it from Python. TEST INFRASTRUCTURE ONLY.
//
// Compiled together with /root/reference/proj/core/src/*.cpp (read in place,
// never copied) by oracle/Makefile into oracle/_ref/libhpsim_ref.so.
// Also supplies the two symbols the reference declares but never defines
// (include/hpsim/reference.hpp:29-51): SingleTrainer and
// max_relative_divergence.
#include <cmath>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "hpsim/cluster.hpp"
#include "hpsim/model.hpp"
#include "hpsim/optimizer.hpp"
#include "hpsim/reference.hpp"
#include "hpsim/rng.hpp"
#include "hpsim/tensor.hpp"
#include "hpsim_oracle.h"

namespace hpsim {

// reference.hpp:29-46 — plain single-worker synchronous SGD on a whole model.
SingleTrainer::SingleTrainer(const ModelSpec& spec, std::uint64_t seed, Precision precision)
    : SingleTrainer(init_model(spec, seed, precision)) {}

SingleTrainer::SingleTrainer(Model model) : model_(std::move(model)) {
  for (const auto& p : model_.conv) {
    conv_momentum_.push_back({Tensor(p.kernels.shape(), p.kernels.precision()),
                              Tensor(p.bias.shape(), p.bias.precision())});
  }
  for (const auto& p : model_.fc) {
    fc_momentum_.push_back({Tensor(p.weight.shape(), p.weight.precision()),
                            Tensor(p.bias.shape(), p.bias.precision())});
  }
}

double SingleTrainer::step(const Tensor& batch, const Tensor& targets, const HyperParams& hp,
                           double lr) {
  ActivationCache cache = forward(model_, batch);
  Gradients g = backward(model_, cache, targets);
  for (std::size_t l = 0; l < model_.fc.size(); ++l) {
    momentum_update(model_.fc[l].weight, fc_momentum_[l].weight, g.fc[l].weight, lr, hp.momentum,
                    hp.weight_decay);
    momentum_update(model_.fc[l].bias, fc_momentum_[l].bias, g.fc[l].bias, lr, hp.momentum,
                    hp.weight_decay);
  }
  for (std::size_t l = 0; l < model_.conv.size(); ++l) {
    momentum_update(model_.conv[l].kernels, conv_momentum_[l].kernels, g.conv[l].kernels, lr,
                    hp.momentum, hp.weight_decay);
    momentum_update(model_.conv[l].bias, conv_momentum_[l].bias, g.conv[l].bias, lr, hp.momentum,
                    hp.weight_decay);
  }
  return g.loss;
}

// reference.hpp:48-51
double max_relative_divergence(const Model& a, const Model& b) {
  double worst = 0.0;
  auto one = [&](const Tensor& x, const Tensor& y) {
    double diff = 0.0, ref = 0.0;
    for (std::int64_t i = 0; i < x.size(); ++i) {
      diff = std::max(diff, std::abs(x.value_at(i) - y.value_at(i)));
      ref = std::max(ref, std::abs(y.value_at(i)));
    }
    worst = std::max(worst, diff / (ref + 1e-30));
  };
  for (std::size_t l = 0; l < a.conv.size(); ++l) {
    one(a.conv[l].kernels, b.conv[l].kernels);
    one(a.conv[l].bias, b.conv[l].bias);
  }
  for (std::size_t l = 0; l < a.fc.size(); ++l) {
    one(a.fc[l].weight, b.fc[l].weight);
    one(a.fc[l].bias, b.fc[l].bias);
  }
  return worst;
}

}  // namespace hpsim

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const hpsim::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const hpsim::DimensionError& e) {
    g_err = e.what();
    return 2;
  } catch (const hpsim::DomainError& e) {
    g_err = e.what();
    return 3;
  } catch (const hpsim::UsageError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

hpsim::ModelSpec to_spec(const or_model_spec* s) {
  hpsim::ModelSpec m;
  for (int i = 0; i < s->n_conv; ++i) {
    const or_conv_layer& l = s->conv[i];
    if (l.floor_mode || l.lrn_size || l.pool_kernel) {
      throw hpsim::ConfigError("model.conv_layers[" + std::to_string(i) +
                               "]: floor mode / LRN / pooling are not expressible in the reference");
    }
    m.conv_layers.push_back({l.in_channels, l.out_channels, l.kernel, l.stride, l.pad, l.relu != 0});
  }
  for (int i = 0; i < s->n_fc; ++i) {
    m.fc_layers.push_back({s->fc[i].in_dim, s->fc[i].out_dim, s->fc[i].relu != 0});
  }
  m.input_shape = {s->input_shape[0], s->input_shape[1], s->input_shape[2]};
  m.num_classes = s->num_classes;
  return m;
}

hpsim::Precision prec(int p) { return p == 0 ? hpsim::Precision::kSingle : hpsim::Precision::kDouble; }

hpsim::HyperParams to_hyper(const or_hyper* h) {
  hpsim::HyperParams hp;
  hp.momentum = h->momentum;
  hp.lr = h->lr;
  hp.weight_decay = h->weight_decay;
  if (h->has_fc_partial_lr) hp.fc_partial_lr = h->fc_partial_lr;
  return hp;
}

struct RefCluster {
  std::unique_ptr<hpsim::Cluster> cluster;
  hpsim::StepTrace trace;
};

hpsim::Tensor from_doubles(std::vector<std::int64_t> shape, const double* v, hpsim::Precision p) {
  std::int64_t n = 1;
  for (auto d : shape) n *= d;
  return hpsim::Tensor::from_values(std::move(shape), std::span<const double>(v, n), p);
}

void to_doubles(const hpsim::Tensor& t, double* out) {
  for (std::int64_t i = 0; i < t.size(); ++i) out[i] = t.value_at(i);
}

const hpsim::Tensor* param_of(const hpsim::WorkerState& w, int which, int layer) {
  const bool mom = which >= 4;
  which &= 3;
  if (which <= 1) {
    const auto& v = mom ? w.conv_momentum : w.conv_params;
    if (layer < 0 || layer >= static_cast<int>(v.size())) return nullptr;
    return which == 0 ? &v[layer].kernels : &v[layer].bias;
  }
  const auto& v = mom ? w.fc_momentum : w.fc_shard;
  if (layer < 0 || layer >= static_cast<int>(v.size())) return nullptr;
  return which == 2 ? &v[layer].weight : &v[layer].bias;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_cluster_create(const or_model_spec* spec, const or_cluster_config* cfg, int* status) {
  RefCluster* rc = nullptr;
  *status = guarded([&] {
    hpsim::ClusterConfig c;
    c.workers = cfg->workers;
    c.per_worker_batch = cfg->per_worker_batch;
    c.scheme = cfg->scheme == 0 ? hpsim::Scheme::A : cfg->scheme == 1 ? hpsim::Scheme::B : hpsim::Scheme::C;
    c.variable_batch = cfg->variable_batch != 0;
    c.precision = prec(cfg->precision);
    c.seed = cfg->seed;
    auto cl = std::make_unique<hpsim::Cluster>(to_spec(spec), c);
    rc = new RefCluster{std::move(cl), {}};
  });
  return rc;
}

void ref_cluster_destroy(void* h) { delete static_cast<RefCluster*>(h); }

void ref_cluster_set_skip_sync_broadcast(void* h, int v) {
  static_cast<RefCluster*>(h)->cluster->set_skip_sync_broadcast(v != 0);
}

int ref_cluster_run_step(void* h, const double* const* batches, const double* const* targets,
                         const or_hyper* hyper, double lr, or_step_metrics* out) {
  auto* rc = static_cast<RefCluster*>(h);
  return guarded([&] {
    const auto& spec = rc->cluster->spec();
    const auto& cfg = rc->cluster->config();
    const auto p = cfg.precision;
    std::vector<hpsim::Tensor> xs, ts;
    for (int i = 0; i < cfg.workers; ++i) {
      xs.push_back(from_doubles({cfg.per_worker_batch, spec.input_shape[0], spec.input_shape[1],
                                 spec.input_shape[2]},
                                batches[i], p));
      ts.push_back(from_doubles({cfg.per_worker_batch, spec.num_classes}, targets[i], p));
    }
    auto res = rc->cluster->run_step(xs, ts, to_hyper(hyper), lr);
    rc->trace = res.trace;
    out->loss = res.metrics.loss;
    out->fc_update_count = res.metrics.fc_update_count;
    out->conv_update_count = res.metrics.conv_update_count;
    for (int i = 0; i < 4; ++i) out->bytes_sent[i] = res.metrics.bytes_sent[i];
    out->n_events = static_cast<int>(res.trace.events.size());
  });
}

int ref_cluster_trace(void* h, or_trace_event* out, int cap) {
  const auto& ev = static_cast<RefCluster*>(h)->trace.events;
  for (int i = 0; i < static_cast<int>(ev.size()) && i < cap; ++i) {
    out[i].phase = static_cast<int>(ev[i].phase);
    out[i].sub_batch = ev[i].sub_batch;
    out[i].worker = ev[i].worker;
    out[i].bytes_total = ev[i].bytes_total;
    out[i].bytes_max_sender = ev[i].bytes_max_sender;
  }
  return static_cast<int>(ev.size());
}

int ref_cluster_worker_bytes(void* h, int worker, int64_t sent[4], int64_t received[4]) {
  return guarded([&] {
    const auto& w = static_cast<RefCluster*>(h)->cluster->worker(worker);
    for (int i = 0; i < 4; ++i) {
      sent[i] = w.bytes.sent[i];
      received[i] = w.bytes.received[i];
    }
  });
}

int64_t ref_cluster_param_size(void* h, int worker, int which, int layer) {
  const auto* t = param_of(static_cast<RefCluster*>(h)->cluster->worker(worker), which, layer);
  return t ? t->size() : -1;
}

int ref_cluster_read_param(void* h, int worker, int which, int layer, double* dst, int64_t n) {
  return guarded([&] {
    const auto* t = param_of(static_cast<RefCluster*>(h)->cluster->worker(worker), which, layer);
    if (!t) throw hpsim::UsageError("read_param: bad worker/which/layer");
    if (t->size() != n) throw hpsim::DimensionError("read_param: size mismatch");
    to_doubles(*t, dst);
  });
}

// Overwrites a parameter through the only mutable path the reference offers
// (a const_cast of the WorkerState it exposes read-only). Test use only.
int ref_cluster_write_param(void* h, int worker, int which, int layer, const double* src, int64_t n) {
  return guarded([&] {
    auto* t = const_cast<hpsim::Tensor*>(
        param_of(static_cast<RefCluster*>(h)->cluster->worker(worker), which, layer));
    if (!t) throw hpsim::UsageError("write_param: bad worker/which/layer");
    if (t->size() != n) throw hpsim::DimensionError("write_param: size mismatch");
    for (int64_t i = 0; i < n; ++i) t->set_value(i, src[i]);
  });
}

// gathered_model (cluster.cpp:417-437); pointers per layer, reference layouts.
int ref_cluster_gathered(void* h, double* const* conv_k, double* const* conv_b, double* const* fc_w,
                         double* const* fc_b) {
  return guarded([&] {
    hpsim::Model m = static_cast<RefCluster*>(h)->cluster->gathered_model();
    for (std::size_t l = 0; l < m.conv.size(); ++l) {
      to_doubles(m.conv[l].kernels, conv_k[l]);
      to_doubles(m.conv[l].bias, conv_b[l]);
    }
    for (std::size_t l = 0; l < m.fc.size(); ++l) {
      to_doubles(m.fc[l].weight, fc_w[l]);
      to_doubles(m.fc[l].bias, fc_b[l]);
    }
  });
}

void ref_gaussian_fill(uint64_t seed, double* out, int64_t n) {
  hpsim::GaussianSampler g(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = g.next();
}

int ref_count_stats(const or_model_spec* spec, int64_t out[5]) {
  return guarded([&] {
    auto s = hpsim::count_stats(to_spec(spec));
    out[0] = s.conv_params;
    out[1] = s.fc_params;
    out[2] = s.conv_flops;
    out[3] = s.fc_flops;
    out[4] = s.last_conv_activation_size;
  });
}

int ref_conv2d_forward(int precision, const double* x, int64_t B, int64_t C, int64_t H, int64_t W,
                       const double* k, int64_t F, int64_t R, int64_t S, int stride, int pad,
                       double* y) {
  return guarded([&] {
    auto p = prec(precision);
    auto out = hpsim::conv2d_forward(from_doubles({B, C, H, W}, x, p), from_doubles({F, C, R, S}, k, p),
                                     stride, pad);
    to_doubles(out, y);
  });
}

int ref_conv2d_backward(int precision, const double* x, int64_t B, int64_t C, int64_t H, int64_t W,
                        const double* k, int64_t F, int64_t R, int64_t S, int stride, int pad,
                        const double* gy, int64_t OH, int64_t OW, double* gx, double* gk) {
  return guarded([&] {
    auto p = prec(precision);
    auto g = hpsim::conv2d_backward(from_doubles({B, C, H, W}, x, p), from_doubles({F, C, R, S}, k, p),
                                    from_doubles({B, F, OH, OW}, gy, p), stride, pad);
    to_doubles(g.grad_input, gx);
    to_doubles(g.grad_kernels, gk);
  });
}

int ref_matmul(int precision, int variant, const double* a, const double* b, double* c, int64_t a0,
               int64_t a1, int64_t b0, int64_t b1) {
  return guarded([&] {
    auto p = prec(precision);
    auto A = from_doubles({a0, a1}, a, p), B = from_doubles({b0, b1}, b, p);
    auto C = variant == 0 ? hpsim::matmul(A, B) : variant == 1 ? hpsim::matmul_tn(A, B) : hpsim::matmul_nt(A, B);
    to_doubles(C, c);
  });
}

int ref_logistic_xent(int precision, const double* z, const double* t, int64_t B, int64_t L,
                      double* grad, double* loss) {
  return guarded([&] {
    auto p = prec(precision);
    auto r = hpsim::logistic_xent(from_doubles({B, L}, z, p), from_doubles({B, L}, t, p));
    *loss = r.loss;
    to_doubles(r.grad_logits, grad);
  });
}

int ref_momentum_update(int precision, double* w, double* d, const double* g, int64_t n, double lr,
                        double mu, double wd) {
  return guarded([&] {
    auto p = prec(precision);
    auto W = from_doubles({n}, w, p), D = from_doubles({n}, d, p);
    auto G = from_doubles({n}, g, p);
    hpsim::momentum_update(W, D, G, lr, mu, wd);
    to_doubles(W, w);
    to_doubles(D, d);
  });
}

double ref_lr_at(double progress, double base_lr, int* status) {
  double r = 0.0;
  *status = guarded([&] { r = hpsim::lr_at(progress, base_lr); });
  return r;
}

// SingleTrainer (the oracle shim of reference.hpp) -----------------------
void* ref_single_create(const or_model_spec* spec, uint64_t seed, int precision, int* status) {
  hpsim::SingleTrainer* t = nullptr;
  *status = guarded([&] { t = new hpsim::SingleTrainer(to_spec(spec), seed, prec(precision)); });
  return t;
}

void ref_single_destroy(void* h) { delete static_cast<hpsim::SingleTrainer*>(h); }

int ref_single_step(void* h, const double* batch, const double* targets, int64_t B,
                    const or_hyper* hyper, double lr, double* loss) {
  return guarded([&] {
    auto* t = static_cast<hpsim::SingleTrainer*>(h);
    const auto& m = t->model();
    auto p = m.precision;
    auto X = from_doubles({B, m.spec.input_shape[0], m.spec.input_shape[1], m.spec.input_shape[2]}, batch, p);
    auto T = from_doubles({B, m.spec.num_classes}, targets, p);
    *loss = t->step(X, T, to_hyper(hyper), lr);
  });
}

int ref_single_read(void* h, int which, int layer, double* dst, int64_t n) {
  return guarded([&] {
    const auto& m = static_cast<hpsim::SingleTrainer*>(h)->model();
    const hpsim::Tensor* t = nullptr;
    if (which == 0) t = &m.conv.at(layer).kernels;
    if (which == 1) t = &m.conv.at(layer).bias;
    if (which == 2) t = &m.fc.at(layer).weight;
    if (which == 3) t = &m.fc.at(layer).bias;
    if (!t || t->size() != n) throw hpsim::DimensionError("single_read: bad tensor");
    to_doubles(*t, dst);
  });
}

}  // extern "C"
