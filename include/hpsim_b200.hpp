// hpsim_b200.hpp — header-only C++ facade over the C ABI (hpsim_b200.h) that
// re-presents the reference's interface: hpsim::ModelSpec / ClusterConfig /
// HyperParams / Cluster / StepMetrics / StepTrace and the four exception
// types (/root/reference/proj/core/include/hpsim/{model,cluster,optimizer,
// errors}.hpp). A caller of hpsim::Cluster switches by including this header
// and linking libhpsim_b200.so; tensors are passed as host (or device) float
// pointers in the reference's layouts instead of hpsim::Tensor objects.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>
#if __cplusplus >= 202002L
#include <span>
#endif

#include "hpsim_b200.h"

namespace hpsim_b200 {

// errors.hpp:22-44
class DimensionError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DomainError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class UsageError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == HP_OK) return;
  const std::string m = hp_last_error();
  switch (rc) {
    case HP_ERR_CONFIG: throw ConfigError(m);
    case HP_ERR_DIMENSION: throw DimensionError(m);
    case HP_ERR_DOMAIN: throw DomainError(m);
    case HP_ERR_USAGE: throw UsageError(m);
    default: throw std::runtime_error(m);  // CUDA / NCCL
  }
}

enum class Scheme { A = HP_SCHEME_A, B = HP_SCHEME_B, C = HP_SCHEME_C };  // cluster.hpp:36
enum class Precision { kSingle = HP_PRECISION_SINGLE, kDouble = HP_PRECISION_DOUBLE };
enum class MathMode { kBF16 = HP_MATH_BF16, kTF32 = HP_MATH_TF32, kF32x3 = HP_MATH_F32X3 };
enum class Phase { kConvFwd, kFcFwd, kFcBwd, kConvBwd, kSync };  // cluster.hpp:86

// model.hpp:24-37 (+ the AlexNet superset, off by default)
struct ConvLayerSpec {
  std::int64_t in_channels = 0;
  std::int64_t out_channels = 0;
  int kernel = 0;
  int stride = 1;
  int pad = 0;
  bool relu = true;
  bool floor_mode = false;
  int lrn_size = 0;
  double lrn_alpha = 0.0, lrn_beta = 0.0, lrn_k = 0.0;
  int pool_kernel = 0, pool_stride = 0;
};

struct FcLayerSpec {
  std::int64_t in_dim = 0;
  std::int64_t out_dim = 0;
  bool relu = false;
};

struct ModelSpec {  // model.hpp:39-58
  std::vector<ConvLayerSpec> conv_layers;
  std::vector<FcLayerSpec> fc_layers;
  std::vector<std::int64_t> input_shape;  // C, H, W
  std::int64_t num_classes = 0;
};

struct ClusterConfig {  // cluster.hpp:59-68
  int workers = 1;
  std::int64_t per_worker_batch = 128;
  Scheme scheme = Scheme::B;
  bool variable_batch = false;
  Precision precision = Precision::kSingle;
  std::uint64_t seed = 0;
  // B200 fields
  MathMode math_mode = MathMode::kBF16;
  bool nccl = false;  // one worker per process (rank) instead of K logical workers
  int rank = 0;
  int device = -1;
  std::array<unsigned char, 128> nccl_id{};
};

struct HyperParams {  // optimizer.hpp:27-51 (schedule fields are host-side)
  double momentum = 0.9;
  double lr = 0.01;
  double weight_decay = 0.0;
  std::optional<double> fc_partial_lr;
};

struct TraceEvent {  // cluster.hpp:91-97
  Phase phase = Phase::kConvFwd;
  int sub_batch = -1;
  int worker = -1;
  std::int64_t bytes_total = 0;
  std::int64_t bytes_max_sender = 0;
};

struct StepTrace {  // cluster.hpp:99-109
  std::vector<TraceEvent> events;
  int count(Phase p) const {
    int n = 0;
    for (const auto& e : events) n += e.phase == p ? 1 : 0;
    return n;
  }
  int pass_count() const {
    int n = 0;
    for (const auto& e : events) n += e.phase != Phase::kSync ? 1 : 0;
    return n;
  }
};

struct StepMetrics {  // cluster.hpp:111-117
  double loss = 0.0;
  int fc_update_count = 0;
  int conv_update_count = 0;
  std::array<std::int64_t, 4> bytes_sent{};
};

// Minimal host tensor standing in for hpsim::Tensor (tensor.hpp:40-90) at
// this boundary: row-major float32 storage plus a shape. The reference's
// Tensor carries its precision; the B200 path computes in fp32/bf16 and takes
// float32 host data, so a kDouble caller converts once (Tensor::converted).
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<std::int64_t> shape) : shape_(std::move(shape)), data_(count(shape_)) {}
  Tensor(std::vector<std::int64_t> shape, std::vector<float> values) : shape_(std::move(shape)), data_(std::move(values)) {
    if (static_cast<std::int64_t>(data_.size()) != count(shape_))
      throw DimensionError("Tensor: value count does not match shape");
  }
  const std::vector<std::int64_t>& shape() const { return shape_; }
  std::size_t rank() const { return shape_.size(); }
  std::int64_t dim(std::size_t i) const { return shape_.at(i); }
  std::int64_t size() const { return static_cast<std::int64_t>(data_.size()); }
  float* data() { return data_.data(); }
  const float* data() const { return data_.data(); }

 private:
  static std::int64_t count(const std::vector<std::int64_t>& s) {
    std::int64_t n = 1;
    for (auto d : s) n *= d;
    return n;
  }
  std::vector<std::int64_t> shape_;
  std::vector<float> data_;
};

struct ConvParams {  // model.hpp:75-78
  Tensor kernels;    // [F x C x R x S]
  Tensor bias;       // [F]
};
struct FcParams {  // model.hpp:80-83
  Tensor weight;   // [in_dim x out_dim] (a worker's shard: [in_dim x out_i])
  Tensor bias;     // [out_dim]
};
struct ByteCounters {  // cluster.hpp:41-57, indexed by Phase (kConvFwd .. kConvBwd)
  std::array<std::int64_t, 4> sent{};
  std::array<std::int64_t, 4> received{};
};
// cluster.hpp:77-84. Cluster::worker() returns a host snapshot read back from
// the device (the reference returns a reference into host memory).
struct WorkerState {
  int worker_id = 0;
  std::vector<ConvParams> conv_params;
  std::vector<ConvParams> conv_momentum;
  std::vector<FcParams> fc_shard;
  std::vector<FcParams> fc_momentum;
  ByteCounters bytes;
};
struct Model {  // model.hpp:88-94
  ModelSpec spec;
  std::vector<ConvParams> conv;
  std::vector<FcParams> fc;
  std::uint64_t rng_seed = 0;
};

class Cluster {  // cluster.hpp:178-212
 public:
  struct StepResult {
    StepMetrics metrics;
    StepTrace trace;
  };

  Cluster(const ModelSpec& spec, const ClusterConfig& config) : spec_(spec), config_(config) {
    std::vector<hp_conv_layer> conv;
    for (const auto& l : spec.conv_layers)
      conv.push_back({l.in_channels, l.out_channels, l.kernel, l.stride, l.pad, l.relu ? 1 : 0,
                      l.floor_mode ? 1 : 0, l.lrn_size, l.lrn_alpha, l.lrn_beta, l.lrn_k,
                      l.pool_kernel, l.pool_stride});
    std::vector<hp_fc_layer> fc;
    for (const auto& l : spec.fc_layers) fc.push_back({l.in_dim, l.out_dim, l.relu ? 1 : 0});
    if (spec.input_shape.size() != 3) throw ConfigError("model.input_shape: expected [C,H,W]");
    hp_model_spec s{conv.data(), static_cast<int32_t>(conv.size()), fc.data(),
                    static_cast<int32_t>(fc.size()), {spec.input_shape[0], spec.input_shape[1],
                                                      spec.input_shape[2]},
                    spec.num_classes};
    hp_cluster_config c{};
    c.workers = config.workers;
    c.per_worker_batch = config.per_worker_batch;
    c.scheme = static_cast<int32_t>(config.scheme);
    c.variable_batch = config.variable_batch ? 1 : 0;
    c.precision = static_cast<int32_t>(config.precision);
    c.seed = config.seed;
    c.math_mode = static_cast<int32_t>(config.math_mode);
    c.transport = config.nccl ? HP_TRANSPORT_NCCL : HP_TRANSPORT_LOGICAL;
    c.rank = config.rank;
    c.device = config.device;
    for (int i = 0; i < 128; ++i) c.nccl_id[i] = config.nccl_id[i];
    check(hp_cluster_create(&s, &c, &h_));
  }
  ~Cluster() { hp_cluster_destroy(h_); }
  Cluster(const Cluster&) = delete;
  Cluster& operator=(const Cluster&) = delete;

  // batches[i]: worker i's [b][C][H][W], targets[i]: [b][L] (host pointers,
  // or device pointers with device = true). K entries (logical), 1 (NCCL).
  StepResult run_step(const std::vector<const float*>& batches, const std::vector<const float*>& targets,
                      const HyperParams& hp, double lr, bool device = false) {
    hp_hyper h{hp.momentum, hp.lr, hp.weight_decay, hp.fc_partial_lr ? 1 : 0,
               hp.fc_partial_lr.value_or(0.0)};
    hp_step_metrics m{};
    check(hp_cluster_run_step(h_, batches.data(), targets.data(), device ? HP_MEM_DEVICE : HP_MEM_HOST,
                              &h, lr, &m));
    StepResult r;
    r.metrics.loss = m.loss;
    r.metrics.fc_update_count = m.fc_update_count;
    r.metrics.conv_update_count = m.conv_update_count;
    for (int i = 0; i < 4; ++i) r.metrics.bytes_sent[i] = m.bytes_sent[i];
    std::vector<hp_trace_event> ev(static_cast<size_t>(m.n_events));
    hp_cluster_trace(h_, ev.data(), m.n_events);
    for (const auto& e : ev)
      r.trace.events.push_back({static_cast<Phase>(e.phase), e.sub_batch, e.worker, e.bytes_total,
                                e.bytes_max_sender});
    return r;
  }

  // cluster.hpp:190-192: the reference's signature over Tensor objects.
  // Shapes are checked here (model.cpp:204-214 DimensionError; rows per
  // worker, cluster.cpp:444-457 UsageError) before any native call.
#if __cplusplus >= 202002L
  StepResult run_step(std::span<const Tensor> batches, std::span<const Tensor> targets, const HyperParams& hp,
                      double lr) {
    return run_step_tensors(batches.data(), batches.size(), targets.data(), targets.size(), hp, lr);
  }
#endif
  StepResult run_step(const std::vector<Tensor>& batches, const std::vector<Tensor>& targets, const HyperParams& hp,
                      double lr) {
    return run_step_tensors(batches.data(), batches.size(), targets.data(), targets.size(), hp, lr);
  }

  int workers() const { return config_.workers; }
  const ClusterConfig& config() const { return config_; }
  const ModelSpec& spec() const { return spec_; }

  // cluster.hpp:197 (host snapshot; NCCL transport: the local rank's worker).
  WorkerState worker(int i) const {
    WorkerState w;
    w.worker_id = i;
    for (int l = 0; l < static_cast<int>(spec_.conv_layers.size()); ++l) {
      const auto& c = spec_.conv_layers[static_cast<std::size_t>(l)];
      const std::vector<std::int64_t> ks{c.out_channels, c.in_channels, c.kernel, c.kernel}, bs{c.out_channels};
      w.conv_params.push_back({Tensor(ks, param(i, HP_P_CONV_K, l)), Tensor(bs, param(i, HP_P_CONV_B, l))});
      w.conv_momentum.push_back({Tensor(ks, param(i, HP_P_CONV_K + HP_P_MOMENTUM, l)),
                                 Tensor(bs, param(i, HP_P_CONV_B + HP_P_MOMENTUM, l))});
    }
    for (int l = 0; l < static_cast<int>(spec_.fc_layers.size()); ++l) {
      const auto& f = spec_.fc_layers[static_cast<std::size_t>(l)];
      const std::vector<float> b = param(i, HP_P_FC_B, l);
      const std::int64_t out = static_cast<std::int64_t>(b.size());
      const std::vector<std::int64_t> ws{f.in_dim, out}, bs{out};
      w.fc_shard.push_back({Tensor(ws, param(i, HP_P_FC_W, l)), Tensor(bs, b)});
      w.fc_momentum.push_back({Tensor(ws, param(i, HP_P_FC_W + HP_P_MOMENTUM, l)),
                               Tensor(bs, param(i, HP_P_FC_B + HP_P_MOMENTUM, l))});
    }
    check(hp_cluster_worker_bytes(h_, i, w.bytes.sent.data(), w.bytes.received.data()));
    return w;
  }

  // cluster.hpp:199-201 / cluster.cpp:417-437: worker 0's conv replica and
  // the fc shards pasted back into whole matrices (NCCL: collective).
  Model gathered_model() const {
    Model m;
    m.spec = spec_;
    m.rng_seed = config_.seed;
    std::vector<float*> ck, cb, fw, fb;
    for (const auto& c : spec_.conv_layers) {
      m.conv.push_back({Tensor({c.out_channels, c.in_channels, c.kernel, c.kernel}), Tensor({c.out_channels})});
      ck.push_back(m.conv.back().kernels.data());
      cb.push_back(m.conv.back().bias.data());
    }
    for (const auto& f : spec_.fc_layers) {
      m.fc.push_back({Tensor({f.in_dim, f.out_dim}), Tensor({f.out_dim})});
      fw.push_back(m.fc.back().weight.data());
      fb.push_back(m.fc.back().bias.data());
    }
    check(hp_cluster_gather_model(h_, ck.data(), cb.data(), fw.data(), fb.data()));
    return m;
  }

  // WorkerState tensors in reference layouts (which: HP_P_*).
  std::vector<float> param(int worker, int which, int layer) const {
    const int64_t n = hp_cluster_param_size(h_, worker, which, layer);
    if (n < 0) throw UsageError("param: bad worker/which/layer");
    std::vector<float> out(static_cast<size_t>(n));
    check(hp_cluster_read_param(h_, worker, which, layer, out.data(), n));
    return out;
  }

  void set_skip_sync_broadcast(bool v) { check(hp_cluster_set_skip_sync_broadcast(h_, v ? 1 : 0)); }

 private:
  StepResult run_step_tensors(const Tensor* b, std::size_t nb, const Tensor* t, std::size_t nt,
                              const HyperParams& hp, double lr) {
    const std::size_t k = config_.nccl ? 1u : static_cast<std::size_t>(config_.workers);
    if (nb != k || nt != k)
      throw UsageError("run_step: expected " + std::to_string(k) + " batches and targets, got " +
                       std::to_string(nb) + " / " + std::to_string(nt));
    std::vector<const float*> bp, tp;
    for (std::size_t i = 0; i < k; ++i) {
      const Tensor& x = b[i];
      const Tensor& y = t[i];
      if (x.rank() < 1 || y.rank() < 1 || x.dim(0) != config_.per_worker_batch || y.dim(0) != config_.per_worker_batch)
        throw UsageError("run_step: worker " + std::to_string(i) + " batch must hold exactly " +
                         std::to_string(config_.per_worker_batch) + " examples");
      if (x.rank() != 4 || x.dim(1) != spec_.input_shape[0] || x.dim(2) != spec_.input_shape[1] ||
          x.dim(3) != spec_.input_shape[2])
        throw DimensionError("forward: batch shape does not match model input");
      if (y.rank() != 2 || y.dim(1) != spec_.num_classes)
        throw DimensionError("logistic_xent: target shape does not match the logits");
      bp.push_back(x.data());
      tp.push_back(y.data());
    }
    return run_step(bp, tp, hp, lr, false);
  }

  ModelSpec spec_;
  ClusterConfig config_;
  hp_cluster* h_ = nullptr;
};

}  // namespace hpsim_b200
