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

  int workers() const { return config_.workers; }
  const ClusterConfig& config() const { return config_; }
  const ModelSpec& spec() const { return spec_; }

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
  ModelSpec spec_;
  ClusterConfig config_;
  hp_cluster* h_ = nullptr;
};

}  // namespace hpsim_b200
