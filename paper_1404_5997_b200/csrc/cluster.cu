// B200 hybrid-parallel training step: device-side replacement of
// hpsim::Cluster (src/cluster.cpp:394-711).
//
// Per worker (one GPU per worker with NCCL; K workers on one GPU with the
// logical transport):
//   conv stack (data parallel): im2col -> tcgen05 GEMM (bias+ReLU fused)
//     -> LRN -> max-pool, activations NHWC in the operand type.
//   boundary: scheme A all-gather / B per-turn broadcast / C per-turn slice
//     all-gather of the [b][A] sample-major conv tops (cluster.cpp:113-194).
//   fc stack (model parallel, worker i owns output rows shard_range(out,K,i)):
//     feature-major activations [features][n] so the column all-gather and the
//     partial-dX reduce-scatter are plain NCCL chunked collectives.
//   backward: fc wgrad/dgrad GEMMs, boundary reduce-scatter / reduce back to
//     the owners (return_gradients, cluster.cpp:196-269), conv backward
//     (pool/LRN/ReLU backward, wgrad GEMM, dgrad GEMM + col2im), conv-gradient
//     all-reduce (sync_conv_gradients, cluster.cpp:273-319), fused momentum SGD.
// Byte counters and the phase trace are the reference's analytic integers,
// computed on the host exactly as cluster.cpp:466-673 does.
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <chrono>
#include <map>
#include <thread>
#include <string>
#include <tuple>

#include "cluster.hpp"
#include "comm.hpp"
#include "errors.hpp"
#include "gemm.cuh"
#include "kernels.cuh"
#include "rng.hpp"

#include <nvtx3/nvToolsExt.h>

namespace hp {

// NVTX ranges around the step's phases (host-side enqueue; visible in any
// NVTX-aware timeline). Cheap when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace {

long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

void shard(long long total, int parts, int idx, long long* b, long long* e) {
  const long long base = total / parts;  // cluster.cpp:69-75
  *b = base * idx;
  *e = idx == parts - 1 ? total : *b + base;
}

bool out_dim(long long in, int k, int s, int p, bool floor_mode, long long* out) {
  const long long num = in + 2LL * p - k;  // model.cpp:25-35
  if (num < 0 || (!floor_mode && num % s != 0)) return false;
  *out = num / s + 1;
  return true;
}

std::string num(long long v) { return std::to_string(v); }

// logistic_xent's DomainError (tensor.cpp:600-603) on host targets: a
// branch-free (vectorisable) scan first, the exact message only on failure.
void check_targets(const float* t, long long n) {
  int bad = 0;
  for (long long e = 0; e < n; ++e) bad |= static_cast<int>(t[e] < 0.f) | static_cast<int>(t[e] > 1.f);
  if (!bad) return;
  for (long long e = 0; e < n; ++e)
    if (t[e] < 0.f || t[e] > 1.f)
      domain_error("logistic_xent: target " + std::to_string(static_cast<double>(t[e])) +
                   " outside [0,1] at flat index " + num(e));
}

}  // namespace

Geometry make_geometry(const hp_model_spec* s, int K, long long b) {
  Geometry g;
  if (s->n_conv < 1 || !s->conv) config_error("model.conv_layers: at least one conv layer required");
  if (s->n_fc < 1 || !s->fc) config_error("model.fc_layers: at least one fc layer required");
  for (int i = 0; i < 3; ++i)
    if (s->input_shape[i] <= 0) config_error("model.input_shape: dimensions must be positive");
  g.conv.assign(s->conv, s->conv + s->n_conv);
  g.fc.assign(s->fc, s->fc + s->n_fc);
  std::memcpy(g.input, s->input_shape, sizeof g.input);
  g.num_classes = s->num_classes;
  long long c = s->input_shape[0], h = s->input_shape[1], w = s->input_shape[2];
  for (int i = 0; i < s->n_conv; ++i) {
    const hp_conv_layer& l = s->conv[i];
    const std::string where = "model.conv_layers[" + num(i) + "]";
    if (l.in_channels != c)
      config_error(where + ".in_channels: expected " + num(c) + ", got " + num(l.in_channels));
    if (l.out_channels <= 0 || l.kernel <= 0 || l.stride <= 0 || l.pad < 0)
      config_error(where + ": out_channels/kernel/stride must be positive, pad non-negative");
    ConvGeom cg{};
    cg.C = static_cast<int>(c);
    cg.H = static_cast<int>(h);
    cg.W = static_cast<int>(w);
    cg.F = static_cast<int>(l.out_channels);
    cg.R = cg.S = l.kernel;
    cg.stride = l.stride;
    cg.pad = l.pad;
    long long oh, ow;
    if (!out_dim(h, l.kernel, l.stride, l.pad, l.floor_mode != 0, &oh))
      config_error(where + " (height): output dimension (" + num(h) + "+2*" + num(l.pad) + "-" +
                   num(l.kernel) + ")/" + num(l.stride) + "+1 is not a positive integer");
    if (!out_dim(w, l.kernel, l.stride, l.pad, l.floor_mode != 0, &ow))
      config_error(where + " (width): output dimension (" + num(w) + "+2*" + num(l.pad) + "-" +
                   num(l.kernel) + ")/" + num(l.stride) + "+1 is not a positive integer");
    cg.OH = static_cast<int>(oh);
    cg.OW = static_cast<int>(ow);
    cg.OWs = cg.OW;
    cg.OHs = cg.OH;
    cg.relu = l.relu != 0;
    if (l.lrn_size < 0) config_error(where + ".lrn_size: must be >= 0");
    if (l.lrn_size > 5 && l.pool_kernel > 0)
      config_error(where + ".lrn_size: LRN fused with pooling supports sizes up to 5 on B200");
    cg.lrn_n = l.lrn_size;
    cg.lrn_alpha = static_cast<float>(l.lrn_alpha);
    cg.lrn_beta = static_cast<float>(l.lrn_beta);
    cg.lrn_k = static_cast<float>(l.lrn_k);
    cg.pk = l.pool_kernel;
    cg.ps = l.pool_stride;
    cg.PH = cg.OH;
    cg.PW = cg.OW;
    if (cg.pk > 0) {
      if (cg.ps <= 0) config_error(where + ".pool_stride: must be positive");
      if (cg.OH < cg.pk || cg.OW < cg.pk) config_error(where + ".pool_kernel: larger than the conv output");
      cg.PH = (cg.OH - cg.pk) / cg.ps + 1;
      cg.PW = (cg.OW - cg.pk) / cg.ps + 1;
    }
    // B200 operand layout: NHWC rows of F channels feed TMA (16-byte rows).
    if (cg.F % 8 != 0)
      config_error(where + ".out_channels: must be a multiple of 8 on B200 (got " + num(cg.F) +
                   "); TMA operand rows are 16-byte aligned");
    cg.Kc = cg.R * cg.S * cg.C;
    cg.ldk = round_up(cg.Kc, 8);
    cg.P = b * cg.OH * cg.OW;
    cg.PP = b * cg.PH * cg.PW;
    cg.ldp = round_up(cg.P, 8);
    g.cg.push_back(cg);
    c = cg.F;
    h = cg.PH;
    w = cg.PW;
  }
  g.A = c * h * w;
  long long dim = g.A;
  for (int i = 0; i < s->n_fc; ++i) {
    const hp_fc_layer& l = s->fc[i];
    const std::string where = "model.fc_layers[" + num(i) + "]";
    if (l.in_dim != dim)
      config_error(where + ".in_dim: expected " + num(dim) + " (flattened preceding output), got " +
                   num(l.in_dim));
    if (l.out_dim <= 0) config_error(where + ".out_dim: must be positive");
    FcGeom fg;
    fg.in = l.in_dim;
    fg.out = l.out_dim;
    fg.relu = l.relu != 0;
    long long mx = 0;
    for (int k = 0; k < K; ++k) {
      long long b0, b1;
      shard(l.out_dim, K, k, &b0, &b1);
      fg.c0.push_back(b0);
      fg.c1.push_back(b1);
      mx = std::max(mx, b1 - b0);
    }
    fg.cmax = round_up(std::max(1LL, mx), 8);
    fg.Ip = i == 0 ? g.A : K * g.fg.back().cmax;
    g.fg.push_back(fg);
    dim = l.out_dim;
  }
  if (s->num_classes <= 0) config_error("model.num_classes: must be positive");
  if (dim != s->num_classes)
    config_error("model.fc_layers: last out_dim " + num(dim) + " does not match num_classes " +
                 num(s->num_classes));
  return g;
}

void step_accounting(const Geometry& g_, int K, long long b, int scheme_,
                     std::vector<std::array<int64_t, 4>>& sent,
                     std::vector<std::array<int64_t, 4>>& received, std::vector<hp_trace_event>& trace,
                     int64_t* bytes_sent) {
  const long long elt = 4, row_bytes = g_.A * elt;
  if (scheme_ == HP_SCHEME_DP) {
    // Pure data parallelism (no reference counterpart): no boundary exchange,
    // no FC-internal traffic; the conv and FC gradient vectors are each
    // all-reduced, charged with the reference's sync formula
    // (G - s_i)*e + (K-1)*s_i*e (cluster.cpp:296-304).
    long long Gc = 0, Gf = 0;
    for (const auto& c : g_.cg) Gc += static_cast<long long>(c.F) * c.Kc + c.F;
    for (const auto& f : g_.fg) Gf += f.in * f.out + f.out;
    long long total = 0, mx = 0;
    for (int i = 0; i < K; ++i) {
      long long sc = 0, sf = 0;
      if (K > 1) {
        long long s0, s1;
        shard(Gc, K, i, &s0, &s1);
        sc = (Gc - (s1 - s0)) * elt + (K - 1) * (s1 - s0) * elt;
        shard(Gf, K, i, &s0, &s1);
        sf = (Gf - (s1 - s0)) * elt + (K - 1) * (s1 - s0) * elt;
      }
      sent[i][HP_MSG_CONV_SYNC] += sc;
      received[i][HP_MSG_CONV_SYNC] += sc;
      sent[i][HP_MSG_FC_GRADIENTS] += sf;
      received[i][HP_MSG_FC_GRADIENTS] += sf;
      bytes_sent[HP_MSG_CONV_SYNC] += sc;
      bytes_sent[HP_MSG_FC_GRADIENTS] += sf;
      total += sc + sf;
      mx = std::max(mx, sc + sf);
    }
    trace.clear();
    trace.push_back({HP_PHASE_CONV_FWD, -1, -1, 0, 0});
    trace.push_back({HP_PHASE_FC_FWD, 0, -1, 0, 0});
    trace.push_back({HP_PHASE_FC_BWD, 0, -1, 0, 0});
    trace.push_back({HP_PHASE_CONV_BWD, -1, -1, 0, 0});
    trace.push_back({HP_PHASE_SYNC, -1, -1, total, mx});
    return;
  }
  const int num_sub = scheme_ == HP_SCHEME_A ? 1 : K;
  const long long n_ = scheme_ == HP_SCHEME_A ? K * b : b;
  auto charge = [&](int i, int cls, long long s, long long r) {
    sent[i][cls] += s;
    received[i][cls] += r;
    bytes_sent[cls] += s;
  };
  auto ex_sent = [&](int j, int i) -> long long {
    if (K <= 1) return 0;
    if (scheme_ == HP_SCHEME_A) return (K - 1) * b * row_bytes;
    if (scheme_ == HP_SCHEME_B) return i == j ? (K - 1) * b * row_bytes : 0;
    return (K - 1) * (b / K) * row_bytes;
  };
  const long long n = n_;
  std::vector<hp_trace_event> fwd(num_sub), bwd(num_sub);
  for (int j = 0; j < num_sub; ++j) {
    long long total = 0, mx = 0;
    for (int i = 0; i < K; ++i) {
      long long inbound = 0;
      if (K > 1) inbound = scheme_ == HP_SCHEME_B ? (i == j ? 0 : b * row_bytes) : ex_sent(j, i);
      charge(i, HP_MSG_FC_ACTIVATIONS, ex_sent(j, i), inbound);
      total += ex_sent(j, i);
      mx = std::max(mx, ex_sent(j, i));
    }
    fwd[j] = {HP_PHASE_FC_FWD, j, scheme_ == HP_SCHEME_B ? j : -1, total, mx};
    for (size_t l = 0; l < g_.fg.size(); ++l) {
      const FcGeom& f = g_.fg[l];
      for (int i = 0; i < K; ++i) {
        const long long ns = f.c1[i] - f.c0[i];
        charge(i, HP_MSG_FC_INTERNAL, (K - 1) * n * ns * elt, n * (f.out - ns) * elt);
      }
    }
    for (size_t li = g_.fg.size(); li-- > 1;) {
      const long long part = n * g_.fg[li].in * elt;
      for (int i = 0; i < K; ++i) charge(i, HP_MSG_FC_INTERNAL, (K - 1) * part, (K - 1) * part);
    }
  }
  for (int j = 0; j < num_sub; ++j) {
    long long total = 0, mx = 0;
    for (int i = 0; i < K; ++i) {
      long long s = 0;
      if (scheme_ == HP_SCHEME_A) s = K > 1 ? (K - 1) * b * row_bytes : 0;
      else if (scheme_ == HP_SCHEME_B) s = i != j ? b * row_bytes : 0;
      else s = K > 1 ? (K - 1) * (b / K) * row_bytes : 0;
      long long r = s;
      if (scheme_ == HP_SCHEME_B) r = (i == j && K > 1) ? (K - 1) * b * row_bytes : 0;
      charge(i, HP_MSG_FC_GRADIENTS, s, r);
      total += s;
      mx = std::max(mx, s);
    }
    bwd[j] = {HP_PHASE_FC_BWD, j, scheme_ == HP_SCHEME_B ? j : -1, total, mx};
  }
  trace.clear();
  trace.push_back({HP_PHASE_CONV_FWD, -1, -1, 0, 0});
  for (int j = 0; j < num_sub; ++j) {
    trace.push_back(fwd[j]);
    trace.push_back(bwd[j]);
  }
  trace.push_back({HP_PHASE_CONV_BWD, -1, -1, 0, 0});
  long long G = 0;
  for (const auto& c : g_.cg) G += static_cast<long long>(c.F) * c.Kc + c.F;
  long long total = 0, mx = 0;
  for (int i = 0; i < K; ++i) {
    long long s = 0;
    if (K > 1) {
      long long s0, s1;
      shard(G, K, i, &s0, &s1);
      const long long shard_bytes = (s1 - s0) * elt;
      s = (G * elt - shard_bytes) + (K - 1) * shard_bytes;
    }
    charge(i, HP_MSG_CONV_SYNC, s, s);
    total += s;
    mx = std::max(mx, s);
  }
  trace.push_back({HP_PHASE_SYNC, -1, -1, total, mx});
}

namespace {

struct DevArena {
  std::vector<void*> ptrs;
  size_t total = 0;
  void* alloc(size_t bytes) {
    void* p = nullptr;
    bytes = std::max<size_t>(bytes, 256);
    HP_CUDA(cudaMalloc(&p, bytes));
    HP_CUDA(cudaMemset(p, 0, bytes));
    ptrs.push_back(p);
    total += bytes;
    return p;
  }
  template <class T>
  T* make(long long n) {
    return static_cast<T*>(alloc(static_cast<size_t>(n) * sizeof(T)));
  }
  ~DevArena() {
    for (void* p : ptrs) cudaFree(p);
  }
};

template <class TA>
struct Worker {
  int gid = 0;
  // inputs
  float* x_nchw = nullptr;  // staging for host batches
  float* xin[2] = {nullptr, nullptr};  // prefetch slots: images
  float* tin[2] = {nullptr, nullptr};  // prefetch slots: targets
  TA* x0 = nullptr;         // [b][H][W][C]
  float* targets = nullptr; // [b][L]
  // conv stack
  std::vector<TA*> col, act, lrn, pool, dz;
  std::vector<float*> lrn_d, dcol, gstage;
  std::vector<uint8_t*> widx;  // pool argmax as window offset
  std::vector<TA*> wrot;        // rotated kernels [C][R][S][F] (implicit dgrad)
  TA* z = nullptr;              // s2d layer 0: space-to-depth input [b][Zh][Zw][Cz]
  TA* wz = nullptr;             // s2d layer 0: kernels [F][Rq][Rq][Cz] (operand type)
  float* dwz = nullptr;         // s2d layer 0: wgrad in the s2d layout
  float* bias2 = nullptr;       // s2d pixel pairs: conv1 bias twice (the 2F GEMM columns)
  const float* x_src = nullptr; // this step's NCHW batch (device)
  // conv params: [kernels F x ldk | bias F] per layer, one arena
  float *cp = nullptr, *cm = nullptr, *cgr = nullptr;
  float* cgr_local = nullptr;  // skip_sync_broadcast: this worker's pre-all-reduce conv gradients
  TA* cpt = nullptr;  // operand copy (bf16 mode)
  // fc stack
  // boundary buffers, double-buffered by turn parity: turn j+1's exchange
  // fills slot (j+1)&1 while turn j's FC compute reads slot j&1
  TA* xb[2] = {nullptr, nullptr};     // [n][A] boundary input
  float* tb[2] = {nullptr, nullptr};  // [n][L] routed targets
  float* fd0[2] = {nullptr, nullptr}; // [n][A] partial boundary gradient (fc0 dgrad -> return)
  std::vector<TA*> fx;     // fx[l] (l>=1): [K*cmax(l-1)][ldn]
  float* logits = nullptr; // [cmax_last][ldn]
  std::vector<TA*> fdz;    // [cmax_l][ldn]
  std::vector<float*> fdpart;
  float* gflat = nullptr;  // [b][A]
  float *fp = nullptr, *fm = nullptr, *fgr = nullptr;
  TA* fpt = nullptr;
  double* loss_parts = nullptr;
  int* bad = nullptr;
  float* colsum_ws = nullptr;
  // GEMM plans
  std::vector<GemmPlan> conv_fwd, conv_wgrad, conv_dgrad, fc_fwd, fc_wgrad, fc_dgrad;
  std::vector<GemmPlan> last_fwd_slices;  // micro-pipelined last conv layer (scheme C): one plan per turn's slice
  GemmPlan fc0_slot1[3];  // fc layer 0 {fwd, wgrad, dgrad} over boundary slot 1 (slot 0: the vectors)
};

template <class TA>
class ClusterImpl final : public ClusterBase {
 public:
  ClusterImpl(const hp_model_spec* spec, const hp_cluster_config* cfg);
  ~ClusterImpl() override;
  void* stream() const override { return st_; }
  void prefetch(const float* const* batches, const float* const* targets) override;
  void rebuild_plans() override {
    HP_CUDA(cudaStreamSynchronize(st_));
    for (auto& kv : graphs_)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs_.clear();
    for (auto& w : w_) build_plans(w);
  }
  void run_step(const float* const* batches, const float* const* targets, int mem_kind,
                const hp_hyper& hp, double lr, hp_step_metrics* out) override;
  void marker_graph(const float* const* batches, const float* const* targets, int mem_kind,
                    const hp_hyper& hp, double lr, std::vector<int>& tags,
                    std::vector<uint8_t>& reach) override;
  int64_t param_size(int worker, int which, int layer) const override;
  void read_param(int worker, int which, int layer, float* dst, int64_t n) override;
  int64_t read_decisions(int worker, int kind, int layer, void* dst, int64_t n) override;
  void fc_mask_now(int l, std::vector<uint8_t>& m);
  void capture_fc_masks(int j);
  std::vector<std::vector<uint8_t>> cap_fc_;  // debug capture: [turn * nf + layer] -> [n][out]
  void write_param(int worker, int which, int layer, const float* src, int64_t n) override;
  void gather_model(float* const* ck, float* const* cb, float* const* fw, float* const* fb) override;

 private:
  static constexpr int kTA = std::is_same<TA, float>::value ? kF32 : kBF16;
  Worker<TA>& local(int gid);
  const Worker<TA>* local_or_null(int gid) const;
  void build_plans(Worker<TA>& w);
  void conv_forward(Worker<TA>& w, int layers);
  void conv_forward_last_slice(Worker<TA>& w, int j);
  // Scheme C micro-pipelining: the last conv layer (and its
  // pool) runs in K image slices in turn order, and turn j's slice exchange
  // waits only for slice j -- turn 0's exchange runs under slices 1..K-1.
  bool slice_last_ = false;
  std::vector<cudaEvent_t> ev_slice_;
  bool slicing() const { return slice_last_ && !w_.empty() && !w_[0].last_fwd_slices.empty(); }
  const TA* stage_in(const Worker<TA>& w, int l) const;
  // what: 1 = the s2d operand copy (conv1), 2 = the dgrad operands (rotated kernels), 3 = both
  void rotate_all(Worker<TA>& w, int what = 3, cudaStream_t s = nullptr);
  struct ConvBwdState {
    const float* gout = nullptr;  // grad wrt the current stage's output
    bool dz_ready = false;        // dz already produced by the layer above's dgrad
  };
  void conv_backward_layer(Worker<TA>& w, int l, ConvBwdState& cs);
  void route_forward(int j, int slot, cudaStream_t s);
  void fc_forward_backward(int j, bool beta, int slot);
  void return_gradients(int j, int slot, cudaStream_t s);
  void marker(int tag, cudaStream_t s) {
    if (!markers && !tl_) return;
    launch_marker(tag, s, tl_, tl_cap_);
    ++launches_;
  }
  // Dev timeline (HP_DEV_TIMELINE=<csv path>): timestamped markers around every
  // GEMM and the main memory-bound kernels, on the stream each runs on; one
  // CSV row per marker per step (step, name, begin/end, ns). A diagnostic of
  // the streams' overlap -- the 1-thread marker kernels perturb the step.
  unsigned long long* tl_ = nullptr;
  int tl_cap_ = 0;
  std::vector<std::string> tl_names_;
  FILE* tl_file_ = nullptr;
  long long tl_step_ = 0;
  void tl_mark(const char* name, int layer, bool end, cudaStream_t s) {
    if (!tl_) return;
    const std::string key = std::string(name) + "[" + std::to_string(layer) + "]";
    size_t id = 0;
    while (id < tl_names_.size() && tl_names_[id] != key) ++id;
    if (id == tl_names_.size()) tl_names_.push_back(key);
    marker(1000000 + 2 * static_cast<int>(id) + (end ? 1 : 0), s);
  }
  void tl_flush() {
    if (!tl_) return;
    std::vector<unsigned long long> h(1 + 2 * static_cast<size_t>(tl_cap_));
    HP_CUDA(cudaMemcpy(h.data(), tl_, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    const unsigned long long n = std::min<unsigned long long>(h[0], static_cast<unsigned long long>(tl_cap_));
    for (unsigned long long i = 0; i < n; ++i) {
      const long long tag = static_cast<long long>(h[1 + 2 * i]);
      const unsigned long long t = h[2 + 2 * i];
      if (tag >= 1000000) {
        const size_t id = static_cast<size_t>((tag - 1000000) / 2);
        fprintf(tl_file_, "%lld,%s,%s,%llu\n", tl_step_, id < tl_names_.size() ? tl_names_[id].c_str() : "?",
                (tag & 1) ? "end" : "begin", t);
      } else {
        fprintf(tl_file_, "%lld,marker%lld,point,%llu\n", tl_step_, tag, t);
      }
    }
    fflush(tl_file_);
    ++tl_step_;
  }
  void sgd_fc(double lr, float gscale, bool has_gscale, const hp_hyper& hp);
  void sgd_conv(double lr, const hp_hyper& hp);
  void account(int num_sub, hp_step_metrics* out);
  void enqueue(const float* const* batches, const float* const* targets, int mem_kind,
               const hp_hyper& hp, double lr);
  struct GraphKey {
    std::vector<const void*> ptrs;
    int mem = 0;
    std::array<double, 4> scal{};
    bool operator<(const GraphKey& o) const {
      return std::tie(ptrs, mem, scal) < std::tie(o.ptrs, o.mem, o.scal);
    }
  };
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
    double flops = 0.0;
    int64_t h2d = 0, d2h = 0;
  };
  std::map<GraphKey, GraphEntry> graphs_;
  double* host_parts_ = nullptr;  // pinned: [nlocal][num_sub * xblocks]
  int* host_bad_ = nullptr;       // pinned: [nlocal]
  void gemm(const GemmPlan& p, const char* tag, int layer, cudaStream_t s = nullptr);
  void collect_profile();
  // param layout helpers
  long long conv_k_off(int l) const { return coff_[l]; }
  long long conv_b_off(int l) const { return coff_[l] + static_cast<long long>(g_.cg[l].F) * g_.cg[l].ldk; }
  long long fc_w_off(int l) const { return foff_[l]; }
  long long fc_b_off(int l) const { return foff_[l] + g_.fg[l].cmax * g_.fg[l].Ip; }
  long long fc_col(int l, long long i) const;  // reference input index -> device column
  void init_params();
  void refresh_copies(Worker<TA>& w);
  void upload_master(Worker<TA>& w, bool conv, const std::vector<float>& host);

  Geometry g_;
  int K_, math_, scheme_;
  bool dp_ = false;  // HP_SCHEME_DP: FC stack replicated (one shard), gradients all-reduced
  int fcK_ = 1;      // FC shards (K_, or 1 under DP)
  int sid(int gid) const { return dp_ ? 0 : gid; }  // FC shard index of a worker
  bool variable_;
  long long b_, n_, ldn_;
  int num_sub_, L_;
  uint64_t seed_;
  // One transport per concurrent stream (NCCL: one communicator each, split
  // from the first, so no two streams ever drive the same communicator):
  // comm_ FC-internal gathers/scatters + loss on st_, comm_x_ the boundary
  // exchange / gradient return on sr_, comm_s_ the conv-gradient all-reduce on sc_.
  std::unique_ptr<Comm> comm_, comm_x_, comm_s_;
  cudaStream_t sr_ = nullptr;  // boundary exchange + gradient return (overlaps the FC compute)
  cudaEvent_t ev_conv_ = nullptr;          // conv tops + targets final on st_
  cudaEvent_t ev_xready_[2] = {nullptr, nullptr};  // boundary slot filled (sr_)
  cudaEvent_t ev_fd0_ = nullptr;           // this turn's fc0 dgrad partial written (st_)
  cudaEvent_t ev_ret_[2] = {nullptr, nullptr};     // slot's gradient return done (sr_)
  cudaEvent_t ev_sr_ = nullptr;            // all of the step's sr_ work done
  void wait_step();  // synchronise st_, polling the transports for asynchronous errors
  void check_device_targets(const float* const* targets);
  bool nccl_ = false;
  bool targets_checked_ = false;  // this step's targets were validated on the host already
  cudaStream_t st_ = nullptr;
  cudaStream_t sc_ = nullptr;  // side stream: per-layer conv-gradient all-reduce
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  std::vector<cudaEvent_t> ev_layer_;  // per conv layer: its gradients are final on st_
  cudaEvent_t ev_comm_ = nullptr;      // all conv-gradient all-reduces done on sc_
  cudaEvent_t ev0_fc_ = nullptr;       // DP: FC gradients final on st_
  cudaStream_t sx_ = nullptr;          // copy stream: prefetch H2D
  struct PrefSlot {
    std::vector<const float*> x, t;  // host pointers staged in this slot
    bool valid = false;
    int64_t bytes = 0;
    cudaEvent_t ready = nullptr;  // copies done (sx_)
    cudaEvent_t used = nullptr;   // the step that consumed the slot is done reading it (st_)
  };
  PrefSlot pref_[2];
  int next_slot_ = 0;
  DevArena arena_;
  std::vector<Worker<TA>> w_;
  std::vector<long long> coff_, foff_;
  long long conv_total_ = 0, fc_total_ = 0;
  float* ws_ = nullptr;  // split-K workspace of the compute-stream GEMMs
  size_t ws_floats_ = 0;
  float* ws2_ = nullptr;  // split-K workspace of the conv wgrad GEMMs (side stream sw_)
  size_t ws2_floats_ = 0;
  cudaStream_t sw_ = nullptr;          // side stream: conv weight gradients (off the dgrad chain)
  cudaStream_t sb_ = nullptr;          // side stream: conv bias gradients (off both chains)
  std::vector<cudaEvent_t> ev_bg_;     // per conv layer: its bias gradient final on sb_
  cudaStream_t sf_ = nullptr;          // side stream: FC weight gradients + fused update (off the backward chain)
  cudaEvent_t ev_fcd_ = nullptr;       // FC dgrad of the current layer done (st_)
  cudaEvent_t ev_fcw_ = nullptr;       // all FC wgrads of the turn done (sf_)
  cudaEvent_t ev_rot0_ = nullptr;      // conv forward enqueued on st_ (forks the dgrad-operand rotation)
  cudaEvent_t ev_rot_ = nullptr;       // dgrad operands of this step's weights rotated
  float* ws3_ = nullptr;               // split-K workspace of the FC wgrad GEMMs (sf_)
  size_t ws3_floats_ = 0;
  std::vector<cudaEvent_t> ev_dz_;     // per conv layer: dz final on st_
  std::vector<cudaEvent_t> ev_wg_;     // per conv layer: its weight + bias gradients final on sw_
  int xblocks_ = 0;
  int64_t launches_ = 0;
  struct ProfSlot {
    cudaEvent_t a, b;
    const char* tag;
    int layer;
    double flops;
  };
  std::vector<ProfSlot> prof_pool_;
  size_t prof_used_ = 0;
  double gemm_flops_ = 0.0;
  // fused FC-weight SGD state for the turn being enqueued
  bool fuse_sgd_ = false, weights_fused_ = false, sgd_has_gscale_ = false;
  hp_hyper sgd_hp_{};
  double sgd_lr_ = 0.0;
  float sgd_gscale_ = 1.f;
};

template <class TA>
ClusterImpl<TA>::ClusterImpl(const hp_model_spec* spec, const hp_cluster_config* cfg) {
  // ClusterConfig::validate (cluster.cpp:50-67)
  if (cfg->workers < 1) config_error("cluster.workers: must be >= 1");
  if (cfg->per_worker_batch < 1) config_error("cluster.per_worker_batch: must be >= 1");
  if (cfg->scheme < 0 || cfg->scheme > 3) config_error("cluster.scheme: expected A|B|C (or DP)");
  if (cfg->scheme == HP_SCHEME_C && cfg->per_worker_batch % cfg->workers != 0)
    config_error("cluster.per_worker_batch: scheme C scatters b/K examples per worker per turn; " +
                 num(cfg->per_worker_batch) + " is not divisible by " + num(cfg->workers));
  if (cfg->variable_batch && cfg->scheme == HP_SCHEME_DP)
    config_error("cluster.variable_batch: pure data parallelism has a single fc pass per step");
  if (cfg->variable_batch && cfg->scheme == HP_SCHEME_A)
    config_error("cluster.variable_batch: scheme A has a single fc pass per step; per-sub-batch "
                 "updates require scheme B or C");
  if (cfg->precision != HP_PRECISION_SINGLE)
    config_error("cluster.precision: the B200 path stores fp32 parameters (single); double is "
                 "served by the CPU oracle only");
  K_ = cfg->workers;
  b_ = cfg->per_worker_batch;
  scheme_ = cfg->scheme;
  variable_ = cfg->variable_batch != 0;
  math_ = cfg->math_mode;
  seed_ = cfg->seed;
  dp_ = scheme_ == HP_SCHEME_DP;
  fcK_ = dp_ ? 1 : K_;
  g_ = make_geometry(spec, fcK_, b_);
  L_ = static_cast<int>(g_.num_classes);
  num_sub_ = (scheme_ == HP_SCHEME_A || scheme_ == HP_SCHEME_DP) ? 1 : K_;
  n_ = scheme_ == HP_SCHEME_A ? K_ * b_ : b_;
  ldn_ = round_up(n_, 8);

  if (cfg->device >= 0) HP_CUDA(cudaSetDevice(cfg->device));
  if (cfg->transport == HP_TRANSPORT_NCCL) {
    if (cfg->rank < 0 || cfg->rank >= K_) usage_error("cluster.rank: out of range");
    comm_ = make_nccl_comm(K_, cfg->rank, cfg->nccl_id);
    nccl_ = true;
  } else {
    comm_ = make_logical_comm(K_);
  }
  comm_x_ = comm_->split();
  comm_s_ = comm_->split();
  HP_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  HP_CUDA(cudaStreamCreateWithFlags(&sr_, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&ev_conv_, &ev_xready_[0], &ev_xready_[1], &ev_fd0_, &ev_ret_[0], &ev_ret_[1], &ev_sr_})
    HP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  HP_CUDA(cudaStreamCreateWithFlags(&sc_, cudaStreamNonBlocking));
  HP_CUDA(cudaEventCreate(&ev0_));
  HP_CUDA(cudaEventCreate(&ev1_));
  HP_CUDA(cudaEventCreateWithFlags(&ev_comm_, cudaEventDisableTiming));
  HP_CUDA(cudaEventCreateWithFlags(&ev0_fc_, cudaEventDisableTiming));
  HP_CUDA(cudaStreamCreateWithFlags(&sx_, cudaStreamNonBlocking));
  HP_CUDA(cudaStreamCreateWithFlags(&sw_, cudaStreamNonBlocking));
  HP_CUDA(cudaStreamCreateWithFlags(&sb_, cudaStreamNonBlocking));
  HP_CUDA(cudaStreamCreateWithFlags(&sf_, cudaStreamNonBlocking));
  HP_CUDA(cudaEventCreateWithFlags(&ev_fcd_, cudaEventDisableTiming));
  HP_CUDA(cudaEventCreateWithFlags(&ev_fcw_, cudaEventDisableTiming));
  HP_CUDA(cudaEventCreateWithFlags(&ev_rot0_, cudaEventDisableTiming));
  HP_CUDA(cudaEventCreateWithFlags(&ev_rot_, cudaEventDisableTiming));
  for (auto& ps : pref_) {
    HP_CUDA(cudaEventCreateWithFlags(&ps.ready, cudaEventDisableTiming));
    HP_CUDA(cudaEventCreateWithFlags(&ps.used, cudaEventDisableTiming));
  }

  // parameter arena layouts (16-byte aligned pieces)
  for (size_t l = 0; l < g_.cg.size(); ++l) {
    coff_.push_back(conv_total_);
    conv_total_ += round_up(static_cast<long long>(g_.cg[l].F) * g_.cg[l].ldk + g_.cg[l].F, 8);
  }
  for (size_t l = 0; l < g_.fg.size(); ++l) {
    foff_.push_back(fc_total_);
    fc_total_ += round_up(g_.fg[l].cmax * g_.fg[l].Ip + g_.fg[l].cmax, 8);
  }

  const int nl = comm_->nlocal();
  w_.resize(nl);
  // implicit GEMM needs 128-byte channel blocks (TMA im2col atoms)
  const int atom = std::is_same<TA, float>::value ? 32 : 64;
  for (size_t l = 0; l < g_.cg.size(); ++l) {
    ConvGeom& c = g_.cg[l];
    c.impl_fwd = c.C % atom == 0;
    // strided first layer with few channels (AlexNet conv1: C=3, s=4 -> 48 of 64
    // channels, 3x3 taps): space-to-depth + implicit GEMM instead of an im2col buffer
    const int cz = static_cast<int>(round_up(static_cast<long long>(c.C) * c.stride * c.stride, atom));
    c.s2d = l == 0 && !c.impl_fwd && c.stride >= 2 && cz <= 2 * atom;
    if (c.s2d) {
      c.Cz = cz;
      c.Rq = (c.R + c.stride - 1) / c.stride;
      static const bool no_pairs = getenv("HP_DEV_NO_PAIRS") != nullptr;  // dev: the N = F s2d GEMMs
      // (the pool -- the only consumer -- reads the stored width; LRN-only / no-pool
      // layers keep the plain layout)
      c.pairs = !std::is_same<TA, float>::value && 2 * c.F <= 256 && (2 * c.F) % 64 == 0 && c.pk > 0 && !no_pairs;
      c.Zh = c.OH + c.Rq - 1;
      c.Zw = c.OW + c.Rq - 1;
      if (c.pairs) {  // pair u reads z columns 2u .. 2u + Rq; even width (whole pair pixels)
        c.Zw = (c.OW + 1) / 2 * 2 + c.Rq - 1;
        c.Zw += c.Zw & 1;
      }
      c.OWs = c.pairs ? c.Zw : c.OW;
      c.OHs = c.pairs ? c.Zh : c.OH;
    }
    c.impl_dgrad = l > 0 && c.stride == 1 && c.F % atom == 0 && c.pad <= c.R - 1 &&
                   c.H == c.OH + c.R - 1 - 2 * c.pad && c.W == c.OW + c.S - 1 - 2 * c.pad;
  }
  {
    // q-layout per layer (stride-1 same convs whose producers/consumers support it)
    const int n = static_cast<int>(g_.cg.size());
    for (int l = 1; l < n; ++l) {
      ConvGeom& c = g_.cg[l];
      const ConvGeom& pc = g_.cg[l - 1];
      c.in_q = c.impl_fwd && c.impl_dgrad && c.stride == 1 && 2 * c.pad == c.R - 1 && c.R == c.S &&
               c.OH == c.H && c.OW == c.W && !(pc.lrn_n > 0 && pc.pk == 0);
      // dz without pool/LRN above: written by mask_cast (last layer, unsupported)
      if (c.pk == 0 && c.lrn_n == 0 && l == n - 1) c.in_q = false;
    }
    // a layer without pool/LRN shares one layout between its output (= next
    // input, the ReLU mask of its dz) and its dz: both q with equal pads or neither
    for (bool changed = true; changed;) {
      changed = false;
      for (int l = 1; l + 1 < n; ++l) {
        ConvGeom& c = g_.cg[l];
        ConvGeom& nx = g_.cg[l + 1];
        if (c.pk == 0 && c.lrn_n == 0 && (c.in_q != nx.in_q || (c.in_q && c.pad != nx.pad))) {
          if (c.in_q || nx.in_q) changed = true;
          c.in_q = nx.in_q = false;
        }
      }
    }
    for (auto& c : g_.cg) {
      c.Hq = c.in_q ? c.H + c.pad : c.H;
      c.Wq = c.in_q ? c.W + c.pad : c.W;
      c.Pq = c.in_q ? b_ * c.Hq * c.Wq : b_ * c.OHs * c.OWs;
    }
  }
  const auto& in = g_.input;
  const long long A = g_.A;
  const int nc = static_cast<int>(g_.cg.size()), nf = static_cast<int>(g_.fg.size());
  xblocks_ = 0;
  for (int l = 0; l < nf; ++l) (void)l;
  xblocks_ = xent_blocks(static_cast<int>(g_.fg.back().cmax), static_cast<int>(n_));
  size_t colsum_ws = 0;
  for (const auto& cg : g_.cg) colsum_ws = std::max(colsum_ws, colsum_ws_floats(cg.Pq, cg.F));
  size_t comm_scratch = 0;
  for (int i = 0; i < nl; ++i) {
    Worker<TA>& w = w_[i];
    w.gid = comm_->first() + i;
    w.x_nchw = arena_.make<float>(b_ * in[0] * in[1] * in[2]);
    for (int k = 0; k < 2; ++k) {
      w.xin[k] = arena_.make<float>(b_ * in[0] * in[1] * in[2]);
      w.tin[k] = arena_.make<float>(b_ * L_);
    }
    w.x0 = g_.cg[0].impl_fwd ? arena_.make<TA>(b_ * in[0] * in[1] * in[2]) : nullptr;
    w.targets = arena_.make<float>(b_ * L_);
    for (int l = 0; l < nc; ++l) {
      const ConvGeom& c = g_.cg[l];
      const bool lrn_only = c.lrn_n > 0 && c.pk == 0;  // fused LRN+pool keeps no LRN output
      // layer 0 explicit: transposed colT [Kc][P]; other explicit layers: col [P][ldk]
      if (c.s2d) {
        const long long kz = static_cast<long long>(c.pairs ? 2 : 1) * c.F * c.Rq * (c.Rq + (c.pairs ? 1 : 0)) * c.Cz;
        w.z = arena_.make<TA>(b_ * c.Zh * c.Zw * c.Cz);
        w.wz = arena_.make<TA>(kz);
        w.dwz = arena_.make<float>(kz);
        w.bias2 = c.pairs ? arena_.make<float>(2LL * c.F) : nullptr;
      }
      w.col.push_back(c.impl_fwd || c.s2d ? nullptr
                                 : (l == 0 ? arena_.make<TA>(static_cast<long long>(c.Kc) * c.ldp)
                                           : arena_.make<TA>(c.P * c.ldk)));
      const bool next_q = l + 1 < nc && g_.cg[l + 1].in_q;
      const long long out_rows = next_q ? g_.cg[l + 1].Pq : -1;  // stage output in the next layer's q-layout
      w.act.push_back(arena_.make<TA>((c.pk == 0 && c.lrn_n == 0 && next_q ? out_rows : c.pairs ? c.Pq : c.P) * c.F));
      w.lrn.push_back(lrn_only ? arena_.make<TA>(c.P * c.F) : nullptr);
      w.lrn_d.push_back(lrn_only ? arena_.make<float>(c.P * c.F) : nullptr);
      w.pool.push_back(c.pk > 0 ? arena_.make<TA>((next_q ? out_rows : c.PP) * c.F) : nullptr);
      w.widx.push_back(c.pk > 0 ? arena_.make<uint8_t>(c.PP * c.F) : nullptr);
      w.dz.push_back(arena_.make<TA>(c.Pq * c.F));
      w.dcol.push_back(l > 0 && !c.impl_dgrad ? arena_.make<float>(c.P * c.ldk) : nullptr);
      w.wrot.push_back(c.impl_dgrad ? arena_.make<TA>(static_cast<long long>(c.F) * c.Kc) : nullptr);
      // grad wrt this stage's output, needed when the stage ends in pool/LRN
      const bool needs_g = (c.pk > 0 || c.lrn_n > 0) && l + 1 < nc;
      w.gstage.push_back(needs_g ? arena_.make<float>(c.PP * c.F) : nullptr);
    }
    w.cp = arena_.make<float>(conv_total_);
    w.cm = arena_.make<float>(conv_total_);
    w.cgr = arena_.make<float>(conv_total_);
    w.cgr_local = K_ > 1 ? arena_.make<float>(conv_total_) : nullptr;
    w.cpt = std::is_same<TA, float>::value ? nullptr : arena_.make<TA>(conv_total_);
    for (int s = 0; s < 2; ++s) {
      w.xb[s] = arena_.make<TA>(n_ * A);
      w.tb[s] = arena_.make<float>(n_ * L_);
      w.fd0[s] = fcK_ > 1 ? arena_.make<float>(n_ * A) : nullptr;
    }
    w.fx.assign(nf, nullptr);
    for (int l = 1; l < nf; ++l) w.fx[l] = arena_.make<TA>(g_.fg[l].Ip * ldn_);
    w.logits = arena_.make<float>(g_.fg.back().cmax * ldn_);
    for (int l = 0; l < nf; ++l) {
      w.fdz.push_back(arena_.make<TA>(g_.fg[l].cmax * ldn_));
      w.fdpart.push_back(l > 0 ? arena_.make<float>(g_.fg[l].Ip * ldn_) : w.fd0[0]);
      if (l > 0) comm_scratch = std::max(comm_scratch, static_cast<size_t>(g_.fg[l - 1].cmax * ldn_));
    }
    comm_scratch = std::max(comm_scratch, static_cast<size_t>(b_ * A));
    w.gflat = arena_.make<float>(b_ * A);
    w.fp = arena_.make<float>(fc_total_);
    w.fm = arena_.make<float>(fc_total_);
    w.fgr = arena_.make<float>(fc_total_);
    w.fpt = std::is_same<TA, float>::value ? nullptr : arena_.make<TA>(fc_total_);
    w.loss_parts = arena_.make<double>(static_cast<long long>(num_sub_) * xblocks_);
    w.bad = arena_.make<int>(1);
    w.colsum_ws = arena_.make<float>(static_cast<long long>(colsum_ws));
  }
  comm_->reserve(comm_scratch * sizeof(float));
  comm_x_->reserve(static_cast<size_t>(b_ * A) * sizeof(float));
  ev_layer_.resize(g_.cg.size());
  for (auto& e : ev_layer_) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  ev_dz_.resize(g_.cg.size());
  ev_wg_.resize(g_.cg.size());
  for (auto& e : ev_dz_) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : ev_wg_) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  ev_bg_.resize(g_.cg.size());
  for (auto& e : ev_bg_) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  HP_CUDA(cudaMallocHost(&host_parts_, sizeof(double) * nl * num_sub_ * xblocks_));
  HP_CUDA(cudaMallocHost(&host_bad_, sizeof(int) * nl));
  {
    const ConvGeom& lc = g_.cg.back();
    // Opt-in (HP_SLICE_LAST_CONV=1, read per cluster): measured a net loss on
    // B200 at b = 128 -- K small slices of the last conv cost a wave each
    // (8 workers, logical transport: 17.5 -> 18.2 ms per step) while the
    // exchange they would hide is a few MB over NVLink 5.
    const char* sl = getenv("HP_SLICE_LAST_CONV");
    slice_last_ = sl && atoi(sl) != 0 && scheme_ == HP_SCHEME_C && !dp_ && K_ > 1 && b_ % K_ == 0 &&
                  num_sub_ == K_ && g_.cg.size() > 1 && lc.in_q && lc.lrn_n == 0;
    ev_slice_.resize(slice_last_ ? static_cast<size_t>(K_) : 0);
    for (auto& e : ev_slice_) HP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // Plans first with a null workspace to size it (for both conv kernel
  // families, so rebuild_plans can switch), then for real.
  const bool shift = use_shift;
  for (bool sh : {false, true}) {
    use_shift = sh;
    for (auto& w : w_) build_plans(w);
  }
  use_shift = shift;
  ws_ = ws_floats_ > 0 ? arena_.make<float>(static_cast<long long>(ws_floats_)) : nullptr;
  ws2_ = ws2_floats_ > 0 ? arena_.make<float>(static_cast<long long>(ws2_floats_)) : nullptr;
  ws3_ = ws3_floats_ > 0 ? arena_.make<float>(static_cast<long long>(ws3_floats_)) : nullptr;
  for (auto& w : w_) build_plans(w);
  if (const char* tl = getenv("HP_DEV_TIMELINE")) {
    tl_cap_ = 4096;
    HP_CUDA(cudaMalloc(&tl_, (1 + 2 * static_cast<size_t>(tl_cap_)) * sizeof(unsigned long long)));
    HP_CUDA(cudaMemset(tl_, 0, sizeof(unsigned long long)));
    tl_file_ = fopen(tl, "w");
    if (!tl_file_) usage_error(std::string("HP_DEV_TIMELINE: cannot open ") + tl);
    fprintf(tl_file_, "step,name,kind,ns\n");
  }
  init_params();
  sent.assign(K_, {0, 0, 0, 0});
  received.assign(K_, {0, 0, 0, 0});
  HP_CUDA(cudaStreamSynchronize(st_));
}

template <class TA>
ClusterImpl<TA>::~ClusterImpl() {
  if (st_) cudaStreamSynchronize(st_);
  for (auto& kv : graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  if (host_parts_) cudaFreeHost(host_parts_);
  if (host_bad_) cudaFreeHost(host_bad_);
  if (tl_) cudaFree(tl_);
  if (tl_file_) fclose(tl_file_);
  if (sr_) cudaStreamSynchronize(sr_);
  if (sc_) cudaStreamSynchronize(sc_);
  comm_s_.reset();
  comm_x_.reset();
  comm_.reset();
  for (cudaEvent_t e : {ev_conv_, ev_xready_[0], ev_xready_[1], ev_fd0_, ev_ret_[0], ev_ret_[1], ev_sr_})
    if (e) cudaEventDestroy(e);
  if (sr_) cudaStreamDestroy(sr_);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  for (auto e : ev_layer_) cudaEventDestroy(e);
  for (auto e : ev_dz_) cudaEventDestroy(e);
  for (auto e : ev_wg_) cudaEventDestroy(e);
  for (auto e : ev_bg_) cudaEventDestroy(e);
  for (auto e : ev_slice_) cudaEventDestroy(e);
  if (sw_) {
    cudaStreamSynchronize(sw_);
    cudaStreamDestroy(sw_);
  }
  if (sb_) {
    cudaStreamSynchronize(sb_);
    cudaStreamDestroy(sb_);
  }
  if (sf_) {
    cudaStreamSynchronize(sf_);
    cudaStreamDestroy(sf_);
  }
  if (ev_fcd_) cudaEventDestroy(ev_fcd_);
  if (ev_fcw_) cudaEventDestroy(ev_fcw_);
  if (ev_rot0_) cudaEventDestroy(ev_rot0_);
  if (ev_rot_) cudaEventDestroy(ev_rot_);
  if (ev_comm_) cudaEventDestroy(ev_comm_);
  if (ev0_fc_) cudaEventDestroy(ev0_fc_);
  if (sc_) cudaStreamDestroy(sc_);
  if (sx_) cudaStreamSynchronize(sx_);
  for (auto& ps : pref_) {
    if (ps.ready) cudaEventDestroy(ps.ready);
    if (ps.used) cudaEventDestroy(ps.used);
  }
  if (sx_) cudaStreamDestroy(sx_);
  for (auto& s : prof_pool_) {
    cudaEventDestroy(s.a);
    cudaEventDestroy(s.b);
  }
  if (st_) cudaStreamDestroy(st_);
}

template <class TA>
Worker<TA>& ClusterImpl<TA>::local(int gid) {
  for (auto& w : w_)
    if (w.gid == gid) return w;
  usage_error("worker " + num(gid) + " is not local to this process (NCCL transport)");
}

template <class TA>
const Worker<TA>* ClusterImpl<TA>::local_or_null(int gid) const {
  for (const auto& w : w_)
    if (w.gid == gid) return &w;
  return nullptr;
}

template <class TA>
static const TA* stage_out_of(const Worker<TA>& w, const ConvGeom& c, int l) {
  if (c.pk > 0) return w.pool[l];
  if (c.lrn_n > 0) return w.lrn[l];
  return w.act[l];
}

template <class TA>
const TA* ClusterImpl<TA>::stage_in(const Worker<TA>& w, int l) const {
  return stage_out_of(w, g_.cg[l - 1], l - 1);
}

template <class TA>
void ClusterImpl<TA>::build_plans(Worker<TA>& w) {
  const int nc = static_cast<int>(g_.cg.size()), nf = static_cast<int>(g_.fg.size());
  const bool bf = !std::is_same<TA, float>::value;
  auto op = [](const void* p, int mn, long long ld) {
    GemmOperand o;
    o.ptr = p;
    o.mn_major = mn;
    o.ld = ld;
    return o;
  };
  auto plan = [&](const GemmOperand& a, const GemmOperand& b, long long M, long long N, long long K,
                  const Epi& e, int side = 0, int bn = 0, int cta2 = -1, const TapPairs* tp = nullptr) {
    // The plan picks its own tile and split-K; the first (sizing) pass runs
    // against a placeholder workspace and records the largest need. Side-stream
    // (wgrad) plans get their own workspace: they run concurrently with the
    // compute stream's GEMMs.
    float* real = side == 1 ? ws2_ : side == 2 ? ws3_ : ws_;
    size_t& need = side == 1 ? ws2_floats_ : side == 2 ? ws3_floats_ : ws_floats_;
    float* ws = real != nullptr ? real : reinterpret_cast<float*>(256);
    GemmPlan pl = gemm_plan(math_, a, b, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), e, 0,
                            ws, bn, cta2, tp);
    if (pl.args.raw_partial) need = std::max(need, static_cast<size_t>(pl.splits * M * N));
    else pl.args.ws = real;
    return pl;
  };
  w.conv_fwd.clear();
  w.last_fwd_slices.clear();
  w.conv_wgrad.clear();
  w.conv_dgrad.clear();
  w.fc_fwd.clear();
  w.fc_wgrad.clear();
  w.fc_dgrad.clear();
  const void* cweights = bf ? static_cast<const void*>(w.cpt) : static_cast<const void*>(w.cp);
  const int es = bf ? 2 : 4;
  for (int l = 0; l < nc; ++l) {
    const ConvGeom& c = g_.cg[l];
    const char* kw = static_cast<const char*>(cweights) + conv_k_off(l) * es;
    const void* in = l == 0 ? static_cast<const void*>(w.x0) : stage_in(w, l);
    Im2col view{1, static_cast<int>(b_), c.H, c.W, c.C, c.R, c.S, c.stride, c.pad, c.OH, c.OW};
    if (c.in_q) {  // x in q-layout: the padding is in memory; walk the valid outputs
      view.H = c.Hq;
      view.W = c.Wq;
      view.corners = 1;
      view.lo = 0;
      view.hi = -c.pad;
    }
    const bool next_q = l + 1 < nc && g_.cg[l + 1].in_q;
    // fprop: Y[P][F] = im2col(x)[P][Kc] . W[F][Kc]^T (+bias, ReLU)
    Epi e;
    e.c = w.act[l];
    e.ldc = c.F;
    e.c_type = kTA;
    e.bias = w.cp + conv_b_off(l);
    e.bias_mode = 2;
    e.relu = c.relu;
    if (next_q && c.pk == 0 && c.lrn_n == 0) {  // conv output = next layer's q-layout input
      const ConvGeom& nx = g_.cg[l + 1];
      e.rows = RowMap{1, c.OH, c.OW, c.OH, c.OW, nx.Hq, nx.Wq, nx.pad};
    }
    GemmOperand xa = l == 0 ? op(w.col[0], 1, c.ldp) : op(w.col[l], 0, c.ldk);
    if (c.impl_fwd) {
      xa = op(in, 0, 0);
      xa.conv = view;
    }
    // s2d: im2col over z (no pairs: fp32 / tf32 math). Pixel pairs: the pair
    // kernel [2F][Rq][Rq+1][Cz] (launch_s2d_weights), N = 2F columns
    const int sq = c.Rq + (c.pairs ? 1 : 0);
    const long long Kz = static_cast<long long>(c.Rq) * sq * c.Cz;
    const Im2col zview{1, static_cast<int>(b_), c.Zh, c.Zw, c.Cz, c.Rq, c.Rq, 1, 0, c.OH, c.OW};
    const int zn = c.pairs ? 2 * c.F : c.F;  // GEMM columns
    // bf16 stride-1 convs over zero-bordered rows: the flat-shift kernel (one
    // smem halo per channel block for all taps); output rows are the stored
    // grid, the RowMap keeps the valid ones
    // Measured on B200 (tests/dev/step_dev.py): the shift kernel wins on every
    // q-layout layer (conv2-5 fprop and dgrad).
    // (conv1's space-to-depth input -- 64 channels, 9 taps, N = 64 -- measures
    // faster on the TMA-im2col kernel: 0.092 vs 0.099 ms)
    const bool shift_fwd = bf && use_shift && !c.s2d && c.in_q && conv_shift_supported(c.C, c.R, c.S, c.Wq, c.F);
    if (shift_fwd) {
      Epi es = e;
      const int gH = c.s2d ? c.Zh : c.Hq, gW = c.s2d ? c.Zw : c.Wq;
      es.rows = e.rows.enabled ? RowMap{1, gH, gW, c.OH, c.OW, e.rows.dH, e.rows.dW, e.rows.dp}
                               : RowMap{1, gH, gW, c.OH, c.OW, c.OH, c.OW, 0};
      GemmPlan pl = c.s2d ? conv_shift_plan(w.z, b_ * gH * gW, c.Cz, c.Rq, c.Rq, gW, w.wz, Kz, c.F, es)
                          : conv_shift_plan(in, c.Pq, c.C, c.R, c.S, gW, kw, c.ldk, c.F, es);
      w.conv_fwd.push_back(pl);
      if (slice_last_ && l == nc - 1 && !c.s2d && !e.rows.enabled) {
        // scheme C micro-pipelining: the same conv on each turn's image slice
        // (q-layout images are Hq*Wq rows apart; rows outside the slice read as
        // the zero border, exactly as inside the whole batch)
        const long long bs = b_ / K_;
        for (int j = 0; j < K_; ++j) {
          Epi ej = es;
          ej.c = w.act[l] + j * bs * c.OHs * c.OWs * c.F;
          w.last_fwd_slices.push_back(conv_shift_plan(static_cast<const TA*>(in) + j * bs * c.Hq * c.Wq * c.C,
                                                      bs * c.Hq * c.Wq, c.C, c.R, c.S, gW, kw, c.ldk, c.F, ej));
        }
      }
    } else if (c.pairs) {
      if (!conv_shift_supported(2 * c.Cz, c.Rq, 2, c.Zw / 2, zn)) config_error("conv1 pixel pairs: unsupported shape");
      // pair pixels (ConvGeom::pairs): conv1 = a stride-1 Rq x 2 conv over
      // z' [b][Zh][Zw/2][2Cz] on the flat-shift kernel. The pair weights
      // [2F][Rq][Rq+1][Cz] are already the [2F][Rq][2][2Cz] kernel of that conv
      // (s' = 2 s2 + q); output rows are the stored z' grid, the RowMap keeps
      // the OH x ceil(OW/2) valid pair pixels.
      Epi es = e;
      es.ldc = zn;
      es.bias = w.bias2;
      const int pw = c.Zw / 2;
      es.rows = RowMap{1, c.Zh, pw, c.OH, (c.OW + 1) / 2, c.OHs, pw, 0};
      w.conv_fwd.push_back(conv_shift_plan(w.z, b_ * c.Zh * pw, 2 * c.Cz, c.Rq, 2, pw, w.wz, Kz, zn, es));
    } else if (c.s2d) {
      xa = op(w.z, 0, 0);
      xa.conv = zview;
      w.conv_fwd.push_back(plan(xa, op(w.wz, 0, Kz), c.P, c.F, Kz, e));
    } else {
      w.conv_fwd.push_back(plan(xa, op(kw, 0, c.ldk), c.P, c.F, c.Kc, e));
    }
    // wgrad: dW[F][Kc] = dz^T[F][P] . im2col(x)[P][Kc]
    Epi eg;
    eg.c = w.cgr + conv_k_off(l);
    eg.ldc = c.ldk;
    GemmOperand xb = l == 0 ? op(w.col[0], 0, c.ldp) : op(w.col[l], 1, c.ldk);
    if (c.impl_fwd) {
      xb = op(in, 1, 0);
      xb.conv = view;
      if (c.in_q) {  // K = every stored q position (dz is zero on the border)
        xb.conv.lo = -c.pad;
        xb.conv.hi = -c.pad;
        xb.conv.OH = c.Hq;
        xb.conv.OW = c.Wq;
        xb.conv.shift = 1;  // tiled boxes at shifted rows of the flat q-layout x
      }
    }
    // Orientation: dW[F][Kc] = dz^T . im2col(x) (M = F), or its transpose
    // dW^T[Kc][F] = im2col(x)^T . dz (M = Kc, stored transposed) when the F-side
    // 256-row CTA-pair tiles are badly filled and F makes one wide N tile.
    // Measured (tests/dev/step_dev.py, after the MMA-issue rework): conv2
    // (F=192) 0.157 -> 0.110 ms swapped; conv1 (F=64) 0.107 vs 0.118, conv3
    // 0.067 vs 0.071, conv4 (F=384) 0.114 vs 0.120 faster unswapped.
    auto mfill = [](long long m) { return static_cast<double>(m) / (((m + 255) / 256) * 256); };
    const long long Kw = c.s2d ? Kz : c.Kc;
    static const bool no_halo = getenv("HP_DEV_NO_HALO") != nullptr;  // dev: per-tap shifted B boxes
    const bool swap = (c.impl_fwd || c.s2d) && !c.pairs && c.F >= 128 && c.F <= 256 && mfill(Kw) > mfill(c.F) + 0.1;
    if (c.s2d) {
      eg.c = w.dwz;
      eg.ldc = Kz;
      xb = op(w.z, 1, 0);
      xb.conv = zview;
    }
    // tap pairs (TapPairs, gemm.cuh) for the swapped stride-1 wgrad: neighbouring
    // taps of a kernel row share one x box (d = 1); an odd row's last taps pair
    // across rows (d = wq); a leftover tap rides alone
    TapPairs tpairs;
    if (swap && c.in_q && xb.conv.shift && bf && c.C % 64 == 0 && !no_halo) {
      std::vector<std::array<int, 3>> tiles;  // {tap0, tap1 (-1: none), channel block}
      for (int cbk = 0; cbk < c.C / 64; ++cbk) {
        std::vector<int> left;
        for (int r = 0; r < c.R; ++r) {
          int sx = 0;
          for (; sx + 1 < c.S; sx += 2) tiles.push_back({r * c.S + sx, r * c.S + sx + 1, cbk});
          if (sx < c.S) left.push_back(r * c.S + sx);
        }
        for (size_t i = 0; i < left.size(); i += 2)
          tiles.push_back({left[i], i + 1 < left.size() ? left[i + 1] : -1, cbk});
      }
      if (tiles.size() <= 16) {
        auto shift_of = [&](int tap) { return (tap / c.S) * c.Wq + tap % c.S; };
        tpairs.n = static_cast<int>(tiles.size());
        eg.rblk.enabled = 1;
        for (int t = 0; t < tpairs.n; ++t) {
          const auto& tl = tiles[static_cast<size_t>(t)];
          tpairs.off[t] = shift_of(tl[0]);
          tpairs.d[t] = tl[1] >= 0 ? shift_of(tl[1]) - shift_of(tl[0]) : 1;
          tpairs.cb[t] = tl[2];
          eg.rblk.blk[2 * t] = tl[0] * c.C + tl[2] * 64;
          eg.rblk.blk[2 * t + 1] = tl[1] >= 0 ? tl[1] * c.C + tl[2] * 64 : -1;
        }
      }
    }
    if (swap && tpairs.n > 0) {
      eg.c_trans = 1;  // element (m = k, n = f) -> dW[f][k], rows through eg.rblk
      w.conv_wgrad.push_back(plan(xb, op(w.dz[l], 1, c.F), 128LL * tpairs.n, c.F, c.Pq, eg, 1, 0, 0, &tpairs));
    } else if (swap) {
      eg.c_trans = 1;  // element (m = k, n = f) -> dW[f][k]
      w.conv_wgrad.push_back(plan(xb, op(w.dz[l], 1, c.F), Kw, c.F, c.s2d ? c.P : c.Pq, eg, 1));
    } else if (c.pairs) {
      // pair pixels: the halo wgrad (Im2col::halo) of the Rq x 2 conv over z'
      // (K = every stored pair pixel; dz is zero off the valid grid). Its column
      // order maps back onto the pair kernel layout [2F][Rq][2][2Cz] = [2F][Rq][Rq+1][Cz]
      const int pw = c.Zw / 2;
      GemmOperand xz = op(w.z, 1, 0);
      xz.conv = Im2col{1, static_cast<int>(b_), c.Zh, pw, 2 * c.Cz, c.Rq, 2, 1, 0, c.Zh, pw};
      xz.conv.shift = 1;
      xz.conv.halo = 1;
      eg.cols = ColMap{1, 2, 2 * c.Cz};
      w.conv_wgrad.push_back(plan(op(w.dz[l], 1, zn), xz, zn, Kz, b_ * c.Zh * pw, eg, 1, 128, 0));
    } else if (c.s2d) {
      w.conv_wgrad.push_back(plan(op(w.dz[l], 1, c.F), xb, c.F, Kz, c.P, eg, 1));
    } else if (c.in_q && xb.conv.shift && bf && c.S * 64 <= 256 && c.C % 64 == 0 && !no_halo) {
      // halo B (Im2col::halo): N tiles of S*64 columns = the S taps of one kernel
      // row of one channel block, read as one x box per k-tile
      xb.conv.halo = 1;
      eg.cols = ColMap{1, c.S, c.C};
      w.conv_wgrad.push_back(plan(op(w.dz[l], 1, c.F), xb, c.F, c.Kc, c.Pq, eg, 1, 64 * c.S, 0));
    } else {
      w.conv_wgrad.push_back(plan(op(w.dz[l], 1, c.F), xb, c.F, c.Kc, c.Pq, eg, 1));
    }
    if (l == 0) {
      w.conv_dgrad.push_back(GemmPlan{});
      continue;
    }
    const ConvGeom& pc = g_.cg[l - 1];
    const bool below_fused = pc.pk > 0 || pc.lrn_n > 0;
    if (c.impl_dgrad) {
      // dX[b*H*W][C] = conv(dz, rotated W) with padding R-1-pad; written straight
      // into the layer below's gradient (ReLU mask fused when nothing sits between)
      Epi ed;
      if (below_fused) {
        ed.c = w.gstage[l - 1];
      } else {
        ed.c = w.dz[l - 1];
        ed.c_type = kTA;
        if (pc.relu) {
          ed.mask = w.act[l - 1];
          ed.ldmask = c.C;
          ed.mask_type = kTA;
        }
        if (pc.in_q) ed.rows = RowMap{1, c.H, c.W, c.H, c.W, pc.Hq, pc.Wq, pc.pad};  // dz (and mask) q-layout
      }
      ed.ldc = c.C;
      GemmOperand dy = op(w.dz[l], 0, 0);
      dy.conv = Im2col{1, static_cast<int>(b_), c.OH, c.OW, c.F, c.R, c.S, 1, c.R - 1 - c.pad, c.H, c.W};
      if (c.in_q) {  // dz in q-layout: same geometry as x (same conv)
        dy.conv.H = c.Hq;
        dy.conv.W = c.Wq;
        dy.conv.corners = 1;
        dy.conv.lo = 0;
        dy.conv.hi = -c.pad;
      }
      const long long kd = static_cast<long long>(c.R) * c.S * c.F;  // dgrad reduces over (r, s, f)
      if (bf && use_shift && c.in_q && conv_shift_supported(c.F, c.R, c.S, c.Wq, c.C)) {
        // dX over the stored q grid of dz: rows (b, h, w) valid for h < H, w < W
        ed.rows = ed.rows.enabled ? RowMap{1, c.Hq, c.Wq, c.H, c.W, ed.rows.dH, ed.rows.dW, ed.rows.dp}
                                  : RowMap{1, c.Hq, c.Wq, c.H, c.W, c.H, c.W, 0};
        w.conv_dgrad.push_back(conv_shift_plan(w.dz[l], c.Pq, c.F, c.R, c.S, c.Wq, w.wrot[l], kd, c.C, ed));
      } else {
        w.conv_dgrad.push_back(plan(dy, op(w.wrot[l], 0, kd), b_ * c.H * c.W, c.C, kd, ed));
      }
    } else {
      // dcol[P][Kc] = dz[P][F] . W[F][Kc], then col2im
      Epi ed;
      ed.c = w.dcol[l];
      ed.ldc = c.ldk;
      w.conv_dgrad.push_back(plan(op(w.dz[l], 0, c.F), op(kw, 1, c.ldk), c.P, c.Kc, c.F, ed));
    }
  }
  const void* fweights = bf ? static_cast<const void*>(w.fpt) : static_cast<const void*>(w.fp);
  for (int l = 0; l < nf; ++l) {
    const FcGeom& f = g_.fg[l];
    const long long rows = f.c1[sid(w.gid)] - f.c0[sid(w.gid)];
    const char* fwp = static_cast<const char*>(fweights) + fc_w_off(l) * es;
    const bool last = l + 1 == nf;
    // fwd: Z^T[rows][n] = W[rows][Ip] . X^T
    Epi e;
    if (last) {
      e.c = w.logits;
      e.c_type = kF32;
    } else {
      e.c = static_cast<TA*>(w.fx[l + 1]) + static_cast<long long>(sid(w.gid)) * f.cmax * ldn_;
      e.c_type = kTA;
    }
    e.ldc = ldn_;
    e.bias = w.fp + fc_b_off(l);
    e.bias_mode = 1;
    e.relu = f.relu;
    const GemmOperand xin = l == 0 ? op(w.xb[0], 0, g_.A) : op(w.fx[l], 1, ldn_);
    w.fc_fwd.push_back(plan(op(fwp, 0, f.Ip), xin, rows, n_, f.Ip, e));
    if (l == 0) w.fc0_slot1[0] = plan(op(fwp, 0, f.Ip), op(w.xb[1], 0, g_.A), rows, n_, f.Ip, e);
    // wgrad: dW[rows][Ip] (+)= dZ[rows][n] . X[n][Ip]
    Epi eg;
    eg.c = w.fgr + fc_w_off(l);
    eg.ldc = f.Ip;
    const GemmOperand xw = l == 0 ? op(w.xb[0], 1, g_.A) : op(w.fx[l], 0, ldn_);
    w.fc_wgrad.push_back(plan(op(w.fdz[l], 0, ldn_), xw, rows, f.Ip, n_, eg, 2));
    if (l == 0) w.fc0_slot1[1] = plan(op(w.fdz[l], 0, ldn_), op(w.xb[1], 1, g_.A), rows, f.Ip, n_, eg, 2);
    // dgrad
    if (l > 0) {
      Epi ed;
      if (fcK_ == 1) {
        ed.c = w.fdz[l - 1];
        ed.c_type = kTA;
      } else {
        ed.c = w.fdpart[l];
      }
      ed.ldc = ldn_;
      if (g_.fg[l - 1].relu) {
        ed.mask = w.fx[l];
        ed.ldmask = ldn_;
        ed.mask_type = kTA;
      }
      w.fc_dgrad.push_back(plan(op(fwp, 1, f.Ip), op(w.fdz[l], 1, ldn_), f.Ip, n_, rows, ed));
    } else {
      Epi ed;
      ed.c = fcK_ == 1 ? w.gflat : w.fd0[0];
      ed.ldc = g_.A;
      w.fc_dgrad.push_back(plan(op(w.fdz[0], 1, ldn_), op(fwp, 1, f.Ip), n_, g_.A, rows, ed));
      ed.c = fcK_ == 1 ? w.gflat : w.fd0[1];
      w.fc0_slot1[2] = plan(op(w.fdz[0], 1, ldn_), op(fwp, 1, f.Ip), n_, g_.A, rows, ed);
    }
  }
  static const bool dump = getenv("HP_DEV_PLANS") != nullptr;  // dev: print every plan's shape and tiling
  if (dump && w.gid == 0) {
    auto show = [](const char* tag, size_t l, const GemmPlan& p) {
      if (!p.valid) return;
      fprintf(stderr, "plan %-10s %zu  M %6d N %6d K %7d  %s bn %3d splits %2d grid %3u%s%s a_mn %d b_mn %d\n", tag, l,
              p.args.M, p.args.N, p.args.K, p.shift ? "shift" : p.cta2 ? "pair " : "1cta ", p.bn, p.splits, p.grid.x,
              p.light ? " light" : "", p.args.epi.c_trans ? " c_trans" : "", p.args.a_mn, p.args.b_mn);
    };
    for (size_t l = 0; l < w.conv_fwd.size(); ++l) show("conv_fwd", l, w.conv_fwd[l]);
    for (size_t l = 0; l < w.conv_wgrad.size(); ++l) show("conv_wgrad", l, w.conv_wgrad[l]);
    for (size_t l = 0; l < w.conv_dgrad.size(); ++l) show("conv_dgrad", l, w.conv_dgrad[l]);
    for (size_t l = 0; l < w.fc_fwd.size(); ++l) show("fc_fwd", l, w.fc_fwd[l]);
    for (size_t l = 0; l < w.fc_wgrad.size(); ++l) show("fc_wgrad", l, w.fc_wgrad[l]);
    for (size_t l = 0; l < w.fc_dgrad.size(); ++l) show("fc_dgrad", l, w.fc_dgrad[l]);
  }
}

// Every tcgen05 GEMM of the step goes through here: launch, count, and (when
// profiling) bracket with CUDA events on the launching stream.
template <class TA>
void ClusterImpl<TA>::gemm(const GemmPlan& p, const char* tag, int layer, cudaStream_t stream) {
  cudaStream_t st = stream ? stream : st_;
  const double flops = 2.0 * p.args.M * static_cast<double>(p.args.N) * p.args.K;
  if (profile) {
    if (prof_used_ == prof_pool_.size()) {
      ProfSlot s{};
      HP_CUDA(cudaEventCreate(&s.a));
      HP_CUDA(cudaEventCreate(&s.b));
      prof_pool_.push_back(s);
    }
    ProfSlot& s = prof_pool_[prof_used_++];
    s.tag = tag;
    s.layer = layer;
    s.flops = flops;
    HP_CUDA(cudaEventRecord(s.a, st));
    gemm_launch(p, st);
    HP_CUDA(cudaEventRecord(s.b, st));
  } else {
    tl_mark(tag, layer, false, st);
    gemm_launch(p, st);
    tl_mark(tag, layer, true, st);
  }
  launches_ += p.args.raw_partial ? 2 : 1;
  gemm_flops_ += flops;
}

template <class TA>
void ClusterImpl<TA>::collect_profile() {
  prof.clear();
  prof_gemm_ms = 0.0;
  for (size_t i = 0; i < prof_used_; ++i) {
    float ms = 0.f;
    HP_CUDA(cudaEventElapsedTime(&ms, prof_pool_[i].a, prof_pool_[i].b));
    prof.push_back({prof_pool_[i].tag, prof_pool_[i].layer, prof_pool_[i].flops, ms});
    prof_gemm_ms += ms;
  }
  prof_used_ = 0;
}

template <class TA>
long long ClusterImpl<TA>::fc_col(int l, long long i) const {
  if (l == 0) {
    // reference flatten C x H x W (model.hpp:40-43) -> device H x W x C
    const ConvGeom& c = g_.cg.back();
    const long long hw = static_cast<long long>(c.PH) * c.PW;
    const long long ch = i / hw, p = i % hw;
    return p * c.F + ch;
  }
  const FcGeom& prev = g_.fg[l - 1];
  for (int q = 0; q < fcK_; ++q)
    if (i >= prev.c0[q] && i < prev.c1[q]) return q * prev.cmax + (i - prev.c0[q]);
  return -1;
}

// init_model (model.cpp:133-162): one GaussianSampler stream on the host;
// conv kernels in layer order, then fc weights; biases zero; 0.01 * N(0,1)
// rounded to float. Each worker uploads its replica / shard.
template <class TA>
void ClusterImpl<TA>::init_params() {
  GaussianSampler gs(seed_);
  std::vector<float> conv(conv_total_, 0.f);
  for (size_t l = 0; l < g_.cg.size(); ++l) {
    const ConvGeom& c = g_.cg[l];
    float* k = conv.data() + conv_k_off(static_cast<int>(l));
    for (int f = 0; f < c.F; ++f)
      for (int ch = 0; ch < c.C; ++ch)
        for (int r = 0; r < c.R; ++r)
          for (int s = 0; s < c.S; ++s)
            k[f * c.ldk + (r * c.S + s) * c.C + ch] = static_cast<float>(0.01 * gs.next());
  }
  for (auto& w : w_) upload_master(w, true, conv);
  // fc: draw the full [in][out] matrices in row-major order, keep this
  // process's shards.
  std::vector<std::vector<float>> fcs(w_.size(), std::vector<float>(fc_total_, 0.f));
  for (size_t l = 0; l < g_.fg.size(); ++l) {
    const FcGeom& f = g_.fg[l];
    std::vector<long long> col(f.in);
    for (long long i = 0; i < f.in; ++i) col[i] = fc_col(static_cast<int>(l), i);
    for (long long i = 0; i < f.in; ++i)
      for (long long o = 0; o < f.out; ++o) {
        const float v = static_cast<float>(0.01 * gs.next());
        for (size_t wi = 0; wi < w_.size(); ++wi) {
          const int gid = sid(w_[wi].gid);
          if (o >= f.c0[gid] && o < f.c1[gid])
            fcs[wi][fc_w_off(static_cast<int>(l)) + (o - f.c0[gid]) * f.Ip + col[i]] = v;
        }
      }
  }
  for (size_t wi = 0; wi < w_.size(); ++wi) upload_master(w_[wi], false, fcs[wi]);
}

template <class TA>
void ClusterImpl<TA>::upload_master(Worker<TA>& w, bool conv, const std::vector<float>& host) {
  float* dst = conv ? w.cp : w.fp;
  HP_CUDA(cudaMemcpyAsync(dst, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice, st_));
  refresh_copies(w);
  HP_CUDA(cudaStreamSynchronize(st_));
}

template <class TA>
void ClusterImpl<TA>::refresh_copies(Worker<TA>& w) {
  rotate_all(w);
  if (std::is_same<TA, float>::value) return;
  launch_cast<TA>(w.cp, w.cpt, conv_total_, st_);
  launch_cast<TA>(w.fp, w.fpt, fc_total_, st_);
}

// ------------------------------------------------------------------ forward
template <class TA>
void ClusterImpl<TA>::conv_forward(Worker<TA>& w, int layers) {
  const int nc = static_cast<int>(g_.cg.size());
  const int B = static_cast<int>(b_);
  for (int l = 0; l < layers; ++l) {
    const ConvGeom& c = g_.cg[l];
    if (c.s2d) {
      tl_mark("s2d_input", l, false, st_);
      launch_s2d_input<TA>(w.x_src, w.z, B, c.C, c.H, c.W, c.stride, c.pad, c.Zh, c.Zw, c.Cz, st_);
      tl_mark("s2d_input", l, true, st_);
      ++launches_;
    } else if (!c.impl_fwd) {
      if (l == 0) {
        launch_im2col_t_nchw<TA>(w.x_src, w.col[0], B, c.C, c.H, c.W, c.R, c.S, c.stride, c.pad, c.OH,
                                 c.OW, c.ldp, st_);
      } else {
        launch_im2col<TA>(stage_in(w, l), w.col[l], B, c.H, c.W, c.C, c.R, c.S, c.stride, c.pad,
                          c.OH, c.OW, c.ldk, st_);
      }
      ++launches_;
    }
    gemm(w.conv_fwd[l], "conv_fwd", l);
    OutLayout yl{};  // stage output in the next layer's q-layout
    if (l + 1 < nc && g_.cg[l + 1].in_q) yl = OutLayout{g_.cg[l + 1].Hq, g_.cg[l + 1].Wq, g_.cg[l + 1].pad};
    if (c.lrn_n > 0 && c.pk > 0) {
      tl_mark("lrn_pool_fwd", l, false, st_);
      launch_lrn_pool_fwd<TA>(w.act[l], w.pool[l], w.widx[l], B, c.OHs, c.OWs, c.F, c.lrn_n, c.lrn_alpha,
                              c.lrn_beta, c.lrn_k, c.pk, c.ps, c.PH, c.PW, st_, yl);
      tl_mark("lrn_pool_fwd", l, true, st_);
      ++launches_;
    } else if (c.lrn_n > 0) {
      launch_lrn_fwd<TA>(w.act[l], w.lrn[l], w.lrn_d[l], c.P, c.F, c.lrn_n, c.lrn_alpha, c.lrn_beta,
                         c.lrn_k, st_);
      ++launches_;
    } else if (c.pk > 0) {
      launch_maxpool_fwd_w<TA>(w.act[l], w.pool[l], w.widx[l], B, c.OHs, c.OWs, c.F, c.pk, c.ps, c.PH,
                               c.PW, st_, yl);
      ++launches_;
    }
  }
}

// Slice j of the last conv layer: images [j*b/K, (j+1)*b/K) through the
// layer's flat-shift GEMM (plan built on the slice's rows) and its pool.
template <class TA>
void ClusterImpl<TA>::conv_forward_last_slice(Worker<TA>& w, int j) {
  const int l = static_cast<int>(g_.cg.size()) - 1;
  const ConvGeom& c = g_.cg[l];
  const long long bs = b_ / K_;
  gemm(w.last_fwd_slices[static_cast<size_t>(j)], "conv_fwd", l);
  const long long ao = j * bs * c.OHs * c.OWs * c.F, po = j * bs * c.PH * c.PW * c.F;
  if (c.pk > 0) {
    launch_maxpool_fwd_w<TA>(w.act[l] + ao, w.pool[l] + po, w.widx[l] + po, static_cast<int>(bs), c.OHs, c.OWs, c.F,
                             c.pk, c.ps, c.PH, c.PW, st_, OutLayout{});
    ++launches_;
  }
}

template <class TA>
void ClusterImpl<TA>::rotate_all(Worker<TA>& w, int what, cudaStream_t s) {
  if (s == nullptr) s = st_;
  for (size_t l = 0; l < g_.cg.size() && (what & 1); ++l) {
    const ConvGeom& c = g_.cg[l];
    if (c.s2d) {  // the s2d operand copy of the (just updated) master kernels
      launch_s2d_weights<TA>(w.cp + conv_k_off(static_cast<int>(l)), c.ldk, w.wz, c.F, c.C, c.R, c.S, c.stride, c.Rq,
                             c.Cz, s, c.pairs ? w.cp + conv_b_off(static_cast<int>(l)) : nullptr, w.bias2);
      ++launches_;
    }
  }
  // the dgrad operands of every implicit-dgrad layer, one launch
  std::vector<RotateTensor> rt;
  for (size_t l = 0; l < g_.cg.size() && (what & 2); ++l) {
    const ConvGeom& c = g_.cg[l];
    if (c.impl_dgrad) rt.push_back({w.cp + conv_k_off(static_cast<int>(l)), c.ldk, w.wrot[l], c.F, c.C, c.R, c.S});
  }
  if (!rt.empty()) {
    launch_rotate_weights_multi<TA>(rt.data(), static_cast<int>(rt.size()), s);
    launches_ += (static_cast<int64_t>(rt.size()) + 7) / 8;
  }
}

// Boundary exchange for turn j (exchange_activations / assemble_rows,
// cluster.cpp:113-194), targets routed with their examples.
template <class TA>
void ClusterImpl<TA>::route_forward(int j, int slot, cudaStream_t st) {
  const int nl = comm_->nlocal();
  const long long A = g_.A;
  const size_t es = sizeof(TA);
  std::vector<const void*> sa(nl), stt(nl);
  std::vector<void*> ra(nl), rt(nl);
  const int last = static_cast<int>(g_.cg.size()) - 1;
  for (int i = 0; i < nl; ++i) {
    const TA* top = stage_out_of(w_[i], g_.cg[last], last);
    sa[i] = top;
    stt[i] = w_[i].targets;
    ra[i] = w_[i].xb[slot];
    rt[i] = w_[i].tb[slot];
  }
  Comm& cx = *comm_x_;
  if (dp_) {  // own examples only
    for (int i = 0; i < nl; ++i) {
      HP_CUDA(cudaMemcpyAsync(ra[i], sa[i], b_ * A * es, cudaMemcpyDeviceToDevice, st));
      HP_CUDA(cudaMemcpyAsync(rt[i], stt[i], b_ * L_ * sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
  } else if (scheme_ == HP_SCHEME_A) {
    cx.allgather(sa, ra, b_ * A * es, st);
    cx.allgather(stt, rt, b_ * L_ * sizeof(float), st);
  } else if (scheme_ == HP_SCHEME_B) {
    for (int i = 0; i < nl; ++i)
      if (w_[i].gid == j) {
        HP_CUDA(cudaMemcpyAsync(ra[i], sa[i], b_ * A * es, cudaMemcpyDeviceToDevice, st));
        HP_CUDA(cudaMemcpyAsync(rt[i], stt[i], b_ * L_ * sizeof(float), cudaMemcpyDeviceToDevice, st));
      }
    cx.broadcast(ra, b_ * A * es, j, st);
    cx.broadcast(rt, b_ * L_ * sizeof(float), j, st);
  } else {
    const long long slice = b_ / K_;
    std::vector<const void*> sa2(nl), st2(nl);
    for (int i = 0; i < nl; ++i) {
      sa2[i] = static_cast<const char*>(sa[i]) + j * slice * A * es;
      st2[i] = static_cast<const char*>(stt[i]) + j * slice * L_ * sizeof(float);
    }
    cx.allgather(sa2, ra, slice * A * es, st);
    cx.allgather(st2, rt, slice * L_ * sizeof(float), st);
  }
}

// Model-parallel fc forward, loss and backward for one sub-batch
// (cluster.cpp:534-584).
template <class TA>
void ClusterImpl<TA>::fc_forward_backward(int j, bool beta, int slot) {
  const int nf = static_cast<int>(g_.fg.size());
  const int nl = comm_->nlocal();
  for (int l = 0; l < nf; ++l) {
    for (auto& w : w_) {
      gemm(l == 0 && slot == 1 ? w.fc0_slot1[0] : w.fc_fwd[l], "fc_fwd", l);
    }
    if (l + 1 < nf && fcK_ > 1) {
      std::vector<void*> bufs(nl);
      for (int i = 0; i < nl; ++i) bufs[i] = w_[i].fx[l + 1];
      comm_->allgather_inplace(bufs, g_.fg[l].cmax * ldn_ * sizeof(TA), st_);
    }
  }
  if (capture_fc) capture_fc_masks(j);
  // logistic cross-entropy on each worker's logit shard (no logit gather:
  // output units are independent).
  const FcGeom& fl = g_.fg.back();
  for (auto& w : w_) {
    const int rows = static_cast<int>(fl.c1[sid(w.gid)] - fl.c0[sid(w.gid)]);
    launch_xent<TA>(w.logits, ldn_, w.tb[slot], L_, static_cast<int>(fl.c0[sid(w.gid)]), rows, static_cast<int>(n_),
                    w.fdz[nf - 1], ldn_, w.loss_parts + static_cast<long long>(j) * xblocks_, w.bad,
                    fl.relu ? 1 : 0, xblocks_, st_);
    ++launches_;
  }
  // FC weight gradients (and the fused update) feed nothing downstream in this
  // step: they run on sf_ (serialised when profiling), layer li's wgrad forked
  // after layer li's dgrad -- which must read the weights before the fused
  // update rewrites them (turn j's dX uses pre-update weights, cluster.cpp:562-601).
  // (Dev HP_DEV_FC_DGRAD_FIRST: the whole dgrad chain first, then every wgrad;
  // measured 1.547 -> 1.575 ms/step on one box: the update then lands on the
  // conv backward instead of between the small FC dgrads.)
  cudaStream_t fs = profile ? st_ : sf_;
  static const bool interleave = getenv("HP_DEV_FC_DGRAD_FIRST") == nullptr;
  auto wgrad = [&](int li, Worker<TA>& w) {
    const FcGeom& f = g_.fg[li];
    const int rows = static_cast<int>(f.c1[sid(w.gid)] - f.c0[sid(w.gid)]);
    GemmPlan pw = li == 0 && slot == 1 ? w.fc0_slot1[1] : w.fc_wgrad[li];
    pw.args.epi.beta = beta ? 1 : 0;
    if (fuse_sgd_) {
      // last (or, in variable mode, every) turn: the weight update runs in
      // the wgrad epilogue; the gradient is never stored
      Epi& e = pw.args.epi;
      e.sgd_w = w.fp + fc_w_off(li);
      e.sgd_m = w.fm + fc_w_off(li);
      e.sgd_copy = kTA == kBF16 ? static_cast<void*>(w.fpt + fc_w_off(li)) : nullptr;
      e.sgd_mu = static_cast<float>(sgd_hp_.momentum);
      e.sgd_s1 = static_cast<float>(-sgd_lr_);
      e.sgd_s2 = static_cast<float>(-sgd_lr_ * sgd_hp_.weight_decay);
      e.sgd_gscale = sgd_gscale_;
      e.sgd_has_gscale = sgd_has_gscale_ ? 1 : 0;
    }
    gemm(pw, "fc_wgrad", li, fs);
    launch_rowsum<TA>(w.fdz[li], rows, static_cast<int>(n_), ldn_, w.fgr + fc_b_off(li), beta ? 1 : 0, fs);
    ++launches_;
  };
  for (int li = nf - 1; li >= 0; --li) {
    for (auto& w : w_) {
      gemm(li == 0 && slot == 1 ? w.fc0_slot1[2] : w.fc_dgrad[li], "fc_dgrad", li);
      if (interleave) {
        if (fs != st_) {
          HP_CUDA(cudaEventRecord(ev_fcd_, st_));
          HP_CUDA(cudaStreamWaitEvent(fs, ev_fcd_, 0));
        }
        wgrad(li, w);
      }
    }
    if (li > 0 && fcK_ > 1) {
      std::vector<const float*> send(nl);
      std::vector<void*> recv(nl);
      for (int i = 0; i < nl; ++i) {
        send[i] = w_[i].fdpart[li];
        recv[i] = w_[i].fdz[li - 1];
      }
      comm_->reduce_scatter(send, recv, g_.fg[li - 1].cmax * ldn_, kTA, 1.f, st_);
      launches_ += nl;
    }
  }
  if (!interleave) {
    if (fs != st_) {
      HP_CUDA(cudaEventRecord(ev_fcd_, st_));
      HP_CUDA(cudaStreamWaitEvent(fs, ev_fcd_, 0));
    }
    for (int li = nf - 1; li >= 0; --li)
      for (auto& w : w_) wgrad(li, w);
  }
  HP_CUDA(cudaEventRecord(ev_fcw_, profile ? st_ : sf_));
  HP_CUDA(cudaEventRecord(ev_fd0_, st_));
}

// return_gradients (cluster.cpp:196-269): each boundary-gradient row goes
// back to the worker whose example it is, summed over the fc shards.
template <class TA>
void ClusterImpl<TA>::return_gradients(int j, int slot, cudaStream_t st) {
  if (fcK_ == 1) return;  // dgrad wrote gflat directly
  const int nl = comm_->nlocal();
  const long long A = g_.A;
  Comm& cx = *comm_x_;
  std::vector<const float*> send(nl);
  for (int i = 0; i < nl; ++i) send[i] = w_[i].fd0[slot];
  if (scheme_ == HP_SCHEME_A) {
    std::vector<void*> recv(nl);
    for (int i = 0; i < nl; ++i) recv[i] = w_[i].gflat;
    // own.scale(K): the big batch's 1/(K*b) scale -> per-worker mean (cluster.cpp:650-652)
    cx.reduce_scatter(send, recv, b_ * A, kF32, static_cast<float>(K_), st);
  } else if (scheme_ == HP_SCHEME_B) {
    void* root_buf = nullptr;
    for (int i = 0; i < nl; ++i)
      if (w_[i].gid == j) root_buf = w_[i].gflat;
    if (!root_buf) root_buf = w_[0].gflat;  // ignored on non-root ranks
    cx.reduce(send, root_buf, b_ * A, j, kF32, 1.f, st);
  } else {
    const long long slice = b_ / K_;
    std::vector<void*> recv(nl);
    for (int i = 0; i < nl; ++i) recv[i] = w_[i].gflat + j * slice * A;
    cx.reduce_scatter(send, recv, slice * A, kF32, 1.f, st);
  }
  launches_ += nl;
}

// ------------------------------------------------------------------ backward
// conv_backward_from_flat (model.cpp:259-283) with the pool / LRN superset.
template <class TA>
void ClusterImpl<TA>::conv_backward_layer(Worker<TA>& w, int l, ConvBwdState& cs) {
  if (l == static_cast<int>(g_.cg.size()) - 1) {
    cs.gout = w.gflat;
    cs.dz_ready = false;
  }
  const ConvGeom& c = g_.cg[l];
  const TA* mask = c.relu ? w.act[l] : nullptr;
  const int B = static_cast<int>(b_);
  const OutLayout zl = c.in_q ? OutLayout{c.Hq, c.Wq, c.pad} : OutLayout{};  // dz layout
  if (c.pk > 0 && c.lrn_n > 0) {
    tl_mark("lrn_pool_bwd", l, false, st_);
    launch_lrn_pool_bwd<TA>(cs.gout, w.widx[l], w.act[l], w.dz[l], B, c.OHs, c.OWs, c.F, c.lrn_n, c.lrn_alpha,
                            c.lrn_beta, c.lrn_k, c.pk, c.ps, c.PH, c.PW, c.relu ? 1 : 0, st_, zl);
    tl_mark("lrn_pool_bwd", l, true, st_);
    ++launches_;
  } else if (c.pk > 0) {
    launch_maxpool_bwd_w<TA, TA>(cs.gout, w.widx[l], w.dz[l], mask, B, c.OHs, c.OWs, c.F, c.pk, c.ps, c.PH,
                                 c.PW, st_, zl);
    ++launches_;
  } else if (c.lrn_n > 0) {
    launch_lrn_bwd<TA, TA>(w.act[l], w.lrn_d[l], cs.gout, w.dz[l], c.P, c.F, c.lrn_n, c.lrn_alpha,
                           c.lrn_beta, c.relu ? 1 : 0, st_);
    ++launches_;
  } else if (!cs.dz_ready) {
    launch_mask_cast<TA, TA>(cs.gout, mask, w.dz[l], c.P * c.F, st_);
    ++launches_;
  }
  // Weight and bias gradients of this layer only feed the update (and the
  // all-reduce), not the backward chain: the weight gradient runs on the side
  // stream sw_, the bias gradient on sb_ (so the wgrad chain never waits for a
  // column sum), both overlapping this layer's dgrad and the layers below
  // (serialised on st_ when profiling, for clean per-GEMM times).
  cudaStream_t ws = profile ? st_ : sw_;
  cudaStream_t bs = profile ? st_ : sb_;
  if (ws != st_) {
    HP_CUDA(cudaEventRecord(ev_dz_[l], st_));
    HP_CUDA(cudaStreamWaitEvent(ws, ev_dz_[l], 0));
    HP_CUDA(cudaStreamWaitEvent(bs, ev_dz_[l], 0));
  }
  // bias grad = channel sums of dz (model.cpp:184-202)
  tl_mark("colsum", l, false, bs);
  launch_colsum<TA>(w.dz[l], c.Pq, c.F, c.F, w.cgr + conv_b_off(l), w.colsum_ws, bs);
  tl_mark("colsum", l, true, bs);
  launches_ += 2;
  HP_CUDA(cudaEventRecord(ev_bg_[l], bs));
  gemm(w.conv_wgrad[l], "conv_wgrad", l, ws);
  if (c.s2d) {
    launch_s2d_wgrad_gather(w.dwz, w.cgr + conv_k_off(l), c.ldk, c.F, c.C, c.R, c.S, c.stride, c.Rq, c.Cz, ws,
                            c.pairs ? 1 : 0);
    ++launches_;
  }
  if (K_ > 1 && skip_sync_broadcast) {  // keep the local gradients for the negative control
    HP_CUDA(cudaStreamWaitEvent(ws, ev_bg_[l], 0));
    const long long cnt = static_cast<long long>(c.F) * c.ldk + c.F;
    HP_CUDA(cudaMemcpyAsync(w.cgr_local + conv_k_off(l), w.cgr + conv_k_off(l), cnt * sizeof(float),
                            cudaMemcpyDeviceToDevice, ws));
  }
  HP_CUDA(cudaEventRecord(ev_wg_[l], ws));
  if (l == 0) return;
  const ConvGeom& pc = g_.cg[l - 1];
  const bool below_fused = pc.pk > 0 || pc.lrn_n > 0;
  gemm(w.conv_dgrad[l], "conv_dgrad", l);
  if (!c.impl_dgrad) {
    if (below_fused) {
      launch_col2im<float, TA>(w.dcol[l], w.gstage[l - 1], nullptr, B, c.H, c.W, c.C, c.R, c.S, c.stride,
                               c.pad, c.OH, c.OW, c.ldk, st_);
    } else {
      launch_col2im<TA, TA>(w.dcol[l], w.dz[l - 1], pc.relu ? w.act[l - 1] : nullptr, B, c.H, c.W, c.C,
                            c.R, c.S, c.stride, c.pad, c.OH, c.OW, c.ldk, st_);
    }
    ++launches_;
  }
  if (below_fused) {
    cs.gout = w.gstage[l - 1];
    cs.dz_ready = false;
  } else {
    cs.dz_ready = true;
  }
}

template <class TA>
void ClusterImpl<TA>::sgd_fc(double lr, float gscale, bool has_gscale, const hp_hyper& hp) {
  std::vector<SgdTensor> ts;
  for (auto& w : w_) {
    if (weights_fused_) {  // weights were updated in the wgrad epilogues: biases only
      for (size_t l = 0; l < g_.fg.size(); ++l) {
        SgdTensor t{};
        const long long off = fc_b_off(static_cast<int>(l));
        t.w = w.fp + off;
        t.mom = w.fm + off;
        t.g = w.fgr + off;
        t.copy = w.fpt ? static_cast<void*>(w.fpt + off) : nullptr;
        t.n = g_.fg[l].cmax;
        t.gscale = gscale;
        t.has_gscale = has_gscale ? 1 : 0;
        ts.push_back(t);
      }
      continue;
    }
    SgdTensor t{};
    t.w = w.fp;
    t.mom = w.fm;
    t.g = w.fgr;
    t.copy = w.fpt;
    t.n = fc_total_;
    t.gscale = gscale;
    t.has_gscale = has_gscale ? 1 : 0;
    ts.push_back(t);
  }
  launch_sgd(ts.data(), static_cast<int>(ts.size()), kTA == kBF16 ? 1 : 0, lr, hp.momentum,
             hp.weight_decay, st_);
  ++launches_;
}

template <class TA>
void ClusterImpl<TA>::sgd_conv(double lr, const hp_hyper& hp) {
  std::vector<SgdTensor> ts;
  for (auto& w : w_) {
    SgdTensor t{};
    t.w = w.cp;
    t.mom = w.cm;
    t.g = w.cgr;
    t.copy = w.cpt;
    t.n = conv_total_;
    // mean.scale(1/K) of sync_conv_gradients (cluster.cpp:293-295); already
    // applied to the owned shard by the skip-broadcast fix-up
    t.gscale = static_cast<float>(1.0 / static_cast<double>(K_));
    t.has_gscale = K_ > 1 && !skip_sync_broadcast ? 1 : 0;
    ts.push_back(t);
  }
  launch_sgd(ts.data(), static_cast<int>(ts.size()), kTA == kBF16 ? 1 : 0, lr, hp.momentum,
             hp.weight_decay, st_);
  ++launches_;
}

// ------------------------------------------------------------------ step
// All device work of one step, stream-ordered on st_ (eager or captured).
template <class TA>
void ClusterImpl<TA>::enqueue(const float* const* batches, const float* const* targets, int mem_kind,
                              const hp_hyper& hp, double lr) {
  const int nl = comm_->nlocal();
  if (tl_) HP_CUDA(cudaMemsetAsync(tl_, 0, sizeof(unsigned long long), st_));
  const double fc_lr = variable_ ? (hp.has_fc_partial_lr ? hp.fc_partial_lr : lr) : lr;
  const auto& in = g_.input;
  const long long xin = b_ * in[0] * in[1] * in[2];
  for (int i = 0; i < nl; ++i) {
    Worker<TA>& w = w_[i];
    const float* src = batches[i];
    if (mem_kind == HP_MEM_HOST) {
      HP_CUDA(cudaMemcpyAsync(w.x_nchw, batches[i], xin * sizeof(float), cudaMemcpyHostToDevice, st_));
      HP_CUDA(cudaMemcpyAsync(w.targets, targets[i], b_ * L_ * sizeof(float), cudaMemcpyHostToDevice, st_));
      io_h2d += (xin + b_ * L_) * static_cast<int64_t>(sizeof(float));
      src = w.x_nchw;
    } else {
      HP_CUDA(cudaMemcpyAsync(w.targets, targets[i], b_ * L_ * sizeof(float), cudaMemcpyDeviceToDevice, st_));
    }
    HP_CUDA(cudaMemsetAsync(w.bad, 0, sizeof(int), st_));
    w.x_src = src;
    if (g_.cg[0].impl_fwd) {
      launch_nchw_to_nhwc<TA>(src, w.x0, static_cast<int>(b_), static_cast<int>(in[0]),
                              static_cast<int>(in[1]), static_cast<int>(in[2]), st_);
      ++launches_;
    }
  }
  {
    NvtxRange r("hp.conv_forward");
    const int nc = static_cast<int>(g_.cg.size());
    for (auto& w : w_) conv_forward(w, slicing() ? nc - 1 : nc);
    if (slicing()) {  // slice-major over the workers: turn j's rows of every worker, then ev_slice_[j]
      for (int j = 0; j < K_; ++j) {
        for (auto& w : w_) conv_forward_last_slice(w, j);
        marker(700 + j, st_);
        HP_CUDA(cudaEventRecord(ev_slice_[static_cast<size_t>(j)], st_));
      }
    }
  }
  {
    // the dgrad operands (rotated bf16 kernels) of the weights the previous
    // step's update left, on the wgrad stream (idle until the backward) once
    // the conv forward is enqueued: the FC GEMMs leave SMs free (grids of 64-
    // 144 CTAs) where the previous step's tail had the rotation on st_ alone
    cudaStream_t rs = profile ? st_ : sw_;
    if (rs != st_) {
      HP_CUDA(cudaEventRecord(ev_rot0_, st_));
      HP_CUDA(cudaStreamWaitEvent(rs, ev_rot0_, 0));
    }
    for (auto& w : w_) rotate_all(w, 2, rs);
    HP_CUDA(cudaEventRecord(ev_rot_, rs));
  }
  // The turns (cluster.cpp:507-614). The boundary exchange and the gradient
  // return run on their own stream sr_ with double-buffered boundary slots:
  // turn j+1's exchange is issued BEFORE turn j's FC compute and depends only
  // on the conv tops and on turn j-1 having released its slot, so it overlaps
  // turn j's FC GEMMs ((K-1)/K of the exchange is hidden);
  // turn j's return overlaps turn j+1's FC compute the same way. The FC
  // compute of consecutive turns stays serialised on st_: it reuses the FC
  // activation buffers, and in variable mode turn j+1 reads the weights turn
  // j updated (cluster.cpp:586-601).
  cudaStream_t xs = profile ? st_ : sr_;  // serialised when profiling
  if (slicing()) {
    HP_CUDA(cudaStreamWaitEvent(xs, ev_slice_[0], 0));  // turn 0 needs slice 0 only
  } else {
    HP_CUDA(cudaEventRecord(ev_conv_, st_));
    HP_CUDA(cudaStreamWaitEvent(xs, ev_conv_, 0));
  }
  marker(100, xs);
  route_forward(0, 0, xs);
  marker(200, xs);
  HP_CUDA(cudaEventRecord(ev_xready_[0], xs));
  for (int j = 0; j < num_sub_; ++j) {
    const int slot = j & 1;
    if (j + 1 < num_sub_) {
      // slot (j+1)&1 was last read by turn j-1: its fc0 forward / xent on st_
      // and its fc0 wgrad on sf_, all before turn j-1's ev_fcw_ record
      if (j >= 1) HP_CUDA(cudaStreamWaitEvent(xs, ev_fcw_, 0));
      if (slicing()) HP_CUDA(cudaStreamWaitEvent(xs, ev_slice_[static_cast<size_t>(j + 1)], 0));
      marker(100 + j + 1, xs);
      route_forward(j + 1, slot ^ 1, xs);
      marker(200 + j + 1, xs);
      HP_CUDA(cudaEventRecord(ev_xready_[slot ^ 1], xs));
    }
    // turn j overwrites the FC activations / gradients the previous turn's
    // wgrads (sf_) read
    if (j > 0) HP_CUDA(cudaStreamWaitEvent(st_, ev_fcw_, 0));
    HP_CUDA(cudaStreamWaitEvent(st_, ev_xready_[slot], 0));
    if (j >= 2) HP_CUDA(cudaStreamWaitEvent(st_, ev_ret_[slot], 0));  // fd0[slot] returned by turn j-2
    // Fused FC weight update in the wgrad epilogue: every turn in variable
    // mode (cluster.cpp:586-601), the last turn of the accumulation in exact
    // mode (Σ_j grads × 1/num_sub, cluster.cpp:602-609, 680-696).
    fuse_sgd_ = fuse_fc_sgd && !dp_ && (variable_ || j == num_sub_ - 1);
    sgd_hp_ = hp;
    sgd_lr_ = variable_ ? fc_lr : lr;
    sgd_has_gscale_ = !variable_ && num_sub_ > 1;
    sgd_gscale_ = static_cast<float>(1.0 / static_cast<double>(num_sub_));
    marker(300 + j, st_);
    NvtxRange turn_range("hp.fc_turn");
    fc_forward_backward(j, !variable_ && j > 0, slot);
    marker(400 + j, st_);
    HP_CUDA(cudaStreamWaitEvent(xs, ev_fd0_, 0));
    marker(500 + j, xs);
    return_gradients(j, slot, xs);
    marker(600 + j, xs);
    HP_CUDA(cudaEventRecord(ev_ret_[slot], xs));
    weights_fused_ = fuse_sgd_;
    if (variable_) {  // per-sub-batch update (cluster.cpp:586-601)
      HP_CUDA(cudaStreamWaitEvent(st_, ev_fcw_, 0));
      sgd_fc(fc_lr, 1.f, false, hp);
    }
  }
  fuse_sgd_ = false;
  HP_CUDA(cudaEventRecord(ev_sr_, xs));
  HP_CUDA(cudaStreamWaitEvent(st_, ev_sr_, 0));  // every boundary gradient returned
  if (dp_ && K_ > 1) {  // pure DP: the FC gradients are all-reduced first (overlapping the conv backward)
    HP_CUDA(cudaStreamWaitEvent(sc_, ev_fcw_, 0));
    std::vector<float*> bufs(nl);
    for (int i = 0; i < nl; ++i) bufs[i] = w_[i].fgr;
    comm_s_->allreduce_f32(bufs, static_cast<size_t>(fc_total_), sc_);
    launches_ += 1;
  }
  // Conv backward; each layer's gradients (all local workers) are all-reduced
  // on the side stream as soon as they are final, overlapping the rest of the
  // backward (sync_conv_gradients, cluster.cpp:273-319, bucketed per layer in
  // backward order -- the same order on every rank).
  const int nc = static_cast<int>(g_.cg.size());
  std::vector<ConvBwdState> cbs(nl);
  NvtxRange bwd_range("hp.conv_backward_sync_sgd");
  if (!profile) HP_CUDA(cudaStreamWaitEvent(st_, ev_rot_, 0));  // the dgrad operands (rotated during the FC phase)
  for (int l = nc - 1; l >= 0; --l) {
    for (int i = 0; i < nl; ++i) conv_backward_layer(w_[i], l, cbs[i]);
    if (K_ > 1) {
      // ev_wg_[l] / ev_bg_[l]: the last local worker's weight / bias gradients of
      // layer l (sw_ and sb_ are in order)
      HP_CUDA(cudaStreamWaitEvent(sc_, ev_wg_[l], 0));
      HP_CUDA(cudaStreamWaitEvent(sc_, ev_bg_[l], 0));
      std::vector<float*> bufs(nl);
      for (int i = 0; i < nl; ++i) bufs[i] = w_[i].cgr + conv_k_off(l);
      const long long cnt = static_cast<long long>(g_.cg[l].F) * g_.cg[l].ldk + g_.cg[l].F;
      comm_s_->allreduce_f32(bufs, static_cast<size_t>(cnt), sc_);
      launches_ += 1;
    }
  }
  HP_CUDA(cudaStreamWaitEvent(st_, ev_wg_[0], 0));  // join sw_ (layer 0 is its last work)
  HP_CUDA(cudaStreamWaitEvent(st_, ev_bg_[0], 0));  // join sb_
  HP_CUDA(cudaStreamWaitEvent(st_, ev_fcw_, 0));    // join sf_
  if (K_ > 1) {
    HP_CUDA(cudaEventRecord(ev_comm_, sc_));
    HP_CUDA(cudaStreamWaitEvent(st_, ev_comm_, 0));
  }
  if (K_ > 1 && skip_sync_broadcast) {
    // sync_conv_gradients(skip_broadcast) (cluster.cpp:306-314): owners keep the
    // mean of their shard of the reference-flattened gradient, everything else
    // stays local; the mean's 1/K is applied here, so sgd_conv skips it
    long long G = 0;
    for (const auto& c : g_.cg) G += static_cast<long long>(c.F) * c.Kc + c.F;
    for (auto& w : w_) {
      long long b0, b1;
      shard(G, K_, w.gid, &b0, &b1);
      long long base = 0;
      for (size_t l = 0; l < g_.cg.size(); ++l) {
        const ConvGeom& c = g_.cg[l];
        launch_skip_sync_fixup(w.cgr + conv_k_off(static_cast<int>(l)), w.cgr_local + conv_k_off(static_cast<int>(l)),
                               c.F, c.C, c.R, c.S, c.ldk, base, b0, b1, static_cast<float>(1.0 / K_), st_);
        ++launches_;
        base += static_cast<long long>(c.F) * c.Kc + c.F;
      }
    }
  }
  if (dp_) {
    sgd_fc(lr, static_cast<float>(1.0 / static_cast<double>(K_)), K_ > 1, hp);  // mean over workers
  } else if (!variable_) {
    const bool scale = num_sub_ > 1;
    sgd_fc(lr, static_cast<float>(1.0 / static_cast<double>(num_sub_)), scale, hp);
  }
  tl_mark("sgd_conv", 0, false, st_);
  sgd_conv(lr, hp);
  tl_mark("sgd_conv", 0, true, st_);
  for (auto& w : w_) rotate_all(w, 1);  // conv1's s2d operand: the next forward's first read
  tl_mark("rotate", 0, true, st_);
  // loss partials (+ the domain-error flag) to pinned host memory
  const size_t np = static_cast<size_t>(num_sub_) * xblocks_;
  if (nl == 1 && K_ > 1) {
    std::vector<double*> b{w_[0].loss_parts};
    comm_->allreduce_f64(b, np, st_);
  }
  for (int i = 0; i < nl; ++i) {
    HP_CUDA(cudaMemcpyAsync(host_parts_ + i * np, w_[i].loss_parts, np * sizeof(double),
                            cudaMemcpyDeviceToHost, st_));
    HP_CUDA(cudaMemcpyAsync(host_bad_ + i, w_[i].bad, sizeof(int), cudaMemcpyDeviceToHost, st_));
    io_d2h += static_cast<int64_t>(np * sizeof(double) + sizeof(int));
  }
}

template <class TA>
void ClusterImpl<TA>::prefetch(const float* const* batches, const float* const* targets) {
  const int nl = comm_->nlocal();
  if (!batches || !targets) usage_error("prefetch: expected " + num(nl) + " batches and targets");
  for (int i = 0; i < nl; ++i)
    if (!batches[i] || !targets[i]) usage_error("prefetch: null batch or target");
  PrefSlot& ps = pref_[next_slot_];
  next_slot_ ^= 1;
  const auto& in = g_.input;
  const long long xin = b_ * in[0] * in[1] * in[2];
  HP_CUDA(cudaStreamWaitEvent(sx_, ps.used, 0));  // the slot's previous consumer is done
  ps.x.assign(batches, batches + nl);
  ps.t.assign(targets, targets + nl);
  ps.bytes = 0;
  const int slot = static_cast<int>(&ps - pref_);
  for (int i = 0; i < nl; ++i) {
    HP_CUDA(cudaMemcpyAsync(w_[i].xin[slot], batches[i], xin * sizeof(float), cudaMemcpyHostToDevice, sx_));
    HP_CUDA(cudaMemcpyAsync(w_[i].tin[slot], targets[i], b_ * L_ * sizeof(float), cudaMemcpyHostToDevice, sx_));
    ps.bytes += (xin + b_ * L_) * static_cast<int64_t>(sizeof(float));
  }
  HP_CUDA(cudaEventRecord(ps.ready, sx_));
  ps.valid = true;
}

template <class TA>
void ClusterImpl<TA>::run_step(const float* const* batches, const float* const* targets, int mem_kind,
                               const hp_hyper& hp, double lr, hp_step_metrics* out) {
  const int nl = comm_->nlocal();
  NvtxRange step_range("hp.run_step");
  if (mem_kind == HP_MEM_HOST && batches && targets) {
    // consume a prefetched slot holding exactly these host buffers
    for (auto& ps : pref_) {
      if (!ps.valid || static_cast<int>(ps.x.size()) != nl) continue;
      bool same = true;
      for (int i = 0; i < nl && same; ++i) same = ps.x[i] == batches[i] && ps.t[i] == targets[i];
      if (!same) continue;
      for (int i = 0; i < nl; ++i) check_targets(targets[i], b_ * L_);
      const int slot = static_cast<int>(&ps - pref_);
      std::vector<const float*> xb(nl), tb(nl);
      for (int i = 0; i < nl; ++i) {
        xb[i] = w_[i].xin[slot];
        tb[i] = w_[i].tin[slot];
      }
      ps.valid = false;
      HP_CUDA(cudaStreamWaitEvent(st_, ps.ready, 0));
      targets_checked_ = true;
      try {
        run_step(xb.data(), tb.data(), HP_MEM_DEVICE, hp, lr, out);
      } catch (...) {
        targets_checked_ = false;
        throw;
      }
      targets_checked_ = false;
      HP_CUDA(cudaEventRecord(ps.used, st_));
      io_h2d = ps.bytes;
      return;
    }
  }
  if (!batches || !targets) usage_error("run_step: expected " + num(nl) + " batches and targets");
  for (int i = 0; i < nl; ++i)
    if (!batches[i] || !targets[i])
      usage_error("run_step: expected " + num(nl) + " batches and targets, got a null entry");
  // logistic_xent's DomainError (tensor.cpp:600-603), checked before any state
  // change: the reference throws inside the loss, before the conv update (and,
  // in exact mode, before any FC update), so no parameter may move.
  if (mem_kind == HP_MEM_HOST) {
    for (int i = 0; i < nl; ++i) check_targets(targets[i], b_ * L_);
  } else if (!targets_checked_) {
    check_device_targets(targets);
  }

  // CUDA graph of the whole step, keyed by everything baked into it (input
  // pointers, memory kind, scalars). Captured on the second occurrence of a
  // key (the first runs eagerly and warms every kernel), replayed after.
  bool pinned = mem_kind == HP_MEM_DEVICE;
  if (!pinned) {
    pinned = true;
    for (int i = 0; i < nl && pinned; ++i)
      for (const float* p : {batches[i], targets[i]}) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeHost) pinned = false;
      }
    cudaGetLastError();
  }
  GraphKey key;
  for (int i = 0; i < nl; ++i) {
    key.ptrs.push_back(batches[i]);
    key.ptrs.push_back(targets[i]);
  }
  key.mem = mem_kind;
  key.scal = {lr, hp.momentum, hp.weight_decay, hp.has_fc_partial_lr ? hp.fc_partial_lr : -1.0};
  key.mem += skip_sync_broadcast ? 16 : 0;  // a different step (fix-up launches)
  const bool graphable = use_graphs && !profile && !capture_fc && pinned;
  GraphEntry* ge = nullptr;
  if (graphable) {
    auto it = graphs_.find(key);
    if (it != graphs_.end()) ge = &it->second;
  }
  launches_ = 0;
  gemm_flops_ = 0.0;
  prof_used_ = 0;
  io_h2d = io_d2h = 0;
  if (ge && ge->exec) {
    HP_CUDA(cudaEventRecord(ev0_, st_));
    HP_CUDA(cudaGraphLaunch(ge->exec, st_));
    HP_CUDA(cudaEventRecord(ev1_, st_));
    launches_ = ge->launches;
    gemm_flops_ = ge->flops;
    io_h2d = ge->h2d;
    io_d2h = ge->d2h;
  } else if (ge) {
    // second occurrence: capture
    if (graphs_.size() > 16) {
      for (auto& kv : graphs_)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      graphs_.clear();
      ge = &graphs_[key];
    }
    cudaGraph_t g = nullptr;
    HP_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue(batches, targets, mem_kind, hp, lr);
    } catch (...) {
      cudaStreamEndCapture(st_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    HP_CUDA(cudaStreamEndCapture(st_, &g));
    HP_CUDA(cudaGraphInstantiate(&ge->exec, g, 0));
    HP_CUDA(cudaGraphDestroy(g));
    ge->launches = launches_;
    ge->flops = gemm_flops_;
    ge->h2d = io_h2d;
    ge->d2h = io_d2h;
    HP_CUDA(cudaEventRecord(ev0_, st_));
    HP_CUDA(cudaGraphLaunch(ge->exec, st_));
    HP_CUDA(cudaEventRecord(ev1_, st_));
  } else {
    HP_CUDA(cudaEventRecord(ev0_, st_));
    enqueue(batches, targets, mem_kind, hp, lr);
    HP_CUDA(cudaEventRecord(ev1_, st_));
    if (graphable) graphs_[key];  // remember: capture on the next occurrence
  }
  wait_step();
  tl_flush();
  float ms = 0.f;
  HP_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
  last_ms = ms;
  last_launches = launches_;
  last_gemm_flops = gemm_flops_;
  if (profile) collect_profile();
  const size_t np = static_cast<size_t>(num_sub_) * xblocks_;
  std::vector<double> parts(np, 0.0);
  for (int i = 0; i < nl; ++i) {
    if (host_bad_[i]) domain_error("logistic_xent: target outside [0,1]");
    for (size_t e = 0; e < np; ++e) parts[e] += host_parts_[i * np + e];
  }
  // loss = sum_j loss_j * n_j / (K*b) (cluster.cpp:555-556, 710)
  double loss_weighted = 0.0;
  const double inv_n = 1.0 / static_cast<double>(n_);
  for (int j = 0; j < num_sub_; ++j) {
    double sj = 0.0;
    for (int k = 0; k < xblocks_; ++k) sj += parts[static_cast<size_t>(j) * xblocks_ + k];
    loss_weighted += (sj * inv_n) * static_cast<double>(n_);
  }
  std::memset(out, 0, sizeof *out);
  out->loss = loss_weighted / static_cast<double>(K_ * b_);
  out->fc_update_count = variable_ ? num_sub_ : 1;
  out->conv_update_count = 1;
  account(num_sub_, out);
}

template <class TA>
void ClusterImpl<TA>::wait_step() {
  if (!nccl_) {
    HP_CUDA(cudaStreamSynchronize(st_));
    return;
  }
  // NCCL: poll, so that a failed peer surfaces as HP_ERR_NCCL (communicators
  // aborted) instead of a hang in cudaStreamSynchronize
  for (int spin = 0;; ++spin) {
    const cudaError_t r = cudaStreamQuery(st_);
    if (r == cudaSuccess) break;
    if (r != cudaErrorNotReady) HP_CUDA(r);
    if (spin % 64 == 63) {
      comm_->check_async();
      comm_x_->check_async();
      comm_s_->check_async();
    }
    std::this_thread::sleep_for(std::chrono::microseconds(spin < 256 ? 2 : 50));
  }
  comm_->check_async();
  comm_x_->check_async();
  comm_s_->check_async();
}

template <class TA>
void ClusterImpl<TA>::check_device_targets(const float* const* targets) {
  const int nl = comm_->nlocal();
  for (int i = 0; i < nl; ++i) {
    HP_CUDA(cudaMemsetAsync(w_[i].bad, 0, sizeof(int), st_));
    launch_target_check(targets[i], b_ * L_, w_[i].bad, st_);
    HP_CUDA(cudaMemcpyAsync(host_bad_ + i, w_[i].bad, sizeof(int), cudaMemcpyDeviceToHost, st_));
  }
  HP_CUDA(cudaStreamSynchronize(st_));
  for (int i = 0; i < nl; ++i) {
    if (!host_bad_[i]) continue;
    std::vector<float> h(static_cast<size_t>(b_ * L_));
    HP_CUDA(cudaMemcpy(h.data(), targets[i], h.size() * sizeof(float), cudaMemcpyDeviceToHost));
    check_targets(h.data(), b_ * L_);  // the reference's exact message
    domain_error("logistic_xent: target outside [0,1]");
  }
}

// Captures one step with marker kernels (never launched: nothing changes) and
// reports marker-to-marker reachability in the graph's dependency DAG.
template <class TA>
void ClusterImpl<TA>::marker_graph(const float* const* batches, const float* const* targets, int mem_kind,
                                   const hp_hyper& hp, double lr, std::vector<int>& tags,
                                   std::vector<uint8_t>& reach) {
  HP_CUDA(cudaStreamSynchronize(st_));
  const bool pm = markers, pp = profile;
  markers = true;
  profile = false;
  const int64_t keep_launches = launches_;
  const int64_t kh = io_h2d, kd = io_d2h;
  cudaGraph_t g = nullptr;
  HP_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue(batches, targets, mem_kind, hp, lr);
  } catch (...) {
    cudaStreamEndCapture(st_, &g);
    if (g) cudaGraphDestroy(g);
    markers = pm;
    profile = pp;
    throw;
  }
  HP_CUDA(cudaStreamEndCapture(st_, &g));
  markers = pm;
  profile = pp;
  launches_ = keep_launches;
  io_h2d = kh;
  io_d2h = kd;
  size_t nn = 0, ne = 0;
  HP_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  HP_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
  HP_CUDA(cudaGraphGetEdges(g, nullptr, nullptr, &ne));
  std::vector<cudaGraphNode_t> from(ne), to(ne);
  HP_CUDA(cudaGraphGetEdges(g, from.data(), to.data(), &ne));
  std::map<cudaGraphNode_t, int> id;
  for (size_t i = 0; i < nn; ++i) id[nodes[i]] = static_cast<int>(i);
  std::vector<std::vector<int>> adj(nn);
  for (size_t e = 0; e < ne; ++e) adj[id[from[e]]].push_back(id[to[e]]);
  std::vector<int> mnode;
  tags.clear();
  for (size_t i = 0; i < nn; ++i) {
    cudaGraphNodeType t;
    HP_CUDA(cudaGraphNodeGetType(nodes[i], &t));
    if (t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams p{};
    HP_CUDA(cudaGraphKernelNodeGetParams(nodes[i], &p));
    if (!is_marker_kernel(p.func)) continue;
    tags.push_back(*static_cast<int*>(p.kernelParams[0]));
    mnode.push_back(static_cast<int>(i));
  }
  const size_t m = mnode.size();
  reach.assign(m * m, 0);
  for (size_t a = 0; a < m; ++a) {
    std::vector<uint8_t> seen(nn, 0);
    std::vector<int> stack{mnode[a]};
    while (!stack.empty()) {
      const int v = stack.back();
      stack.pop_back();
      for (int u : adj[v])
        if (!seen[u]) {
          seen[u] = 1;
          stack.push_back(u);
        }
    }
    for (size_t b = 0; b < m; ++b) reach[a * m + b] = seen[mnode[b]];
  }
  HP_CUDA(cudaGraphDestroy(g));
}

// Analytic byte counters and phase trace, exactly as the reference charges
// them (cluster.cpp:466-471, 511-528, 549-550, 576-580, 616-633, 666-670).
template <class TA>
void ClusterImpl<TA>::account(int num_sub, hp_step_metrics* out) {
  (void)num_sub;
  step_accounting(g_, K_, b_, scheme_, sent, received, trace, out->bytes_sent);
  out->n_events = static_cast<int>(trace.size());
}

// ------------------------------------------------------------------ params
template <class TA>
int64_t ClusterImpl<TA>::param_size(int worker, int which, int layer) const {
  if (worker < 0 || worker >= K_) return -1;
  const int base = which & 3;
  if (base <= 1) {
    if (layer < 0 || layer >= static_cast<int>(g_.cg.size())) return -1;
    const ConvGeom& c = g_.cg[layer];
    return base == 0 ? static_cast<int64_t>(c.F) * c.Kc : c.F;
  }
  if (layer < 0 || layer >= static_cast<int>(g_.fg.size())) return -1;
  const FcGeom& f = g_.fg[layer];
  const int64_t ns = f.c1[sid(worker)] - f.c0[sid(worker)];
  return base == 2 ? f.in * ns : ns;
}

template <class TA>
void ClusterImpl<TA>::read_param(int worker, int which, int layer, float* dst, int64_t n) {
  const int64_t want = param_size(worker, which, layer);
  if (want < 0) usage_error("read_param: bad worker/which/layer");
  if (n != want) dimension_error("read_param: size " + num(n) + ", expected " + num(want));
  Worker<TA>& w = local(worker);
  const bool mom = which >= 4;
  const int base = which & 3;
  HP_CUDA(cudaStreamSynchronize(st_));
  if (base <= 1) {
    const ConvGeom& c = g_.cg[layer];
    std::vector<float> h(static_cast<size_t>(c.F) * c.ldk + c.F);
    HP_CUDA(cudaMemcpy(h.data(), (mom ? w.cm : w.cp) + conv_k_off(layer), h.size() * sizeof(float),
                       cudaMemcpyDeviceToHost));
    if (base == 1) {
      std::memcpy(dst, h.data() + static_cast<size_t>(c.F) * c.ldk, c.F * sizeof(float));
      return;
    }
    for (int f = 0; f < c.F; ++f)
      for (int ch = 0; ch < c.C; ++ch)
        for (int r = 0; r < c.R; ++r)
          for (int s = 0; s < c.S; ++s)
            dst[((static_cast<long long>(f) * c.C + ch) * c.R + r) * c.S + s] =
                h[f * c.ldk + (r * c.S + s) * c.C + ch];
    return;
  }
  const FcGeom& f = g_.fg[layer];
  const long long ns = f.c1[sid(worker)] - f.c0[sid(worker)];
  std::vector<float> h(static_cast<size_t>(f.cmax * f.Ip + f.cmax));
  HP_CUDA(cudaMemcpy(h.data(), (mom ? w.fm : w.fp) + fc_w_off(layer), h.size() * sizeof(float),
                     cudaMemcpyDeviceToHost));
  if (base == 3) {
    std::memcpy(dst, h.data() + f.cmax * f.Ip, ns * sizeof(float));
    return;
  }
  for (long long i = 0; i < f.in; ++i) {
    const long long col = fc_col(layer, i);
    for (long long o = 0; o < ns; ++o) dst[i * ns + o] = h[o * f.Ip + col];
  }
}

// The last step's discrete forward decisions in the reference layouts (the
// parity tests replay them in the CPU checker, tests/test_alexnet_parity_gpu.py):
//   kind 0: conv layer ReLU mask, uint8 [b][F][OH][OW] (stored activation > 0)
//   kind 1: conv layer pool argmax, int32 [b][F][PH][PW], index h*OW + w in the
//           conv output plane (or_maxpool_forward's convention)
//   kind 2: fc layer ReLU mask, uint8 [n][out] of the last sub-batch (one fc
//           shard: K == 1 or the DP scheme)
// dst == nullptr: returns the element count only.
template <class TA>
int64_t ClusterImpl<TA>::read_decisions(int worker, int kind, int layer, void* dst, int64_t n) {
  Worker<TA>& w = local(worker);
  const int nc = static_cast<int>(g_.cg.size()), nf = static_cast<int>(g_.fg.size());
  auto pos = [](const TA& v) { return static_cast<float>(v) > 0.f; };
  if (kind == 0 || kind == 1) {
    if (layer < 0 || layer >= nc) usage_error("read_decisions: bad conv layer");
    const ConvGeom& c = g_.cg[layer];
    if (kind == 1 && c.pk == 0) usage_error("read_decisions: layer has no pool");
    const int64_t want = kind == 0 ? b_ * c.F * c.OH * c.OW : b_ * c.F * c.PH * c.PW;
    if (!dst) return want;
    if (n != want) dimension_error("read_decisions: size " + num(n) + ", expected " + num(want));
    HP_CUDA(cudaStreamSynchronize(st_));
    if (kind == 0) {
      const bool next_q = layer + 1 < nc && g_.cg[layer + 1].in_q && c.pk == 0 && c.lrn_n == 0;
      const long long H = next_q ? g_.cg[layer + 1].Hq : c.OHs, W = next_q ? g_.cg[layer + 1].Wq : c.OWs;
      const long long p = next_q ? g_.cg[layer + 1].pad : 0;
      std::vector<TA> h(static_cast<size_t>((next_q ? g_.cg[layer + 1].Pq : b_ * c.OHs * c.OWs) * c.F));
      HP_CUDA(cudaMemcpy(h.data(), w.act[layer], h.size() * sizeof(TA), cudaMemcpyDeviceToHost));
      uint8_t* m = static_cast<uint8_t*>(dst);
      for (long long b = 0; b < b_; ++b)
        for (long long f = 0; f < c.F; ++f)
          for (long long y = 0; y < c.OH; ++y)
            for (long long x = 0; x < c.OW; ++x)
              m[((b * c.F + f) * c.OH + y) * c.OW + x] = pos(h[((b * H + y + p) * W + x + p) * c.F + f]) ? 1 : 0;
    } else {
      std::vector<uint8_t> h(static_cast<size_t>(c.PP * c.F));
      HP_CUDA(cudaMemcpy(h.data(), w.widx[layer], h.size(), cudaMemcpyDeviceToHost));
      int32_t* o = static_cast<int32_t*>(dst);
      for (long long b = 0; b < b_; ++b)
        for (long long f = 0; f < c.F; ++f)
          for (long long y = 0; y < c.PH; ++y)
            for (long long x = 0; x < c.PW; ++x) {
              const int off = h[((b * c.PH + y) * c.PW + x) * c.F + f];
              o[((b * c.F + f) * c.PH + y) * c.PW + x] =
                  static_cast<int32_t>((y * c.ps + off / c.pk) * c.OW + x * c.ps + off % c.pk);
            }
    }
    return want;
  }
  // kind 2: layer = turn * nf + fc layer
  if (kind != 2 || layer < 0 || layer >= num_sub_ * nf) usage_error("read_decisions: bad kind/layer");
  const int j = layer / nf, l = layer % nf;
  const int64_t want = n_ * g_.fg[l].out;
  if (!dst) return want;
  if (n != want) dimension_error("read_decisions: size " + num(n) + ", expected " + num(want));
  if (static_cast<int>(cap_fc_.size()) == num_sub_ * nf && !cap_fc_[layer].empty()) {
    std::memcpy(dst, cap_fc_[layer].data(), static_cast<size_t>(want));
    return want;
  }
  if (j != num_sub_ - 1) usage_error("read_decisions: earlier turns need hp_cluster_set_debug_capture");
  HP_CUDA(cudaStreamSynchronize(st_));
  std::vector<uint8_t> m;
  fc_mask_now(l, m);
  std::memcpy(dst, m.data(), static_cast<size_t>(want));
  return want;
}

// The current turn's fc layer-l ReLU mask [n][out] (gathered activation > 0;
// the last layer: the local workers' logit shards). Stream must be idle.
template <class TA>
void ClusterImpl<TA>::fc_mask_now(int l, std::vector<uint8_t>& m) {
  const int nf = static_cast<int>(g_.fg.size());
  const FcGeom& f = g_.fg[l];
  m.assign(static_cast<size_t>(n_ * f.out), 0);
  if (l + 1 < nf) {
    std::vector<TA> h(static_cast<size_t>(g_.fg[l + 1].Ip * ldn_));
    HP_CUDA(cudaMemcpy(h.data(), w_[0].fx[l + 1], h.size() * sizeof(TA), cudaMemcpyDeviceToHost));
    for (long long o = 0; o < f.out; ++o) {
      const long long row = fc_col(l + 1, o);
      for (long long i = 0; i < n_; ++i) m[i * f.out + o] = static_cast<float>(h[row * ldn_ + i]) > 0.f ? 1 : 0;
    }
    return;
  }
  std::vector<float> h(static_cast<size_t>(f.cmax * ldn_));
  for (auto& w : w_) {
    HP_CUDA(cudaMemcpy(h.data(), w.logits, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
    const long long c0 = f.c0[sid(w.gid)], c1 = f.c1[sid(w.gid)];
    for (long long o = c0; o < c1; ++o)
      for (long long i = 0; i < n_; ++i) m[i * f.out + o] = h[(o - c0) * ldn_ + i] > 0.f ? 1 : 0;
  }
}

// Debug capture (hp_cluster_set_debug_capture): every turn's fc ReLU masks,
// taken right after the turn's forward (stream synchronised; graphs off).
template <class TA>
void ClusterImpl<TA>::capture_fc_masks(int j) {
  const int nf = static_cast<int>(g_.fg.size());
  if (static_cast<int>(cap_fc_.size()) != num_sub_ * nf) cap_fc_.assign(num_sub_ * nf, {});
  HP_CUDA(cudaStreamSynchronize(st_));
  for (int l = 0; l < nf; ++l) fc_mask_now(l, cap_fc_[j * nf + l]);
}

template <class TA>
void ClusterImpl<TA>::write_param(int worker, int which, int layer, const float* src, int64_t n) {
  const int64_t want = param_size(worker, which, layer);
  if (want < 0) usage_error("write_param: bad worker/which/layer");
  if (n != want) dimension_error("write_param: size " + num(n) + ", expected " + num(want));
  Worker<TA>& w = local(worker);
  const bool mom = which >= 4;
  const int base = which & 3;
  HP_CUDA(cudaStreamSynchronize(st_));
  float* dbase;
  std::vector<float> h;
  if (base <= 1) {
    const ConvGeom& c = g_.cg[layer];
    dbase = (mom ? w.cm : w.cp) + conv_k_off(layer);
    h.resize(static_cast<size_t>(c.F) * c.ldk + c.F);
    HP_CUDA(cudaMemcpy(h.data(), dbase, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
    if (base == 1) {
      std::memcpy(h.data() + static_cast<size_t>(c.F) * c.ldk, src, c.F * sizeof(float));
    } else {
      for (int f = 0; f < c.F; ++f)
        for (int ch = 0; ch < c.C; ++ch)
          for (int r = 0; r < c.R; ++r)
            for (int s = 0; s < c.S; ++s)
              h[f * c.ldk + (r * c.S + s) * c.C + ch] =
                  src[((static_cast<long long>(f) * c.C + ch) * c.R + r) * c.S + s];
    }
  } else {
    const FcGeom& f = g_.fg[layer];
    const long long ns = f.c1[sid(worker)] - f.c0[sid(worker)];
    dbase = (mom ? w.fm : w.fp) + fc_w_off(layer);
    h.resize(static_cast<size_t>(f.cmax * f.Ip + f.cmax));
    HP_CUDA(cudaMemcpy(h.data(), dbase, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
    if (base == 3) {
      std::memcpy(h.data() + f.cmax * f.Ip, src, ns * sizeof(float));
    } else {
      for (long long i = 0; i < f.in; ++i) {
        const long long col = fc_col(layer, i);
        for (long long o = 0; o < ns; ++o) h[o * f.Ip + col] = src[i * ns + o];
      }
    }
  }
  HP_CUDA(cudaMemcpy(dbase, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  refresh_copies(w);
  HP_CUDA(cudaStreamSynchronize(st_));
}

// gathered_model (cluster.cpp:417-437): conv from a local replica (identical
// on every worker after the all-reduce), FC shards pasted back by column.
// NCCL transport: a collective -- every rank calls it; the FC shard arenas
// (same padded layout on every rank) are all-gathered over the library's
// communicator and every rank unpacks the full model.
template <class TA>
void ClusterImpl<TA>::gather_model(float* const* ck, float* const* cb, float* const* fw,
                                   float* const* fb) {
  const int first = w_[0].gid;
  for (size_t l = 0; l < g_.cg.size(); ++l) {
    read_param(first, 0, static_cast<int>(l), ck[l], param_size(first, 0, static_cast<int>(l)));
    read_param(first, 1, static_cast<int>(l), cb[l], param_size(first, 1, static_cast<int>(l)));
  }
  std::vector<float> all;
  if (nccl_ && fcK_ > 1) {
    float* tmp = nullptr;
    HP_CUDA(cudaStreamSynchronize(st_));
    HP_CUDA(cudaMalloc(&tmp, static_cast<size_t>(fc_total_) * K_ * sizeof(float)));
    try {
      comm_->allgather(std::vector<const void*>{w_[0].fp}, std::vector<void*>{tmp},
                       static_cast<size_t>(fc_total_) * sizeof(float), st_);
      wait_step();
      all.resize(static_cast<size_t>(fc_total_) * K_);
      HP_CUDA(cudaMemcpy(all.data(), tmp, all.size() * sizeof(float), cudaMemcpyDeviceToHost));
    } catch (...) {
      cudaFree(tmp);
      throw;
    }
    HP_CUDA(cudaFree(tmp));
  }
  for (size_t l = 0; l < g_.fg.size(); ++l) {
    const FcGeom& f = g_.fg[l];
    for (int k = 0; k < fcK_; ++k) {
      const long long ns = f.c1[k] - f.c0[k];
      if (!all.empty()) {  // unpack worker k's all-gathered arena (layout as read_param)
        const float* base = all.data() + static_cast<size_t>(k) * fc_total_ + fc_w_off(static_cast<int>(l));
        for (long long i = 0; i < f.in; ++i) {
          const long long col = fc_col(static_cast<int>(l), i);
          for (long long o = 0; o < ns; ++o) fw[l][i * f.out + f.c0[k] + o] = base[o * f.Ip + col];
        }
        for (long long o = 0; o < ns; ++o) fb[l][f.c0[k] + o] = base[f.cmax * f.Ip + o];
        continue;
      }
      const int wk = fcK_ == 1 ? first : k;  // DP: every worker holds the whole (replicated) FC stack
      std::vector<float> shard(static_cast<size_t>(f.in * ns));
      read_param(wk, 2, static_cast<int>(l), shard.data(), static_cast<int64_t>(shard.size()));
      for (long long i = 0; i < f.in; ++i)
        for (long long o = 0; o < ns; ++o) fw[l][i * f.out + f.c0[k] + o] = shard[i * ns + o];
      read_param(wk, 3, static_cast<int>(l), fb[l] + f.c0[k], ns);
    }
  }
}

}  // namespace

std::unique_ptr<ClusterBase> make_cluster(const hp_model_spec* spec, const hp_cluster_config* cfg) {
  if (cfg->math_mode == HP_MATH_BF16) return std::make_unique<ClusterImpl<bf16>>(spec, cfg);
  if (cfg->math_mode == HP_MATH_TF32 || cfg->math_mode == HP_MATH_F32X3)
    return std::make_unique<ClusterImpl<float>>(spec, cfg);
  config_error("cluster.math_mode: expected bf16 | tf32 | f32x3");
}

}  // namespace hp
