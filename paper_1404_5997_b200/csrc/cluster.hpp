// The B200 hybrid-parallel cluster: the device-side replacement of
// hpsim::Cluster (include/hpsim/cluster.hpp:178-212, src/cluster.cpp:394-711).
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "hpsim_b200.h"

namespace hp {

struct ConvGeom {
  int C, H, W;                 // stage input (NHWC)
  int F, R, S, stride, pad;    // conv
  int OH, OW;                  // conv output
  bool relu;
  int lrn_n;                   // 0: no LRN
  float lrn_alpha, lrn_beta, lrn_k;
  int pk, ps;                  // max-pool (pk == 0: none)
  int PH, PW;                  // stage output
  int Kc;                      // R*S*C (im2col width)
  bool impl_fwd = false;       // fprop + wgrad as implicit GEMM (TMA im2col), no col buffer
  bool impl_dgrad = false;     // stride-1 dgrad as a conv over dY with rotated weights
  bool s2d = false;            // strided first layer as a stride-1 conv over its space-to-depth input
  int Rq = 0, Zh = 0, Zw = 0, Cz = 0;  // s2d: taps, z extents, padded z channels
  // s2d pixel pairs (bf16, 2F <= 256): the conv1 GEMM takes one row per pair of
  // horizontally adjacent output pixels and N = 2F columns (F = 64 alone is a
  // shared-memory-bound N); the output and its gradient are
  // stored OWs = OW rounded up to even wide (the extra column never feeds the
  // pool, its gradient stays zero).
  // With pairs the stored grid is z's own (OHs x OWs = Zh x Zw): viewed as
  // "pair pixels" (two horizontally adjacent pixels, 2F channels) conv1 is a
  // stride-1 3x2 conv over z' [b][Zh][Zw/2][2*Cz] -- a flat shift of the pair
  // row index -- so it runs on the flat-shift kernel (fprop) and the halo wgrad.
  bool pairs = false;
  int OWs = 0, OHs = 0;        // stored conv-output grid (OW x OH, or z's grid for pairs)
  // q-layout (see RowMap, gemm.cuh): this layer's input x and its dz are
  // stored as (H+pad) x (W+pad) row slots per image with a shared zero border
  // (stride-1 "same" convs): the conv is a flat shift of the row index.
  bool in_q = false;
  int Hq = 0, Wq = 0;
  long long Pq = 0;  // b*Hq*Wq (rows of x / dz when in_q)
  long long ldk;               // padded row stride of col / kernels (16-byte multiple)
  long long P;                 // b*OH*OW rows per worker
  long long PP;                // b*PH*PW
  long long ldp;               // P rounded up to 8 (row stride of layer 0's transposed col)
};

struct FcGeom {
  long long in, out;   // reference dims
  long long Ip;        // device input width: A (layer 0) or K*cmax(prev)
  long long cmax;      // padded rows per shard chunk
  bool relu;
  std::vector<long long> c0, c1;  // shard_range per worker
};

// Validated spec + derived geometry (ModelSpec::validate, model.cpp:39-91,
// plus the floor-mode / LRN / pool superset).
struct Geometry {
  std::vector<hp_conv_layer> conv;
  std::vector<hp_fc_layer> fc;
  int64_t input[3];
  int64_t num_classes;
  std::vector<ConvGeom> cg;
  std::vector<FcGeom> fg;
  long long A;  // flattened conv output
};

Geometry make_geometry(const hp_model_spec* spec, int K, long long b);

class ClusterBase {
 public:
  virtual ~ClusterBase() = default;
  virtual void run_step(const float* const* batches, const float* const* targets, int mem_kind,
                        const hp_hyper& hp, double lr, hp_step_metrics* out) = 0;
  virtual int64_t param_size(int worker, int which, int layer) const = 0;
  virtual void read_param(int worker, int which, int layer, float* dst, int64_t n) = 0;
  virtual void write_param(int worker, int which, int layer, const float* src, int64_t n) = 0;
  // Debug / parity: the last step's ReLU masks and pool argmax (see cluster.cu).
  virtual int64_t read_decisions(int worker, int kind, int layer, void* dst, int64_t n) = 0;
  virtual void gather_model(float* const* ck, float* const* cb, float* const* fw,
                            float* const* fb) = 0;

  virtual void* stream() const = 0;
  virtual void rebuild_plans() = 0;  // after a kernel-choice toggle (drops captured graphs)
  // Stage the NEXT step's host batches/targets into a device slot on the copy
  // stream (async); a later run_step with the same host pointers consumes the
  // slot instead of copying on the compute stream (double buffering: the copy
  // of step i+1 overlaps the compute of step i).
  virtual void prefetch(const float* const* batches, const float* const* targets) = 0;
  // Debug: capture one step (never executed) with marker kernels at the turn
  // boundaries and report, for every pair of markers (tags[i], tags[j]),
  // whether j is reachable from i in the captured graph's dependency DAG.
  virtual void marker_graph(const float* const* batches, const float* const* targets, int mem_kind,
                            const hp_hyper& hp, double lr, std::vector<int>& tags,
                            std::vector<uint8_t>& reach) = 0;

  struct GemmProf {
    const char* tag;
    int layer;
    double flops;
    float ms;
  };
  bool profile = false;            // bracket every GEMM with CUDA events
  bool markers = false;            // debug: tagged 1-thread marker kernels at the turn boundaries
  bool use_graphs = true;          // replay the step as a captured CUDA graph
  bool fuse_fc_sgd = true;         // FC weight update in the wgrad GEMM epilogue
  bool use_shift = true;           // bf16 stride-1 convs via the flat-shift kernel (else TMA im2col)
  bool capture_fc = false;         // debug: keep every turn's fc ReLU masks (read_decisions kind 2; no graphs)
  std::vector<GemmProf> prof;      // last step, launch order
  double prof_gemm_ms = 0.0;
  double last_gemm_flops = 0.0;    // algorithmic GEMM FLOPs of the last step
  int64_t io_h2d = 0, io_d2h = 0;  // bytes copied host<->device by the last step

  std::vector<hp_trace_event> trace;
  std::vector<std::array<int64_t, 4>> sent, received;  // per worker (all K)
  bool skip_sync_broadcast = false;
  double last_ms = 0.0;
  int64_t last_launches = 0;
};

// Host-only analytic accounting of one step (adds into sent/received/bytes_sent,
// replaces trace). Every rank computes the counters of all K workers.
void step_accounting(const Geometry& g, int K, long long b, int scheme,
                     std::vector<std::array<int64_t, 4>>& sent,
                     std::vector<std::array<int64_t, 4>>& received, std::vector<hp_trace_event>& trace,
                     int64_t* bytes_sent);

std::unique_ptr<ClusterBase> make_cluster(const hp_model_spec* spec, const hp_cluster_config* cfg);

}  // namespace hp
