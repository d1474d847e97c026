/*
 * hpsim_b200 — C ABI of the B200-native hybrid-parallel training step.
 *
 * This is the drop-in boundary for the reference's `hpsim::Cluster` path
 * (/root/reference/proj/core/include/hpsim/cluster.hpp:178-212,
 *  src/cluster.cpp:394-711). Every entry point below names the reference
 * interface it replaces. Plain C types only: no torch, no C++ in signatures.
 *
 * Conventions (mirroring the reference):
 *   - Status codes map 1:1 onto the reference's exception types
 *     (include/hpsim/errors.hpp:22-44): CONFIG <-> ConfigError, DIMENSION <->
 *     DimensionError, DOMAIN <-> DomainError, USAGE <-> UsageError. CUDA and
 *     NCCL failures have their own codes. hp_last_error() returns the message
 *     (thread-local), with the reference's field-path wording.
 *   - Tensors cross the boundary in the reference's layouts: batches NCHW
 *     [b][C][H][W], targets [b][L], conv kernels [F][C][R][S], fc weights
 *     [in][out] (shards: columns shard_range(out, K, i)). Device-side layouts
 *     (NHWC activations, [out][in] fc weights, HWC flatten order) are private.
 *   - The library owns all device memory. Host pointers are borrowed for the
 *     duration of the call; device pointers (HP_MEM_DEVICE) must be ready on
 *     the current device before the call (the call synchronises internally).
 *   - One caller thread drives a cluster at a time (reference: single
 *     conceptual writer).
 */
#ifndef HPSIM_B200_H_
#define HPSIM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HP_API __attribute__((visibility("default")))
#else
#define HP_API
#endif

/* ---- status codes (errors.hpp:22-44) ---------------------------------- */
enum {
  HP_OK = 0,
  HP_ERR_CONFIG = 1,    /* hpsim::ConfigError    */
  HP_ERR_DIMENSION = 2, /* hpsim::DimensionError */
  HP_ERR_DOMAIN = 3,    /* hpsim::DomainError    */
  HP_ERR_USAGE = 4,     /* hpsim::UsageError     */
  HP_ERR_CUDA = 5,
  HP_ERR_NCCL = 6
};

enum { HP_SCHEME_A = 0, HP_SCHEME_B = 1, HP_SCHEME_C = 2, /* cluster.hpp:36 */
       /* B200 extension (BASELINE config 5 comparison, no reference
        * counterpart): pure data parallelism -- every worker holds the whole FC
        * stack, runs it on its own b examples, and the FC gradients are
        * all-reduced with the conv gradients (one exact update per step). */
       HP_SCHEME_DP = 3 };
enum { HP_PRECISION_SINGLE = 0, HP_PRECISION_DOUBLE = 1 };  /* tensor.hpp:28 */
enum {
  HP_MATH_BF16 = 0,  /* bf16 operands, fp32 accumulate (throughput mode) */
  HP_MATH_TF32 = 1,  /* fp32 operands read as tf32                      */
  HP_MATH_F32X3 = 2  /* 3xTF32 split: near-fp32 (parity mode)           */
};
enum { HP_TRANSPORT_LOGICAL = 0, HP_TRANSPORT_NCCL = 1 };
enum { HP_MEM_HOST = 0, HP_MEM_DEVICE = 1 };
enum { /* MsgClass, cluster.hpp:41-46 */
  HP_MSG_FC_ACTIVATIONS = 0,
  HP_MSG_FC_GRADIENTS = 1,
  HP_MSG_FC_INTERNAL = 2,
  HP_MSG_CONV_SYNC = 3
};
enum { /* Phase, cluster.hpp:86 */
  HP_PHASE_CONV_FWD = 0,
  HP_PHASE_FC_FWD = 1,
  HP_PHASE_FC_BWD = 2,
  HP_PHASE_CONV_BWD = 3,
  HP_PHASE_SYNC = 4
};

/* ---- model spec (model.hpp:24-58), superset for AlexNet ---------------- */
typedef struct hp_conv_layer {
  int64_t in_channels;
  int64_t out_channels;
  int32_t kernel;
  int32_t stride;
  int32_t pad;
  int32_t relu;
  /* Superset (absent from the reference, zero = off): */
  int32_t floor_mode;  /* output = floor((H+2p-k)/s)+1 instead of exact division */
  int32_t lrn_size;    /* cross-channel LRN after ReLU (Krizhevsky 2012)        */
  double lrn_alpha;    /* b = a / (k + alpha * sum_{window} a^2)^beta (alpha NOT /n) */
  double lrn_beta;
  double lrn_k;
  int32_t pool_kernel; /* max-pool after (LRN,) ReLU; floor mode                   */
  int32_t pool_stride;
} hp_conv_layer;

typedef struct hp_fc_layer {
  int64_t in_dim;
  int64_t out_dim;
  int32_t relu;
} hp_fc_layer;

typedef struct hp_model_spec {
  const hp_conv_layer* conv;
  int32_t n_conv;
  const hp_fc_layer* fc;
  int32_t n_fc;
  int64_t input_shape[3]; /* C, H, W */
  int64_t num_classes;
} hp_model_spec;

/* ---- cluster config (cluster.hpp:59-68) + device fields ---------------- */
typedef struct hp_cluster_config {
  int32_t workers;            /* K */
  int64_t per_worker_batch;   /* b */
  int32_t scheme;             /* HP_SCHEME_*            */
  int32_t variable_batch;     /* approximate variant     */
  int32_t precision;          /* HP_PRECISION_SINGLE only (double -> CONFIG) */
  uint64_t seed;
  int32_t math_mode;          /* HP_MATH_*               */
  int32_t transport;          /* HP_TRANSPORT_*          */
  int32_t rank;               /* NCCL: this process's worker id */
  int32_t device;             /* CUDA device ordinal (-1: current) */
  unsigned char nccl_id[128]; /* NCCL: ncclUniqueId from hp_nccl_unique_id on rank 0 */
} hp_cluster_config;

/* ---- hyperparameters (optimizer.hpp:27-51) ----------------------------- */
typedef struct hp_hyper {
  double momentum;
  double lr;
  double weight_decay;
  int32_t has_fc_partial_lr;
  double fc_partial_lr;
} hp_hyper;

/* ---- metrics / trace (cluster.hpp:86-117) ------------------------------ */
typedef struct hp_trace_event {
  int32_t phase;
  int32_t sub_batch;
  int32_t worker;
  int64_t bytes_total;
  int64_t bytes_max_sender;
} hp_trace_event;

typedef struct hp_step_metrics {
  double loss;
  int32_t fc_update_count;
  int32_t conv_update_count;
  int64_t bytes_sent[4];
  int32_t n_events; /* full trace via hp_cluster_trace */
} hp_step_metrics;

typedef struct hp_cluster hp_cluster;

/* ---- errors ------------------------------------------------------------- */
HP_API const char* hp_last_error(void);
HP_API const char* hp_version(void);

/* ---- cluster lifecycle --------------------------------------------------
 * Replaces hpsim::Cluster::Cluster (cluster.hpp:180, cluster.cpp:394-415):
 * validates spec and config (ModelSpec::validate model.cpp:39-91,
 * ClusterConfig::validate cluster.cpp:50-67), draws the initial model with the
 * reference's GaussianSampler stream (init_model model.cpp:133-162) on the
 * host, and uploads the conv replicas and fc column shards. */
HP_API int hp_cluster_create(const hp_model_spec* spec, const hp_cluster_config* cfg,
                             hp_cluster** out);
HP_API void hp_cluster_destroy(hp_cluster* c);

/* NCCL transport: rank 0 creates the id and ships it to the other ranks
 * (bench.py uses torch.distributed for that plumbing). */
HP_API int hp_nccl_unique_id(unsigned char out[128]);

/* Replaces Cluster::run_step (cluster.hpp:190-192, cluster.cpp:439-711).
 * batches[i] / targets[i]: worker i's [b][C][H][W] images and [b][L] targets.
 * LOGICAL transport: K entries. NCCL transport: 1 entry (this rank's).
 * mem_kind: HP_MEM_HOST (copied in) or HP_MEM_DEVICE. */
HP_API int hp_cluster_run_step(hp_cluster* c, const float* const* batches,
                               const float* const* targets, int mem_kind, const hp_hyper* hp,
                               double lr, hp_step_metrics* out);

/* B200 extension (no reference counterpart): stage the NEXT step's HOST
 * batches/targets (same shapes as run_step) into one of two device slots on a
 * copy stream and return immediately. A later hp_cluster_run_step with
 * mem_kind HP_MEM_HOST and the same host pointers consumes the slot instead of
 * copying on the compute stream, so the copy of step i+1 overlaps the compute
 * of step i. The host buffers must stay valid (and unchanged) until that
 * run_step returns; pinned memory makes the copy truly asynchronous. */
HP_API int hp_cluster_prefetch(hp_cluster* c, const float* const* batches, const float* const* targets);

/* Trace of the last step (StepTrace, cluster.hpp:103-109). Returns count. */
HP_API int hp_cluster_trace(const hp_cluster* c, hp_trace_event* out, int cap);
/* Cumulative per-worker ByteCounters (cluster.hpp:49-57). */
HP_API int hp_cluster_worker_bytes(const hp_cluster* c, int worker, int64_t sent[4],
                                   int64_t received[4]);

/* Parameter access in reference layouts (WorkerState, cluster.hpp:77-84).
 * which: 0 conv kernels [F][C][R][S], 1 conv bias [F], 2 fc weight shard
 * [in][out_i], 3 fc bias shard [out_i]; +4 = the matching momentum tensor.
 * NCCL transport: only the local rank's worker is addressable. */
enum { HP_P_CONV_K = 0, HP_P_CONV_B = 1, HP_P_FC_W = 2, HP_P_FC_B = 3, HP_P_MOMENTUM = 4 };
HP_API int64_t hp_cluster_param_size(const hp_cluster* c, int worker, int which, int layer);
HP_API int hp_cluster_read_param(hp_cluster* c, int worker, int which, int layer, float* dst,
                                 int64_t n);
/* Parity / debug (no reference counterpart): the last step's discrete forward
 * decisions in the reference layouts -- kind 0: conv layer ReLU mask, uint8
 * [b][F][OH][OW]; kind 1: conv pool argmax, int32 [b][F][PH][PW] as the index
 * h*OW+w in the conv output plane; kind 2: fc layer ReLU mask, uint8 [n][out]
 * of the last sub-batch (K == 1 or scheme DP). dst NULL: returns the count.
 * Returns the element count, or -1 (hp_last_error). */
/* Debug capture of every turn's fc ReLU masks for hp_cluster_debug_decisions
 * (synchronises inside the step; disables graph replay while on). */
HP_API int hp_cluster_set_debug_capture(hp_cluster* c, int on);
HP_API int64_t hp_cluster_debug_decisions(hp_cluster* c, int worker, int kind, int layer, void* dst,
                                          int64_t n);
HP_API int hp_cluster_write_param(hp_cluster* c, int worker, int which, int layer,
                                  const float* src, int64_t n);

/* Cluster::gathered_model (cluster.cpp:417-437): worker 0's conv replica and
 * the fc shards pasted back by column. Pointers are host buffers in reference
 * layouts, one per layer. NCCL transport: collective (every rank calls). */
HP_API int hp_cluster_gather_model(hp_cluster* c, float* const* conv_k, float* const* conv_b,
                                   float* const* fc_w, float* const* fc_b);

/* Cluster::set_skip_sync_broadcast (cluster.hpp:203-205) negative control. */
HP_API int hp_cluster_set_skip_sync_broadcast(hp_cluster* c, int v);

/* Wall-clock of the last step's device work, ms (CUDA events). */
HP_API double hp_cluster_last_step_ms(const hp_cluster* c);
/* Number of kernels this library launched in the last step. */
HP_API int64_t hp_cluster_last_step_launches(const hp_cluster* c);

/* ---- instrumentation (bench.py / profiling; not in the reference) -------- */
/* The CUDA stream every kernel of this cluster is launched on (cudaStream_t). */
HP_API void* hp_cluster_stream(const hp_cluster* c);
/* Host<->device bytes the last step copied (inputs in, loss partials out). */
HP_API void hp_cluster_last_step_io(const hp_cluster* c, int64_t* h2d, int64_t* d2h);
/* Algorithmic FLOPs (2*M*N*K) of the tcgen05 GEMMs the last step ran. */
HP_API double hp_cluster_last_gemm_flops(const hp_cluster* c);
/* Bracket every GEMM with CUDA events on the launching stream (adds event
 * records; off for timed runs). */
HP_API int hp_cluster_set_profile(hp_cluster* c, int on);
/* FC weight update fused into the FC wgrad GEMM epilogue (default on); off
 * stores the FC gradients and runs the multi-tensor SGD kernel instead. */
HP_API int hp_cluster_set_fuse_fc_sgd(hp_cluster* c, int on);
/* bf16 stride-1 convs through the flat-shift kernel (default on); off uses the
 * TMA-im2col implicit GEMM for them (A/B comparisons; rebuilds the plans). */
HP_API int hp_cluster_set_shift_conv(hp_cluster* c, int on);
/* Replay each step as a captured CUDA graph (default on). A graph is keyed by
 * the step's input pointers, memory kind and scalars; it is captured the second
 * time a key is seen (the first runs eagerly) and replayed afterwards. Host
 * inputs are graphed only when they are pinned. */
HP_API int hp_cluster_set_graphs(hp_cluster* c, int on);
/* Per-GEMM record of the last profiled step: tag ("conv_fwd", ...), layer,
 * FLOPs and event-timed ms. Returns the count. */
typedef struct hp_gemm_prof {
  char tag[16];
  int32_t layer;
  double flops;
  double ms;
} hp_gemm_prof;
HP_API int hp_cluster_gemm_profile(const hp_cluster* c, hp_gemm_prof* out, int cap);
/* Debug (graph-structure tests): capture one step WITHOUT running it, with a
 * 1-thread tagged marker kernel at each turn boundary -- 100+j / 200+j around
 * turn j's boundary exchange (stream sr), 300+j / 400+j around turn j's FC
 * forward+backward (compute stream), 500+j / 600+j around turn j's gradient
 * return -- and report reach[i*n+k] = 1 when marker k is reachable from
 * marker i in the captured dependency DAG. tags/reach: cap and cap*cap. */
HP_API int hp_cluster_debug_marker_graph(hp_cluster* c, const float* const* batches,
                                         const float* const* targets, int mem_kind, const hp_hyper* hp,
                                         double lr, int32_t* tags, uint8_t* reach, int cap,
                                         int* n_markers);

/* ---- host-side helpers shared with the reference ------------------------ */
/* Analytic byte counters + phase trace of `steps` steps (cluster.cpp:466-673)
 * without running anything: validates spec/config like hp_cluster_create,
 * fills bytes_sent[4] (summed over steps), the last step's trace, and the
 * per-worker cumulative ByteCounters (worker_sent / worker_received: K*4).
 * This is the host logic every rank runs for all K workers. */
HP_API int hp_step_accounting(const hp_model_spec* spec, const hp_cluster_config* cfg, int steps,
                              int64_t bytes_sent[4], hp_trace_event* trace, int cap, int* n_events,
                              int64_t* worker_sent, int64_t* worker_received);
/* shard_range (cluster.cpp:69-75). */
HP_API void hp_shard_range(int64_t total, int parts, int idx, int64_t* begin, int64_t* end);
/* GaussianSampler(seed).next() x n (rng.hpp:26-56), replayed on the host. */
HP_API void hp_gaussian_fill(uint64_t seed, double* out, int64_t n);
/* Same stream, scaled by `scale`, rounded to float. */
HP_API void hp_gaussian_fill_f32(uint64_t seed, double scale, float* out, int64_t n);

/* ---- kernel-level entry points (device pointers, for parity tests) ------
 * Each mirrors one dense kernel of include/hpsim/tensor.hpp:92-139 with the
 * B200 kernel that replaces it inside the step. */
typedef struct hp_gemm_desc {
  int32_t math;
  const void* a; int32_t a_mn; int64_t lda;
  const void* b; int32_t b_mn; int64_t ldb;
  int32_t M, N, K;
  void* c; int64_t ldc; int32_t c_type; int32_t c_trans;
  float alpha; int32_t beta;
  const float* bias; int32_t bias_mode; int32_t relu;
  const void* mask; int64_t ldmask; int32_t mask_type; int32_t mask_trans;
  int32_t splits; int32_t bn;
  float* ws; /* splits*M*N floats when splits > 1 */
  int32_t cta2; /* -1 auto (CTA pairs, M=256 tiles, for M >= 256), 0 single-CTA, 1 force pairs */
} hp_gemm_desc;
/* D = A * B^T on tcgen05 (replaces matmul/_tn/_nt, tensor.cpp:254-305). */
HP_API int hp_kernel_gemm(const hp_gemm_desc* d, void* stream);
HP_API int hp_kernel_gemm_splits(const hp_gemm_desc* d);
/* Dev hook for microbenchmarks: force later auto-configured GEMM plans to
 * (cta2, bn); (-1, 0) restores the automatic tile choice. */
HP_API void hp_debug_gemm_force(int cta2, int bn);
/* Dev hook: flags for later plans; bit 0 skips the epilogue's global traffic
 * (mainloop-only timing; results are garbage). */
HP_API void hp_debug_gemm_flags(int flags);

/* Implicit-GEMM convolution on tcgen05 with TMA im2col operand loads (no
 * im2col buffer); NHWC activations in the operand type (bf16 for
 * HP_MATH_BF16, fp32 otherwise), fp32 outputs. C must be a multiple of 128
 * bytes of operand (64 bf16 / 32 fp32 channels). Replaces conv2d_forward /
 * conv2d_backward (tensor.cpp:419-516, 520-552).
 *   fprop: y[B*OH*OW][F] = conv(x[B][H][W][C], w[F][R][S][C])
 *   wgrad: dw[F][R*S*C]  = sum_pixels dy[B*OH*OW][F] (x) im2col(x)
 *   dgrad (stride 1): dx[B*H*W][C] = conv(dy[B][OH][OW][F], wrot[C][R][S][F]) with
 *         wrot[c][r][s][f] = w[f][R-1-r][S-1-s][c] and padding R-1-pad. */
HP_API int hp_kernel_conv_fprop(int math, const void* x, int B, int H, int W, int C, const void* w,
                                int F, int R, int S, int stride, int pad, float* y, void* stream);
HP_API int hp_kernel_conv_wgrad(int math, const void* x, int B, int H, int W, int C, const void* dy,
                                int F, int R, int S, int stride, int pad, float* dw, float* ws,
                                int64_t ws_floats, void* stream);
HP_API int hp_kernel_conv_dgrad(int math, const void* dy, int B, int OH, int OW, int F,
                                const void* wrot, int C, int R, int S, int pad, float* dx,
                                void* stream);
/* Stride-1 conv as a flat-shift implicit GEMM on tcgen05 (bf16, CTA pairs):
 * y[rows][N] fp32 = sum_{r,s} x[row + r*wq + s][0..C) . w[N][(r*S+s)*C + c],
 * one smem halo per 64-channel block reused by all R*S taps. x is a
 * zero-bordered "q-layout" activation (or any [rows][C] bf16 matrix); border
 * and wrap-around rows of y are garbage. C % 64 == 0, 128 + (R-1)*wq + S-1 <= 256.
 * Replaces conv2d_forward / the stride-1 conv2d_backward dgrad (tensor.cpp:419-516). */
HP_API int hp_kernel_conv_shift(const void* x, int64_t rows, int C, int R, int S, int wq, const void* w,
                                int N, float* y, int boff_mode, void* stream);

/* Fused LRN + overlapping max-pool of one conv stage (the AlexNet superset;
 * no reference counterpart -- parity pinned by the oracle's torch-checked
 * restatement, oracle/hpsim_oracle.c or_lrn_* / or_maxpool_*). The same
 * launch the step makes. math: HP_MATH_BF16 (a, y, dz bf16) or fp32.
 * a [B][H][W][C] conv output (post-ReLU), y [B][PH][PW][C] with
 * PH = (H - pk) / ps + 1, widx [B][PH][PW][C] uint8 window offset r*pk + q of
 * the FIRST maximum in row-major window order (strict >, NaN wins), gy fp32
 * [B][PH][PW][C], dz [B][H][W][C] (x ReLU mask of a when relu_mask); bias_grad (optional,
 * LRN stages) [C] = channel sums of the stored dz (model.cpp:184-202), the step's colsum.
 * LRN (Krizhevsky 2012): b_c = a_c (k + alpha sum_{|i-c|<=n/2} a_i^2)^-beta,
 * alpha NOT divided by n. lrn_size 0: max-pool only. */
HP_API int hp_kernel_lrn_pool_fwd(int math, const void* a, int B, int H, int W, int C, int lrn_size,
                                  float alpha, float beta, float k, int pk, int ps, void* y,
                                  uint8_t* widx, void* stream);
HP_API int hp_kernel_lrn_pool_bwd(int math, const float* gy, const uint8_t* widx, const void* a, int B,
                                  int H, int W, int C, int lrn_size, float alpha, float beta, float k,
                                  int pk, int ps, int relu_mask, void* dz, float* bias_grad, void* stream);
/* The step's momentum SGD (momentum_update, optimizer.cpp:19-31) on one fp32
 * tensor: g *= gscale (if has_gscale), delta = mu*delta; delta += -lr*g;
 * delta += -lr*wd*w; w += delta -- four rounded passes, scalars formed in
 * double and rounded to float once (tensor.cpp:195-229). bf16_copy: optional
 * bf16 copy of the updated w. */
HP_API int hp_kernel_sgd(float* w, float* mom, const float* g, int64_t n, double lr, double momentum,
                         double weight_decay, float gscale, int has_gscale, void* bf16_copy, void* stream);

/* ---- input pipeline: SPEC data_gen ----------------------
 * The deterministic synthetic classification dataset (class-conditional
 * Gaussian blobs), generated on the GPU. The reference specifies this module
 * but has no code for it; the generator is defined in csrc/datagen.cu:
 *   class(i) = perm(i) mod L  (perm: seeded bijection of [0, N); every class
 *              holds floor(N/L) or ceil(N/L) examples)
 *   x_i[e]   = separation * mean(class(i), e) + noise(i, e), both N(0, 1) from
 *              Philox4x32-10 keyed by seed (the class means are separation-scaled
 *              standard normals; unit-variance noise)
 *   t_i      = one_hot(class(i))
 * Examples [first, first + count) are written as inputs [count][C][H][W] and
 * targets [count][L] (the run_step batch layouts) -- bit-identical to the same
 * rows of the whole dataset. mem_kind HP_MEM_DEVICE: device pointers, stream-
 * ordered on `stream` (the input pipeline: run_step consumes the batch with
 * HP_MEM_DEVICE, no host copy); HP_MEM_HOST: generated on the current device
 * and copied out before return.
 * Errors: HP_ERR_CONFIG for num_classes < 2, negative num_examples, empty
 * shape, negative separation; HP_ERR_USAGE for a range outside [0, N). */
typedef struct hp_dataset_spec {
  int64_t num_examples;
  int32_t channels, height, width;
  int32_t num_classes;
  uint64_t seed;
  double separation; /* std of the class means: two class means differ by separation*sqrt(2) per
                        coordinate (RMS) -- 10/sqrt(2) puts them 10 sigma apart */
} hp_dataset_spec;
HP_API int hp_data_generate(const hp_dataset_spec* spec, int64_t first, int64_t count, float* inputs,
                            float* targets, int mem_kind, void* stream);
/* *cls = the class of example `index` (host evaluation of the same permutation). */
HP_API int hp_data_class_of(const hp_dataset_spec* spec, int64_t index, int64_t* cls);

#ifdef __cplusplus
}
#endif

#endif /* HPSIM_B200_H_ */
