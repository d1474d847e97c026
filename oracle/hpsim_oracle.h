/*
 * hpsim_oracle — CPU restatement of the reference's hybrid-parallel step.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_1404_5997_b200/)
 * links, imports or calls this; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may, and only as the
 * checker or the timed CPU baseline.
 *
 * Restates /root/reference/proj/core (hpsim) in plain C, double precision,
 * with the reference's loop and summation orders, so that on the reference's
 * own configurations it is bit-identical to the reference built in double
 * (pinned by tests/test_oracle_vs_reference.py against oracle/_ref). It adds
 * the AlexNet superset the reference cannot express (floor-mode geometry,
 * cross-channel LRN, overlapping max-pool); those three are
 * "parity unpinned by the reference" and are cross-checked against
 * torch.nn.functional on CPU instead (tests/test_oracle_extensions.py).
 */
#ifndef HPSIM_ORACLE_H_
#define HPSIM_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same memory layout as hp_conv_layer / hp_fc_layer / hp_model_spec in
 * include/hpsim_b200.h, so one ctypes description serves both. */
typedef struct or_conv_layer {
  int64_t in_channels, out_channels;
  int32_t kernel, stride, pad, relu;
  int32_t floor_mode;
  int32_t lrn_size;
  double lrn_alpha, lrn_beta, lrn_k;
  int32_t pool_kernel, pool_stride;
} or_conv_layer;

typedef struct or_fc_layer {
  int64_t in_dim, out_dim;
  int32_t relu;
} or_fc_layer;

typedef struct or_model_spec {
  const or_conv_layer* conv;
  int32_t n_conv;
  const or_fc_layer* fc;
  int32_t n_fc;
  int64_t input_shape[3];
  int64_t num_classes;
} or_model_spec;

typedef struct or_cluster_config {
  int32_t workers;
  int64_t per_worker_batch;
  int32_t scheme; /* 0 A, 1 B, 2 C */
  int32_t variable_batch;
  int32_t precision; /* 0 single, 1 double: byte accounting only (compute is double) */
  uint64_t seed;
} or_cluster_config;

typedef struct or_hyper {
  double momentum, lr, weight_decay;
  int32_t has_fc_partial_lr;
  double fc_partial_lr;
} or_hyper;

typedef struct or_trace_event {
  int32_t phase, sub_batch, worker;
  int64_t bytes_total, bytes_max_sender;
} or_trace_event;

typedef struct or_step_metrics {
  double loss;
  int32_t fc_update_count, conv_update_count;
  int64_t bytes_sent[4];
  int32_t n_events;
} or_step_metrics;

typedef struct or_cluster or_cluster;

/* Status codes as in hpsim_b200.h: 1 config, 2 dimension, 3 domain, 4 usage. */
const char* or_last_error(void);
int or_validate(const or_model_spec* spec);
int or_conv_output_sizes(const or_model_spec* spec, int64_t* hw /* 2 per layer, after pool */);
int64_t or_flattened_conv_size(const or_model_spec* spec);

or_cluster* or_cluster_create(const or_model_spec* spec, const or_cluster_config* cfg, int* status);
void or_cluster_destroy(or_cluster* c);
int or_cluster_run_step(or_cluster* c, const double* const* batches, const double* const* targets,
                        const or_hyper* hp, double lr, or_step_metrics* out);
int or_cluster_trace(const or_cluster* c, or_trace_event* out, int cap);
int or_cluster_worker_bytes(const or_cluster* c, int worker, int64_t sent[4], int64_t received[4]);
int64_t or_cluster_param_size(const or_cluster* c, int worker, int which, int layer);
int or_cluster_read_param(const or_cluster* c, int worker, int which, int layer, double* dst,
                          int64_t n);
int or_cluster_write_param(or_cluster* c, int worker, int which, int layer, const double* src,
                           int64_t n);
void or_cluster_set_skip_sync_broadcast(or_cluster* c, int v);
/* test-only: 0 = all double (the reference restatement), 1 = bf16 storage
 * emulation of the B200 bf16 math mode (see hpsim_oracle.c). */
int or_cluster_set_storage_rounding(or_cluster* c, int mode);
/* test-only decision replay: see hpsim_oracle.c */
int or_cluster_force_decisions(or_cluster* c, int worker, int kind, int layer, const void* src, int64_t n);
int or_cluster_decision_stats(const or_cluster* c, int worker, int kind, int layer, int64_t* mismatches,
                              double* max_gap);
void or_set_threads(int n);

/* Primitives (tensor.cpp / model.cpp restated, plus the extensions). */
void or_gaussian_fill(uint64_t seed, double* out, int64_t n);
void or_uniform_u64(uint64_t seed, uint64_t* out, int64_t n);
int or_conv2d_forward(const double* x, int64_t B, int64_t C, int64_t H, int64_t W, const double* k,
                      int64_t F, int64_t R, int64_t S, int stride, int pad, int floor_mode,
                      double* y);
int or_conv2d_backward(const double* x, int64_t B, int64_t C, int64_t H, int64_t W,
                       const double* k, int64_t F, int64_t R, int64_t S, int stride, int pad,
                       int floor_mode, const double* gy, double* gx, double* gk);
void or_matmul(const double* a, const double* b, double* c, int64_t m, int64_t p, int64_t n);
void or_matmul_tn(const double* a, const double* b, double* c, int64_t p, int64_t m, int64_t n);
void or_matmul_nt(const double* a, const double* b, double* c, int64_t m, int64_t p, int64_t n);
int or_logistic_xent(const double* z, const double* t, int64_t B, int64_t L, double* grad,
                     double* loss);
void or_momentum_update(double* w, double* delta, const double* g, int64_t n, double lr,
                        double momentum, double weight_decay);
void or_momentum_update_f32(float* w, float* delta, const float* g, int64_t n, double lr,
                            double momentum, double weight_decay);
void or_maxpool_forward(const double* x, int64_t B, int64_t C, int64_t H, int64_t W, int k, int s,
                        double* y, int32_t* idx);
void or_maxpool_backward(const double* gy, const int32_t* idx, int64_t B, int64_t C, int64_t H,
                         int64_t W, int k, int s, double* gx);
void or_lrn_forward(const double* a, int64_t B, int64_t C, int64_t HW, int n, double alpha,
                    double beta, double k, double* b, double* scale);
void or_lrn_backward(const double* a, const double* scale, const double* gb, int64_t B, int64_t C,
                     int64_t HW, int n, double alpha, double beta, double* ga);

#ifdef __cplusplus
}
#endif

#endif
