// C ABI: error state, host helpers, and kernel-level entry points.
#include <cstring>
#include <string>

#include "datagen.hpp"
#include "errors.hpp"
#include "gemm.cuh"
#include "kernels.cuh"
#include "hpsim_b200.h"
#include "rng.hpp"

namespace hp {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
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

using namespace hp;

extern "C" {

HP_API const char* hp_last_error(void) { return g_last_error.c_str(); }
HP_API const char* hp_version(void) { return "hpsim_b200 0.1 (sm_100a)"; }

HP_API void hp_shard_range(int64_t total, int parts, int idx, int64_t* begin, int64_t* end) {
  const int64_t base = total / parts;
  *begin = base * idx;
  *end = idx == parts - 1 ? total : *begin + base;
}

HP_API void hp_gaussian_fill(uint64_t seed, double* out, int64_t n) {
  GaussianSampler g(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = g.next();
}

HP_API void hp_gaussian_fill_f32(uint64_t seed, double scale, float* out, int64_t n) {
  GaussianSampler g(seed);
  const double s = scale;
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<float>(s * g.next());
}

static GemmPlan plan_from_desc(const hp_gemm_desc* d) {
  GemmOperand a, b;
  a.ptr = d->a;
  a.mn_major = d->a_mn;
  a.ld = d->lda;
  b.ptr = d->b;
  b.mn_major = d->b_mn;
  b.ld = d->ldb;
  Epi e;
  e.c = d->c;
  e.ldc = d->ldc;
  e.c_type = d->c_type;
  e.c_trans = d->c_trans;
  e.alpha = d->alpha;
  e.beta = d->beta;
  e.bias = d->bias;
  e.bias_mode = d->bias_mode;
  e.relu = d->relu;
  e.mask = d->mask;
  e.ldmask = d->ldmask;
  e.mask_type = d->mask_type;
  e.mask_trans = d->mask_trans;
  return gemm_plan(d->math, a, b, d->M, d->N, d->K, e, d->splits, d->ws, d->bn, d->cta2);
}

HP_API void hp_debug_gemm_force(int cta2, int bn) { gemm_force_config(cta2, bn); }
HP_API void hp_debug_gemm_flags(int flags) { gemm_debug_flags(flags); }

HP_API int hp_kernel_gemm_splits(const hp_gemm_desc* d) {
  int splits = 1;
  const int rc = guarded([&] {
    hp_gemm_desc q = *d;
    if (q.ws == nullptr) q.ws = reinterpret_cast<float*>(256);  // sizing only; never dereferenced
    splits = plan_from_desc(&q).splits;
  });
  return rc == HP_OK ? splits : -rc;
}

HP_API int hp_kernel_gemm(const hp_gemm_desc* d, void* stream) {
  return guarded([&] {
    GemmPlan p = plan_from_desc(d);
    gemm_launch(p, static_cast<cudaStream_t>(stream));
    HP_CUDA(cudaGetLastError());
  });
}


static int conv_out(int in, int k, int s, int p) { return (in + 2 * p - k) / s + 1; }

HP_API int hp_kernel_conv_fprop(int math, const void* x, int B, int H, int W, int C, const void* w,
                                int F, int R, int S, int stride, int pad, float* y, void* stream) {
  return guarded([&] {
    GemmOperand a, b;
    a.ptr = x;
    a.conv = Im2col{1, B, H, W, C, R, S, stride, pad, conv_out(H, R, stride, pad), conv_out(W, S, stride, pad)};
    b.ptr = w;
    b.ld = static_cast<long long>(R) * S * C;
    Epi e;
    e.c = y;
    e.ldc = F;
    const int M = B * a.conv.OH * a.conv.OW;
    GemmPlan p = gemm_plan(math, a, b, M, F, R * S * C, e, 1, nullptr, 0);
    gemm_launch(p, static_cast<cudaStream_t>(stream));
    HP_CUDA(cudaGetLastError());
  });
}

HP_API int hp_kernel_conv_wgrad(int math, const void* x, int B, int H, int W, int C, const void* dy,
                                int F, int R, int S, int stride, int pad, float* dw, float* ws,
                                int64_t ws_floats, void* stream) {
  return guarded([&] {
    const int OH = conv_out(H, R, stride, pad), OW = conv_out(W, S, stride, pad);
    GemmOperand a, b;
    a.ptr = dy;
    a.mn_major = 1;
    a.ld = F;
    b.ptr = x;
    b.mn_major = 1;
    b.conv = Im2col{1, B, H, W, C, R, S, stride, pad, OH, OW};
    Epi e;
    e.c = dw;
    e.ldc = static_cast<long long>(R) * S * C;
    const int N = R * S * C, K = B * OH * OW;
    int splits = gemm_choose_splits(math, F, N, K);
    if (static_cast<int64_t>(splits) * F * N > ws_floats) splits = 1;
    GemmPlan p = gemm_plan(math, a, b, F, N, K, e, splits, ws, 0);
    gemm_launch(p, static_cast<cudaStream_t>(stream));
    HP_CUDA(cudaGetLastError());
  });
}

HP_API int hp_kernel_conv_dgrad(int math, const void* dy, int B, int OH, int OW, int F,
                                const void* wrot, int C, int R, int S, int pad, float* dx,
                                void* stream) {
  return guarded([&] {
    const int H = OH + R - 1 - 2 * pad, W = OW + S - 1 - 2 * pad;
    GemmOperand a, b;
    a.ptr = dy;
    a.conv = Im2col{1, B, OH, OW, F, R, S, 1, R - 1 - pad, H, W};
    b.ptr = wrot;
    b.ld = static_cast<long long>(R) * S * F;
    Epi e;
    e.c = dx;
    e.ldc = C;
    GemmPlan p = gemm_plan(math, a, b, B * H * W, C, R * S * F, e, 1, nullptr, 0);
    gemm_launch(p, static_cast<cudaStream_t>(stream));
    HP_CUDA(cudaGetLastError());
  });
}

/* Flat-shift implicit-GEMM conv (bf16, see conv_shift_plan): y[rows][N] (fp32,
 * every row position; border rows hold garbage) = sum over taps of
 * x[row + r*wq + s][C] . w[N][(r*S+s)*C + c]. Returns HP_ERR_CONFIG when the
 * shape is unsupported. boff_mode: descriptor base-offset convention (dev). */
HP_API int hp_kernel_conv_shift(const void* x, int64_t rows, int C, int R, int S, int wq, const void* w, int N,
                                float* y, int boff_mode, void* stream) {
  return guarded([&] {
    Epi e;
    e.c = y;
    e.ldc = N;
    GemmPlan p = conv_shift_plan(x, rows, C, R, S, wq, w, static_cast<long long>(R) * S * C, N, e, boff_mode);
    if (!p.valid) config_error("conv_shift: unsupported shape");
    gemm_launch(p, static_cast<cudaStream_t>(stream));
    HP_CUDA(cudaGetLastError());
  });
}

// Fused LRN + max-pool of one conv stage, exactly the launch the step makes
// (kernels.cu launch_lrn_pool_* / launch_maxpool_*_w); lrn_size 0: pool only.
HP_API int hp_kernel_lrn_pool_fwd(int math, const void* a, int B, int H, int W, int C, int lrn_size, float alpha,
                                  float beta, float k, int pk, int ps, void* y, uint8_t* widx, void* stream) {
  return guarded([&] {
    if (!a || !y || !widx) usage_error("lrn_pool_fwd: null pointer");
    if (pk < 1 || ps < 1 || pk > 16 || H < pk || W < pk) config_error("lrn_pool_fwd: bad pool window");
    const int PH = (H - pk) / ps + 1, PW = (W - pk) / ps + 1;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto go = [&](auto tag) {
      using T = decltype(tag);
      if (lrn_size > 0)
        launch_lrn_pool_fwd<T>(static_cast<const T*>(a), static_cast<T*>(y), widx, B, H, W, C, lrn_size, alpha, beta,
                               k, pk, ps, PH, PW, st);
      else
        launch_maxpool_fwd_w<T>(static_cast<const T*>(a), static_cast<T*>(y), widx, B, H, W, C, pk, ps, PH, PW, st);
    };
    if (math == HP_MATH_BF16) go(bf16{});
    else go(float{});
    HP_CUDA(cudaGetLastError());
  });
}

HP_API int hp_kernel_lrn_pool_bwd(int math, const float* gy, const uint8_t* widx, const void* a, int B, int H, int W,
                                  int C, int lrn_size, float alpha, float beta, float k, int pk, int ps, int relu_mask,
                                  void* dz, float* bias_grad, void* stream) {
  return guarded([&] {
    if (!gy || !widx || !a || !dz) usage_error("lrn_pool_bwd: null pointer");
    if (pk < 1 || ps < 1 || pk > 16 || H < pk || W < pk) config_error("lrn_pool_bwd: bad pool window");
    const int PH = (H - pk) / ps + 1, PW = (W - pk) / ps + 1;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto go = [&](auto tag) {
      using T = decltype(tag);
      if (lrn_size > 0) {
        launch_lrn_pool_bwd<T>(gy, widx, static_cast<const T*>(a), static_cast<T*>(dz), B, H, W, C, lrn_size, alpha,
                               beta, k, pk, ps, PH, PW, relu_mask, st);
        if (bias_grad) {  // the step's bias gradient: channel sums of the stored dz (model.cpp:184-202)
          float* ws = nullptr;
          const long long M = static_cast<long long>(B) * H * W;
          HP_CUDA(cudaMalloc(&ws, sizeof(float) * colsum_ws_floats(M, C)));
          launch_colsum<T>(static_cast<const T*>(dz), M, C, C, bias_grad, ws, st);
          HP_CUDA(cudaStreamSynchronize(st));
          HP_CUDA(cudaFree(ws));
        }
      } else {
        launch_maxpool_bwd_w<T, T>(gy, widx, static_cast<T*>(dz), relu_mask ? static_cast<const T*>(a) : nullptr, B,
                                   H, W, C, pk, ps, PH, PW, st);
      }
    };
    if (math == HP_MATH_BF16) go(bf16{});
    else go(float{});
    HP_CUDA(cudaGetLastError());
  });
}

// The step's momentum SGD kernel on one fp32 tensor (optimizer.cpp:19-31).
HP_API int hp_kernel_sgd(float* w, float* mom, const float* g, int64_t n, double lr, double momentum,
                         double weight_decay, float gscale, int has_gscale, void* bf16_copy, void* stream) {
  return guarded([&] {
    if (!w || !mom || !g) usage_error("sgd: null pointer");
    SgdTensor t{};
    t.w = w;
    t.mom = mom;
    t.g = g;
    t.copy = bf16_copy;
    t.n = n;
    t.gscale = gscale;
    t.has_gscale = has_gscale;
    launch_sgd(&t, 1, bf16_copy ? 1 : 0, lr, momentum, weight_decay, static_cast<cudaStream_t>(stream));
    HP_CUDA(cudaGetLastError());
  });
}

}  // extern "C"

HP_API int hp_data_generate(const hp_dataset_spec* spec, int64_t first, int64_t count, float* inputs,
                            float* targets, int mem_kind, void* stream) {
  return guarded([&] {
    if (!spec) usage_error("data_generate: null spec");
    datagen_validate(*spec);
    if (count > 0 && (!inputs || !targets)) usage_error("data_generate: null output");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (mem_kind == HP_MEM_DEVICE) {
      datagen_launch(*spec, first, count, inputs, targets, st);
      return;
    }
    if (mem_kind != HP_MEM_HOST) usage_error("data_generate: bad mem_kind");
    datagen_check_range(*spec, first, count);
    if (count == 0) return;
    const size_t nx = static_cast<size_t>(count) * spec->channels * spec->height * spec->width;
    const size_t nt = static_cast<size_t>(count) * spec->num_classes;
    float* d = nullptr;
    HP_CUDA(cudaMalloc(&d, (nx + nt) * sizeof(float)));
    try {
      datagen_launch(*spec, first, count, d, d + nx, st);
      HP_CUDA(cudaMemcpyAsync(inputs, d, nx * sizeof(float), cudaMemcpyDeviceToHost, st));
      HP_CUDA(cudaMemcpyAsync(targets, d + nx, nt * sizeof(float), cudaMemcpyDeviceToHost, st));
      HP_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cudaFree(d);
      throw;
    }
    HP_CUDA(cudaFree(d));
  });
}

HP_API int hp_data_class_of(const hp_dataset_spec* spec, int64_t index, int64_t* cls) {
  return guarded([&] {
    if (!spec || !cls) usage_error("data_class_of: null argument");
    *cls = datagen_class_of(*spec, index);
  });
}
