// C ABI: error state, host helpers, and kernel-level entry points.
#include <cstring>
#include <string>

#include "errors.hpp"
#include "gemm.cuh"
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
  return gemm_plan(d->math, a, b, d->M, d->N, d->K, e, d->splits, d->ws, d->bn);
}

HP_API int hp_kernel_gemm_splits(const hp_gemm_desc* d) {
  return gemm_choose_splits(d->math, d->M, d->N, d->K, d->bn);
}

HP_API int hp_kernel_gemm(const hp_gemm_desc* d, void* stream) {
  return guarded([&] {
    GemmPlan p = plan_from_desc(d);
    gemm_launch(p, static_cast<cudaStream_t>(stream));
    HP_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
