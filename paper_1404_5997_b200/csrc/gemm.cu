// tcgen05 / TMEM / TMA GEMM for sm_100a. See gemm.cuh for the contract.
//
// One CTA computes one 128 x BN output tile over a contiguous range of
// k-tiles (split-K when the tile grid cannot fill 148 SMs). Warp roles:
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      TMEM allocator + MMA issuer (one lane issues tcgen05.mma)
//   warps 2..5  epilogue: tcgen05.ld -> fused elementwise -> global stores
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "gemm.cuh"
#include "ptx.cuh"

namespace hp {

namespace {

constexpr int kBM = 128;
constexpr uint32_t kMaxDynSmem = 232448;  // 227 KB
constexpr uint32_t kEpiSmemBytes = 4u * 32u * 36u * 4u;  // staged epilogue tiles (see epi_chunk)

__host__ __device__ constexpr uint32_t stage_bytes(int bn, int math) {
  return (kBM * 128u + static_cast<uint32_t>(bn) * 128u) * (math == kMathF32x3 ? 2u : 1u);
}
#ifndef HP_GEMM_CAP
#define HP_GEMM_CAP 6
#endif
__host__ __device__ constexpr int num_stages(int bn, int math) {
  return static_cast<int>((kMaxDynSmem - 2048u - kEpiSmemBytes) / stage_bytes(bn, math)) > HP_GEMM_CAP
             ? HP_GEMM_CAP
             : static_cast<int>((kMaxDynSmem - 2048u - kEpiSmemBytes) / stage_bytes(bn, math));
}
// TMEM columns of one accumulator (power of two >= 32); two are allocated.
__host__ __device__ constexpr uint32_t tmem_cols(int bn) {
  return bn <= 32 ? 32u : bn <= 64 ? 64u : bn <= 128 ? 128u : 256u;
}

__device__ __forceinline__ float load_as_float(const void* p, long long off, int type) {
  if (type == kBF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[off]);
  return reinterpret_cast<const float*>(p)[off];
}

__device__ __forceinline__ float sgd_apply(const Epi& e, long long off, float g) {
  if (e.sgd_has_gscale) g = __fmul_rn(g, e.sgd_gscale);
  const float w = e.sgd_w[off];
  float d = __fmul_rn(e.sgd_m[off], e.sgd_mu);
  d = __fadd_rn(d, __fmul_rn(e.sgd_s1, g));
  d = __fadd_rn(d, __fmul_rn(e.sgd_s2, w));
  const float nw = __fadd_rn(w, d);
  e.sgd_m[off] = d;
  e.sgd_w[off] = nw;
  if (e.sgd_copy) reinterpret_cast<__nv_bfloat16*>(e.sgd_copy)[off] = __float2bfloat16_rn(nw);
  return nw;
}

// Output column of GEMM column n under e.cols (Im2col::halo order).
__device__ __forceinline__ int map_col(const ColMap& c, int n) {
  if (!c.enabled) return n;
  const int blk = n >> 6, c_lo = n & 63;
  const int s = blk % c.S, rcb = blk / c.S;
  const int cbs = c.C >> 6, r = rcb / cbs, cb = rcb - r * cbs;
  return (r * c.S + s) * c.C + cb * 64 + c_lo;
}

// Output row of GEMM row m under e.rows (-1: not stored).
__device__ __forceinline__ int map_row(const RowMap& r, int m) {
  if (!r.enabled) return m;
  const int plane = r.sH * r.sW;
  const int b = m / plane, rem = m - b * plane;
  const int y = rem / r.sW, x = rem - y * r.sW;
  if (y >= r.vH || x >= r.vW) return -1;
  return (b * r.dH + y + r.dp) * r.dW + x + r.dp;
}

__device__ __forceinline__ void epi_elem(const Epi& e, int m, int n, float v) {
  const int gm = m;  // GEMM row (per-row bias)
  n = map_col(e.cols, n);
  if (e.rblk.enabled) {
    const int b0 = e.rblk.blk[m >> 6];
    if (b0 < 0) return;
    m = b0 + (m & 63);
  }
  if (e.rows.enabled) {
    m = map_row(e.rows, m);
    if (m < 0) return;
  }
  const long long off = e.c_trans ? static_cast<long long>(n) * e.ldc + m
                                  : static_cast<long long>(m) * e.ldc + n;
  v *= e.alpha;
  if (e.beta) v += reinterpret_cast<const float*>(e.c)[off];
  if (e.sgd_w) {
    sgd_apply(e, off, v);
    return;
  }
  if (e.bias_mode == 1) v += e.bias[gm];
  if (e.bias_mode == 2) v += e.bias[n];
  if (e.relu) v = v > 0.f ? v : 0.f;
  if (e.mask) {
    const long long mo = e.mask_trans ? static_cast<long long>(n) * e.ldmask + m
                                      : static_cast<long long>(m) * e.ldmask + n;
    if (!(load_as_float(e.mask, mo, e.mask_type) > 0.f)) v = 0.f;
  }
  if (e.c_type == kBF16) {
    reinterpret_cast<__nv_bfloat16*>(e.c)[off] = __float2bfloat16_rn(v);
  } else {
    reinterpret_cast<float*>(e.c)[off] = v;
  }
}

// 256-bit global accesses (sm_100): one request per 32 contiguous bytes of a
// row -- the row-per-thread epilogue's stores touch a different line per lane,
// so request count, not bytes, is what they cost.
__device__ __forceinline__ void st256(void* p, const uint32_t (&u)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(u[0]), "r"(u[1]),
               "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7])
               : "memory");
}
__device__ __forceinline__ void ld256(const void* p, uint32_t (&u)[8]) {
  asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
               : "l"(p));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// The row-per-thread vector path applies (32 contiguous outputs of one row).
__device__ __forceinline__ bool epi_row_vec(const GemmArgs& a, int n0) {
  const Epi& e = a.epi;
  return !e.c_trans && n0 + 32 <= a.N && (e.c_type == kF32 ? (e.ldc & 3) == 0 : (e.ldc & 7) == 0) &&
         (!e.sgd_w || ((e.ldc & 7) == 0 && e.c_type == kF32)) && (!e.beta || e.c_type == kF32) &&
         (!e.mask ||
          (e.mask_trans == 0 && (e.mask_type == kF32 ? (e.ldmask & 3) == 0 : (e.ldmask & 7) == 0)));
}

// bf16 ReLU-mask words of one row's 32 columns, loaded a chunk ahead so the
// load latency hides behind the previous chunk's epilogue.
struct MaskPre {
  uint4 v[4];
  bool ok = false;
};
__device__ __forceinline__ void epi_mask_load(const GemmArgs& a, int mo, int n0, MaskPre& p) {
  p.ok = false;
  const Epi& e = a.epi;
  if (!e.mask || e.mask_type != kBF16 || a.raw_partial || mo < 0 || (a.dbg & 16) || !epi_row_vec(a, n0)) return;
  const __nv_bfloat16* mp = reinterpret_cast<const __nv_bfloat16*>(e.mask) + static_cast<long long>(mo) * e.ldmask + n0;
  if ((reinterpret_cast<uintptr_t>(mp) & 31) == 0) {
    uint32_t u[8];
    ld256(mp, u);
    p.v[0] = make_uint4(u[0], u[1], u[2], u[3]);
    p.v[1] = make_uint4(u[4], u[5], u[6], u[7]);
    ld256(mp + 16, u);
    p.v[2] = make_uint4(u[0], u[1], u[2], u[3]);
    p.v[3] = make_uint4(u[4], u[5], u[6], u[7]);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) p.v[i] = reinterpret_cast<const uint4*>(mp)[i];
  }
  p.ok = true;
}

// Epilogue for 32 consecutive columns [n0, n0+32) of row m.
// mo: the output row of GEMM row m under the epilogue RowMap (-1: dropped).
__device__ __forceinline__ void epi_row32(const GemmArgs& a, int m, int n0, int split,
                                          const float (&v)[32], int mo, const float* sbias = nullptr,
                                          const MaskPre* mpre = nullptr) {
  if (m >= a.M) return;
  if (a.raw_partial) {
    float* dst = a.ws + static_cast<long long>(split) * a.M * a.N +
                 static_cast<long long>(m) * a.N;
    if (n0 + 32 <= a.N && (reinterpret_cast<uintptr_t>(dst + n0) & 31) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint32_t u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = __float_as_uint(v[i + j]);
        st256(dst + n0 + i, u);
      }
    } else if (n0 + 32 <= a.N && (a.N & 3) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(dst + n0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (n0 + i < a.N) dst[n0 + i] = v[i];
    }
    return;
  }
  const Epi& e = a.epi;
  // Vector path: 32 contiguous outputs of row m (bias/ReLU/alpha/beta/mask fused).
  if (mo < 0) return;
  const bool vec = epi_row_vec(a, n0);
  if (vec) {
    float x[32];
    const float bm = e.bias_mode == 1 ? e.bias[m] : 0.f;
    if (e.alpha != 1.f) {  // (x * 1 == x exactly: skip 32 multiplies per chunk on the common path)
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = v[i] * e.alpha;
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = v[i];
    }
    const long long off = static_cast<long long>(mo) * e.ldc + n0;
    if (e.beta) {
      const float4* old = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.c) + off);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 o = old[i];
        x[4 * i] += o.x;
        x[4 * i + 1] += o.y;
        x[4 * i + 2] += o.z;
        x[4 * i + 3] += o.w;
      }
    }
    if (e.sgd_w) {
      float* wp = e.sgd_w + off;
      float* mp = e.sgd_m + off;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 w4 = reinterpret_cast<const float4*>(wp)[i];
        float4 m4 = reinterpret_cast<const float4*>(mp)[i];
        float* wv = reinterpret_cast<float*>(&w4);
        float* mv = reinterpret_cast<float*>(&m4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float g = x[4 * i + j];
          if (e.sgd_has_gscale) g = __fmul_rn(g, e.sgd_gscale);
          float d = __fmul_rn(mv[j], e.sgd_mu);
          d = __fadd_rn(d, __fmul_rn(e.sgd_s1, g));
          d = __fadd_rn(d, __fmul_rn(e.sgd_s2, wv[j]));
          mv[j] = d;
          wv[j] = __fadd_rn(wv[j], d);
          x[4 * i + j] = wv[j];
        }
        reinterpret_cast<float4*>(wp)[i] = w4;
        reinterpret_cast<float4*>(mp)[i] = m4;
      }
      if (e.sgd_copy) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.sgd_copy) + off);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __align__(16) __nv_bfloat16 t[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) t[j] = __float2bfloat16_rn(x[8 * i + j]);
          dst[i] = *reinterpret_cast<const uint4*>(t);
        }
      }
      return;
    }
    if (e.bias_mode == 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] += bm;
    } else if (e.bias_mode == 2 && !(a.dbg & 4)) {  // dbg 4: skip the bias loads (dev)
      const float4* bb = reinterpret_cast<const float4*>((sbias ? sbias : e.bias) + n0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 o = bb[i];
        x[4 * i] += o.x;
        x[4 * i + 1] += o.y;
        x[4 * i + 2] += o.z;
        x[4 * i + 3] += o.w;
      }
    }
    if (e.relu) {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = x[i] > 0.f ? x[i] : 0.f;
    }
    if (e.mask && !(a.dbg & 16)) {  // dbg 16: skip the mask loads (dev)
      const long long mko = static_cast<long long>(mo) * e.ldmask + n0;
      if (e.mask_type == kBF16) {
        const uint4* mp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.mask) + mko);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 u = (mpre && mpre->ok) ? mpre->v[i] : mp[i];
          const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (!(__bfloat162float(h[j]) > 0.f)) x[8 * i + j] = 0.f;
        }
      } else {
        const float4* mp = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.mask) + mko);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 o = mp[i];
          if (!(o.x > 0.f)) x[4 * i] = 0.f;
          if (!(o.y > 0.f)) x[4 * i + 1] = 0.f;
          if (!(o.z > 0.f)) x[4 * i + 2] = 0.f;
          if (!(o.w > 0.f)) x[4 * i + 3] = 0.f;
        }
      }
    }
    if (a.dbg & 8) {  // dev: skip the stores (keep the values live)
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += x[i];
      if (acc == 12345.678f) reinterpret_cast<float*>(e.c)[off] = acc;
    } else if (e.c_type == kF32) {
      float* dst = reinterpret_cast<float*>(e.c) + off;
      if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t u[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) u[j] = __float_as_uint(x[i + j]);
          st256(dst + i, u);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          reinterpret_cast<float4*>(dst)[i] = make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
      }
    } else {
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(e.c) + off;
      if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 16) {
          uint32_t u[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) u[j] = pack_bf16x2(x[i + 2 * j], x[i + 2 * j + 1]);
          st256(dst + i, u);
        }
      } else {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __align__(16) __nv_bfloat16 t[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) t[j] = __float2bfloat16_rn(x[8 * i + j]);
          d4[i] = *reinterpret_cast<const uint4*>(t);
        }
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (n0 + i < a.N) epi_elem(e, m, n0 + i, v[i]);
  }
}

// ---------------------------------------------------------------- staged epilogue
// tcgen05.ld hands each thread one accumulator ROW; stores straight from that
// layout put 32 different rows (32 cache lines) behind every warp access.
// Instead each epilogue warp transposes its 32x32 fp32 chunk through a padded
// smem tile (row stride 36 floats: float4 writes and reads are bank-conflict
// free) so that 8 consecutive lanes cover 32 consecutive columns of one row:
// every global access of the epilogue (beta read, mask, SGD w/m read+write,
// output) is then a full 128-byte row segment. The loads of all 8 row groups
// are issued before any store so the memory-bound epilogues (FC wgrad with the
// fused SGD update) keep 16+ accesses in flight per thread.
constexpr int kEpiLd = 36;                               // floats per staged row
static_assert(kEpiSmemBytes == 4u * 32u * kEpiLd * 4u, "epilogue tile size");

__device__ __forceinline__ bool epi_vec_ok(const GemmArgs& a) {
  if (a.raw_partial) return (a.N & 3) == 0;
  const Epi& e = a.epi;
  if (e.c_trans || e.mask_trans) return false;
  if (e.ldc & 3) return false;
  if (e.beta && e.c_type != kF32) return false;
  if (e.sgd_w && e.c_type != kF32) return false;
  if (e.mask && (e.ldmask & 3)) return false;
  return true;
}

__device__ __forceinline__ float4 ld_bf16x4(const void* p, long long off) {
  const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(p) + off);
  const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  const float2 a = __bfloat1622float2(lo), b = __bfloat1622float2(hi);
  return make_float4(a.x, a.y, b.x, b.y);
}

#ifndef HP_SGD_STREAMING
#define HP_SGD_STREAMING 1
#endif
#if HP_SGD_STREAMING
#define SGD_LD(p) __ldcs(p)
#define SGD_ST(p, v) __stcs(p, v)
#else
#define SGD_LD(p) (*(p))
#define SGD_ST(p, v) (*(p) = (v))
#endif
__device__ __forceinline__ void st_bf16x4_cs(void* p, long long off, float4 x) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y);
  __nv_bfloat162 hi = __floats2bfloat162_rn(x.z, x.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  SGD_ST(reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p) + off), u);
}
__device__ __forceinline__ void st_bf16x4(void* p, long long off, float4 x) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y);
  __nv_bfloat162 hi = __floats2bfloat162_rn(x.z, x.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p) + off) = u;
}

__device__ __forceinline__ float f4get(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ void f4set(float4& v, int j, float x) {
  if (j == 0) v.x = x;
  else if (j == 1) v.y = x;
  else if (j == 2) v.z = x;
  else v.w = x;
}

__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
               : "memory");
  return v;
}

// Direct (row-per-thread) epilogues with per-column bias read it from smem:
// every lane needs the same 32 values per chunk, and a global load there is a
// full L2 round trip on the epilogue's critical path (measured: ~1/8 of conv
// fprop time). The epilogue warps (threads 64..191) copy bias[0, N) into the
// staging area the direct path does not use; returns it, or nullptr.
__device__ __forceinline__ const float* epi_stage_bias(const GemmArgs& a, float* base) {
  const bool direct = !(a.dbg & 2) && !a.raw_partial && !a.epi.beta && !a.epi.sgd_w;
  if (!direct || a.epi.bias_mode != 2 || a.epi.c_trans || a.N > static_cast<int>(kEpiSmemBytes / 4)) return nullptr;
  for (int i = static_cast<int>(threadIdx.x) - 64; i < a.N; i += 128) base[i] = a.epi.bias[i];
  asm volatile("bar.sync 1, 128;" ::: "memory");
  return base;
}

// Output rows of the 8 GEMM rows m0 + 4i + (lane >> 3) a thread stores in
// epi_chunk (-1: past M or dropped by the RowMap). Depends only on the tile
// and the thread, so the kernels compute it once per tile.
__device__ __forceinline__ bool epi_direct(const GemmArgs& a) {
  return !(a.dbg & 2) && (a.raw_partial || (!a.epi.beta && !a.epi.sgd_w));
}
__device__ __forceinline__ void epi_rows(const GemmArgs& a, int m0, int (&mrow)[8], int& mself) {
  const int ms = m0 + (threadIdx.x & 31);
  mself = ms < a.M ? map_row(a.epi.rows, ms) : -1;
  // the 8 staged-layout rows only where epi_chunk takes the staged path: the
  // direct (row-per-thread) epilogues use mself alone, and the RowMap's
  // divisions were ~40% of the conv fprop epilogue's instructions
  if (epi_direct(a) || !epi_vec_ok(a)) return;
  const int rsub = (threadIdx.x & 31) >> 3;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + 4 * i + rsub;
    mrow[i] = m < a.M ? map_row(a.epi.rows, m) : -1;
  }
}

// Epilogue of one warp's 32 rows [m0, m0+32) x 32 columns [n0, n0+32).
// All 32 lanes must call it (warp-synchronous); `stg` is the warp's tile.
__device__ __forceinline__ void epi_chunk(const GemmArgs& a, int m0, int n0, int split, const float (&v)[32],
                                          float* stg, const int (&mrow)[8], int mself,
                                          const float* sbias = nullptr, const MaskPre* mpre = nullptr) {
  const int lane = threadIdx.x & 31;
  if (a.dbg & 1) return;  // dev: mainloop-only timing
  // Store-only epilogues (no beta / mask / SGD reads) and transposed outputs
  // write straight from the row-per-thread layout: 32 contiguous outputs per
  // thread, no smem round trip (the staged transpose costs shared-memory
  // bandwidth the MMAs need; it pays only when the epilogue also reads HBM).
  if (epi_direct(a) || !epi_vec_ok(a)) {
    epi_row32(a, m0 + lane, n0, split, v, mself, sbias, mpre);
    return;
  }
  const uint32_t sbase = smem_u32(stg);
  __syncwarp();  // the previous chunk's reads of the tile are done
#pragma unroll
  for (int i = 0; i < 8; ++i)
    sts128(sbase + (lane * kEpiLd + 4 * i) * 4, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
  __syncwarp();
  const int rsub = lane >> 3, cq = (lane & 7) * 4;
  const int n = n0 + cq;
  float4 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = lds128(sbase + ((4 * i + rsub) * kEpiLd + cq) * 4);
  // (the next chunk's entry __syncwarp orders these reads before its writes)
  const bool nfull = n + 4 <= a.N;
  if (a.raw_partial) {
    float* dst = a.ws + static_cast<long long>(split) * a.M * a.N;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + 4 * i + rsub;
      if (m >= a.M || n >= a.N) continue;
      float* p = dst + static_cast<long long>(m) * a.N + n;
      if (nfull) {
        *reinterpret_cast<float4*>(p) = x[i];
      } else {
        for (int j = 0; j < 4 && n + j < a.N; ++j) p[j] = stg[(4 * i + rsub) * kEpiLd + cq + j];
      }
    }
    return;
  }
  const Epi& e = a.epi;
  if (!nfull) {  // ragged right edge: scalar, straight from the (warp-private) staged tile (epi_elem maps rows)
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + 4 * i + rsub;
      if (m >= a.M) continue;
      for (int j = 0; j < 4 && n + j < a.N; ++j) epi_elem(e, m, n + j, stg[(4 * i + rsub) * kEpiLd + cq + j]);
    }
    return;
  }
  // full 4-wide columns; mrow[i]: output row of GEMM row m0 + 4i + rsub (-1:
  // past M or dropped by the row map); bias_mode 1 uses the GEMM row.
  float4 aux[8], aux2[8];
  if (e.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i].x *= e.alpha;
      x[i].y *= e.alpha;
      x[i].z *= e.alpha;
      x[i].w *= e.alpha;
    }
  }
  if (e.beta) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = mrow[i];
      aux[i] = m >= 0 ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.c) +
                                                         static_cast<long long>(m) * e.ldc + n)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i].x += aux[i].x;
      x[i].y += aux[i].y;
      x[i].z += aux[i].z;
      x[i].w += aux[i].w;
    }
  }
  if (e.sgd_w) {
    // fused momentum SGD (optimizer.cpp:19-31): four rounded passes, no FMA
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = mrow[i];
      const long long off = static_cast<long long>(m) * e.ldc + n;
      if (m >= 0) {  // streamed once: evict-first (leave L2 to the concurrent GEMMs)
        aux[i] = SGD_LD(reinterpret_cast<const float4*>(e.sgd_w + off));
        aux2[i] = SGD_LD(reinterpret_cast<const float4*>(e.sgd_m + off));
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = mrow[i];
      if (m < 0) continue;
      const long long off = static_cast<long long>(m) * e.ldc + n;
      float4 w4 = aux[i], m4 = aux2[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float g = f4get(x[i], j);
        if (e.sgd_has_gscale) g = __fmul_rn(g, e.sgd_gscale);
        float d = __fmul_rn(f4get(m4, j), e.sgd_mu);
        d = __fadd_rn(d, __fmul_rn(e.sgd_s1, g));
        d = __fadd_rn(d, __fmul_rn(e.sgd_s2, f4get(w4, j)));
        f4set(m4, j, d);
        f4set(w4, j, __fadd_rn(f4get(w4, j), d));
      }
      SGD_ST(reinterpret_cast<float4*>(e.sgd_w + off), w4);
      SGD_ST(reinterpret_cast<float4*>(e.sgd_m + off), m4);
      if (e.sgd_copy) st_bf16x4_cs(e.sgd_copy, off, w4);
    }
    return;
  }
  if (e.bias_mode == 2) {
    const float4 bb = *reinterpret_cast<const float4*>(e.bias + n);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i].x += bb.x;
      x[i].y += bb.y;
      x[i].z += bb.z;
      x[i].w += bb.w;
    }
  } else if (e.bias_mode == 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + 4 * i + rsub;
      const float bm = m < a.M ? e.bias[m] : 0.f;
      x[i].x += bm;
      x[i].y += bm;
      x[i].z += bm;
      x[i].w += bm;
    }
  }
  if (e.relu) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i].x = x[i].x > 0.f ? x[i].x : 0.f;
      x[i].y = x[i].y > 0.f ? x[i].y : 0.f;
      x[i].z = x[i].z > 0.f ? x[i].z : 0.f;
      x[i].w = x[i].w > 0.f ? x[i].w : 0.f;
    }
  }
  if (e.mask) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = mrow[i];
      if (m < 0) continue;
      const long long mo = static_cast<long long>(m) * e.ldmask + n;
      aux[i] = e.mask_type == kBF16 ? ld_bf16x4(e.mask, mo)
                                    : *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.mask) + mo);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (!(aux[i].x > 0.f)) x[i].x = 0.f;
      if (!(aux[i].y > 0.f)) x[i].y = 0.f;
      if (!(aux[i].z > 0.f)) x[i].z = 0.f;
      if (!(aux[i].w > 0.f)) x[i].w = 0.f;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = mrow[i];
    if (m < 0) continue;
    const long long off = static_cast<long long>(m) * e.ldc + n;
    if (e.c_type == kF32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(e.c) + off) = x[i];
    } else {
      st_bf16x4(e.c, off, x[i]);
    }
  }
}

template <bool TWO>
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int x, int y) {
  if (TWO) {
    tma_load_2d_2sm(dst, tm, bar, x, y);
  } else {
    tma_load_2d(dst, tm, bar, x, y);
  }
}
template <bool TWO>
__device__ __forceinline__ void tma_im2col(void* dst, const CUtensorMap* tm, uint64_t* bar, int c, int w,
                                           int h, int n, uint16_t s, uint16_t r) {
  if (TWO) {
    tma_load_im2col_4d_2sm(dst, tm, bar, c, w, h, n, s, r);
  } else {
    tma_load_im2col_4d(dst, tm, bar, c, w, h, n, s, r);
  }
}

template <bool TWO, int BK, int ATOM>
__device__ __forceinline__ void load_tile_t(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar,
                                            int mn_major, int row0, int rows, int k0) {
  if (!mn_major) {
    tma2d<TWO>(dst, tm, bar, k0, row0);
  } else {
    for (int a = 0; a < rows / ATOM; ++a) tma2d<TWO>(dst + a * (BK * 128), tm, bar, row0 + a * ATOM, k0);
  }
}

// im2col A tile (fprop / rotated dgrad): 128 consecutive output pixels x one
// 128-byte channel block of filter tap (r, s) for k-tile kt.
template <bool TWO, int ATOM>
__device__ __forceinline__ void load_a_im2col(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar,
                                              const ConvArgs& c, int m0, int kt) {
  const int cblks = c.C / ATOM;
  const int cb = kt % cblks, rs = kt / cblks;
  const int r = rs / c.S, s = rs - r * c.S;
  const int ohw = c.OH * c.OW;
  const int n = m0 / ohw, rem = m0 - n * ohw;
  const int oh = rem / c.OW, ow = rem - oh * c.OW;
  tma_im2col<TWO>(dst, tm, bar, cb * ATOM, c.lo_w + ow * c.stride, c.lo_h + oh * c.stride_h, n,
                  static_cast<uint16_t>(s), static_cast<uint16_t>(r));
}

// im2col B tile (wgrad, MN-major): BK consecutive output pixels (the K
// dimension) x `rows` columns = rows/ATOM channel blocks, each at its own tap.
template <bool TWO, int BK, int ATOM>
__device__ __forceinline__ void load_b_im2col(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar,
                                              const ConvArgs& c, int n0, int rows, int kt) {
  const int ohw = c.OH * c.OW;
  const int p0 = kt * BK;
  const int n = p0 / ohw, rem = p0 - n * ohw;
  const int oh = rem / c.OW, ow = rem - oh * c.OW;
  for (int a = 0; a < rows / ATOM; ++a) {
    const int col = n0 + a * ATOM;
    const int rs = col / c.C, ch = col - rs * c.C;
    const int r = rs / c.S, s = rs - r * c.S;
    tma_im2col<TWO>(dst + a * (BK * 128), tm, bar, ch, c.lo_w + ow * c.stride, c.lo_h + oh * c.stride_h, n,
                    static_cast<uint16_t>(s), static_cast<uint16_t>(r));
  }
}

// Shift-mode MN-major conv operand (wgrad over q-layout x): `rows` columns =
// rows/ATOM channel blocks, each at its own tap, as tiled boxes at shifted rows.
template <bool TWO, int BK, int ATOM>
__device__ __forceinline__ void load_mn_shift(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar, const ConvArgs& c,
                                              int n0, int rows, int kt) {
  for (int a = 0; a < rows / ATOM; ++a) {
    const int col = n0 + a * ATOM;
    const int tap = col / c.C, ch = col - tap * c.C;
    const int r = tap / c.S, s = tap - r * c.S;
    tma2d<TWO>(dst + a * (BK * 128), tm, bar, ch, kt * BK + r * c.wq + s + c.base_off);
  }
}

// Persistent tile loop. Tiles t = blockIdx.x, blockIdx.x + gridDim.x, ... in
// (split, m, n) order with n fastest, so co-resident CTAs share A tiles in L2.
// Two TMEM accumulators: the epilogue of tile i overlaps the MMAs of tile i+1.
// 3xTF32 runs one tile per CTA (its epilogue warps double as tile converters).
struct TileIdx {
  int m0, n0, split, kt0, kt1;
};

template <int BN>
__device__ __forceinline__ TileIdx tile_idx(const GemmArgs& a, int t, int tiles_m, int tiles_n) {
  TileIdx r;
  const int mn = tiles_m * tiles_n;
  r.split = t / mn;
  const int rem = t - r.split * mn;
  const int mb = rem / tiles_n;
  r.m0 = mb * kBM;
  r.n0 = (rem - mb * tiles_n) * BN;
  r.kt0 = r.split * a.k_tiles_per_split;
  r.kt1 = min(a.k_tiles_total, r.kt0 + a.k_tiles_per_split);
  return r;
}

// LIGHT: short-K GEMMs whose epilogue is the work (FC wgrad + fused SGD, K =
// 128): 2 stages, one accumulator, two CTAs per SM -- twice the epilogue warps
// (memory-level parallelism) per SM.
template <int BN, int MATH, bool LIGHT>
#ifndef HP_LIGHT_CTAS
#define HP_LIGHT_CTAS 2  // light kernel CTAs per SM
#endif
#ifndef HP_LIGHT_STAGES
#define HP_LIGHT_STAGES 2
#endif
__global__ void __launch_bounds__(192, LIGHT ? HP_LIGHT_CTAS : 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                const GemmArgs args) {
  constexpr bool SPLIT = MATH == kMathF32x3;
  constexpr int ES = MATH == kMathBF16 ? 2 : 4;
  constexpr int BK = 128 / ES;
  constexpr int UK = 32 / ES;
  constexpr int ATOM = 128 / ES;
  constexpr uint32_t A_BYTES = kBM * 128;
  constexpr uint32_t B_BYTES = BN * 128;
  constexpr uint32_t SB = stage_bytes(BN, MATH);
  constexpr int STAGES = LIGHT ? HP_LIGHT_STAGES : num_stages(BN, MATH);
  constexpr int NACC = (SPLIT || LIGHT) ? 1 : 2;
  constexpr uint32_t ACOLS = tmem_cols(BN);
  constexpr uint32_t TCOLS = ACOLS * NACC;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  uint64_t* conv = empty + STAGES;  // 3xTF32: split done (converter -> MMA)
  uint64_t* tfull = conv + STAGES;  // [NACC]
  uint64_t* tempty = tfull + 2;     // [NACC]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_m = (args.M + kBM - 1) / kBM;
  const int tiles_n = (args.N + BN - 1) / BN;
  const int total = tiles_m * tiles_n * ((args.k_tiles_total + args.k_tiles_per_split - 1) / args.k_tiles_per_split);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 128);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_barrier_init();
    tma_prefetch(&ta);
    tma_prefetch(&tb);
  }
  if (warp == 1) tmem_alloc(tslot, TCOLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();  // predecessor's outputs (our inputs / output buffers) are final

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TileIdx ti = tile_idx<BN>(args, t, tiles_m, tiles_n);
        for (int kt = ti.kt0; kt < ti.kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SB;
          uint8_t* sb = sa + A_BYTES;
          // dev (dbg 32 / 64): skip the B / A loads of odd k-tiles (results garbage) -- is the
          // mainloop bound by operand delivery?
          const bool skip_b = (args.dbg & 32) && (kt & 1), skip_a = (args.dbg & 64) && (kt & 1);
          const uint32_t b_bytes = args.cb.halo ? static_cast<uint32_t>(args.cb.halo_rows) * 128u : B_BYTES;
          const uint32_t a_bytes = args.tp.n > 0 ? static_cast<uint32_t>(args.tp_rows) * 128u : A_BYTES;
          mbar_arrive_expect_tx(&full[stage], (skip_a ? 0u : a_bytes) + (skip_b ? 0u : b_bytes));
          if (skip_a) {
          } else if (args.tp.n > 0) {  // tap-pair A: one box, both atoms (TapPairs)
            const int mt = ti.m0 / kBM;
            tma2d<false>(sa, &ta, &full[stage], args.tp.cb[mt] * ATOM, kt * BK + args.tp.off[mt] + args.ca.base_off);
          } else if (args.ca.enabled && args.a_mn && args.ca.shift) {
            load_mn_shift<false, BK, ATOM>(sa, &ta, &full[stage], args.ca, ti.m0, kBM, kt);
          } else if (args.ca.enabled && args.a_mn) {  // wgrad with im2col(x)^T as A: K = pixels
            load_b_im2col<false, BK, ATOM>(sa, &ta, &full[stage], args.ca, ti.m0, kBM, kt);
          } else if (args.ca.enabled) {
            load_a_im2col<false, ATOM>(sa, &ta, &full[stage], args.ca, ti.m0, kt);
          } else {
            load_tile_t<false, BK, ATOM>(sa, &ta, &full[stage], args.a_mn, ti.m0, kBM, kt * BK);
          }
          if (skip_b) {
          } else if (args.cb.enabled && args.cb.halo) {
            // one box: rows kt*BK + r*wq + base_off .. + halo_rows of channel block cb
            const int grp = ti.n0 / BN;  // = r * (C / 64) + cb (BN = S * 64)
            const int cbs = args.cb.C / ATOM, r = grp / cbs, cb = grp - r * cbs;
            tma2d<false>(sb, &tb, &full[stage], cb * ATOM, kt * BK + r * args.cb.wq + args.cb.base_off);
          } else if (args.cb.enabled && args.cb.shift) {
            load_mn_shift<false, BK, ATOM>(sb, &tb, &full[stage], args.cb, ti.n0, BN, kt);
          } else if (args.cb.enabled) {
            load_b_im2col<false, BK, ATOM>(sb, &tb, &full[stage], args.cb, ti.n0, BN, kt);
          } else {
            load_tile_t<false, BK, ATOM>(sb, &tb, &full[stage], args.b_mn, ti.n0, BN, kt * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();  // all of this CTA's loads are issued: the next kernel may launch
    }
  } else if (warp == 1) {
    {  // whole warp: warp-uniform loop (uniform-register descriptors), one elected issuer
      constexpr uint32_t fmt = MATH == kMathBF16 ? 1u : 2u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                             (static_cast<uint32_t>(args.a_mn) << 15) |
                             (static_cast<uint32_t>(args.b_mn) << 16) |
                             (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>(kBM >> 4) << 24);
      const uint32_t a_lbo0 = args.a_mn ? BK * 128 : 16;
      // (halo B: the S atoms of the tile are one row apart in the same box)
      const uint32_t b_lbo = args.cb.halo ? 128u : args.b_mn ? BK * 128 : 16;
      // MN-major 32-bit operands use the 32B-granule 128B swizzle: 4-row
      // swizzle groups (SBO 512) instead of 8-row groups (SBO 1024).
      const uint32_t a_sbo = (ES == 4 && args.a_mn) ? 512 : 1024;
      const uint32_t b_sbo = (ES == 4 && args.b_mn) ? 512 : 1024;
      const uint32_t a_lay = (ES == 4 && args.a_mn) ? 1 : 2;
      const uint32_t b_lay = (ES == 4 && args.b_mn) ? 1 : 2;
      const uint32_t a_kstep = args.a_mn ? UK * 128 : UK * ES;
      const uint32_t b_kstep = args.b_mn ? UK * 128 : UK * ES;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const TileIdx ti = tile_idx<BN>(args, t, tiles_m, tiles_n);
        // tap-pair A: the tile's two atoms are d rows apart in one box
        const uint32_t a_lbo = args.tp.n > 0 ? static_cast<uint32_t>(args.tp.d[ti.m0 / kBM]) * 128u : a_lbo0;
        const int buf = NACC == 2 ? (local & 1) : 0;
        const uint32_t use = NACC == 2 ? static_cast<uint32_t>(local >> 1) : static_cast<uint32_t>(local);
        mbar_wait(&tempty[buf], (use & 1) ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(buf) * ACOLS;
        for (int kt = ti.kt0; kt < ti.kt1; ++kt) {
          mbar_wait(SPLIT ? &conv[stage] : &full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * SB);
          const uint32_t sb = sa + A_BYTES;
          if (elect_one()) {  // the stage's MMAs back to back, then the commit
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
              const uint64_t ad = umma_desc_sw128(sa + k * a_kstep, a_lbo, a_sbo, a_lay);
              const uint64_t bd = umma_desc_sw128(sb + k * b_kstep, b_lbo, b_sbo, b_lay);
              const uint32_t acc = (kt > ti.kt0 || k > 0) ? 1u : 0u;
              if (MATH == kMathBF16) {
                mma_f16(d, ad, bd, idesc, acc);
              } else {
                mma_tf32(d, ad, bd, idesc, acc);
                if (SPLIT) {
                  const uint64_t ad2 = umma_desc_sw128(sb + B_BYTES + k * a_kstep, a_lbo, a_sbo, a_lay);
                  const uint64_t bd2 = umma_desc_sw128(sb + B_BYTES + A_BYTES + k * b_kstep, b_lbo, b_sbo, b_lay);
                  mma_tf32(d, ad, bd2, idesc, 1u);
                  mma_tf32(d, ad2, bd, idesc, 1u);
                }
              }
            }
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) mma_commit(&tfull[buf]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const float* sbias = epi_stage_bias(args, reinterpret_cast<float*>(smem + STAGES * SB + 256));
    int cstage = 0;
    uint32_t cphase = 0;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const TileIdx ti = tile_idx<BN>(args, t, tiles_m, tiles_n);
      if (SPLIT) {
        // 3xTF32: split every landed fp32 tile in place into hi = rna_tf32(x)
        // and lo = x - hi (exact) so D = Ahi*Bhi + Ahi*Blo + Alo*Bhi. The
        // swizzle is elementwise, so lo tiles share the hi tiles' layout.
        const int tt = threadIdx.x - 64;
        for (int kt = ti.kt0; kt < ti.kt1; ++kt) {
          mbar_wait(&full[cstage], cphase);
          float4* hi = reinterpret_cast<float4*>(smem + cstage * SB);
          float4* lo = reinterpret_cast<float4*>(smem + cstage * SB + A_BYTES + B_BYTES);
          constexpr int NV = (A_BYTES + B_BYTES) / 16;
#pragma unroll 4
          for (int i = tt; i < NV; i += 128) {
            float4 x = hi[i], h, l;
            h.x = tf32_rna(x.x); l.x = x.x - h.x;
            h.y = tf32_rna(x.y); l.y = x.y - h.y;
            h.z = tf32_rna(x.z); l.z = x.z - h.z;
            h.w = tf32_rna(x.w); l.w = x.w - h.w;
            hi[i] = h;
            lo[i] = l;
          }
          fence_proxy_async_smem();
          mbar_arrive(&conv[cstage]);
          if (++cstage == STAGES) {
            cstage = 0;
            cphase ^= 1;
          }
        }
      }
      const int buf = NACC == 2 ? (local & 1) : 0;
      const uint32_t use = NACC == 2 ? static_cast<uint32_t>(local >> 1) : static_cast<uint32_t>(local);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      float* stg = reinterpret_cast<float*>(smem + STAGES * SB + 256) + q * 32 * kEpiLd;
      const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf) * ACOLS;
      int mrow[8], mself;
      epi_rows(args, ti.m0 + q * 32, mrow, mself);
      MaskPre mcur, mnext;  // (not in the LIGHT kernel: FC wgrad has no mask, and registers are tight)
      if (!LIGHT) epi_mask_load(args, mself, ti.n0, mcur);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(base + static_cast<uint32_t>(c), r);
        if (!LIGHT && c + 32 < BN) epi_mask_load(args, mself, ti.n0 + c + 32, mnext);
        tmem_ld_wait();
        if (c + 32 >= BN) {  // accumulator fully in registers: hand it back to the MMA warp
          tc_fence_before();
          mbar_arrive(&tempty[buf]);
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (ti.n0 + c < args.N) epi_chunk(args, ti.m0 + q * 32, ti.n0 + c, ti.split, v, stg, mrow, mself, sbias, &mcur);
        mcur = mnext;
      }
    }
  }
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TCOLS);
  }
}

// CTA-pair GEMM: tcgen05.mma.cta_group::2 over a 256 x BN tile. Each CTA
// stages its own 128 rows of A and half (BN/2 rows) of B; the leader (rank 0)
// issues the M=256 MMAs; each CTA's TMEM holds its 128 accumulator rows and
// its epilogue stores them. Halves the B (and L2) traffic per SM vs 1-CTA.
__host__ __device__ constexpr uint32_t stage_bytes2(int bn) {
  return kBM * 128u + static_cast<uint32_t>(bn / 2) * 128u;
}
#ifndef HP_GEMM2_CAP
#define HP_GEMM2_CAP 8
#endif
__host__ __device__ constexpr int num_stages2(int bn) {
  return static_cast<int>((kMaxDynSmem - 2048u - kEpiSmemBytes) / stage_bytes2(bn)) > HP_GEMM2_CAP
             ? HP_GEMM2_CAP
             : static_cast<int>((kMaxDynSmem - 2048u - kEpiSmemBytes) / stage_bytes2(bn));
}

template <int BN, int MATH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                 const GemmArgs args) {
  static_assert(MATH != kMathF32x3, "3xTF32 runs on the 1-CTA kernel");
  constexpr int ES = MATH == kMathBF16 ? 2 : 4;
  constexpr int BK = 128 / ES;
  constexpr int UK = 32 / ES;
  constexpr int ATOM = 128 / ES;
  constexpr int BNH = BN / 2;
  constexpr uint32_t A_BYTES = kBM * 128;
  constexpr uint32_t SB = stage_bytes2(BN);
  constexpr int STAGES = num_stages2(BN);
  constexpr uint32_t ACOLS = tmem_cols(BN);
  constexpr uint32_t TCOLS = ACOLS * 2;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1;
  const int ncl = gridDim.x >> 1;
  const int tiles_m = (args.M + 2 * kBM - 1) / (2 * kBM);
  const int tiles_n = (args.N + BN - 1) / BN;
  const int splits = (args.k_tiles_total + args.k_tiles_per_split - 1) / args.k_tiles_per_split;
  const int total = tiles_m * tiles_n * splits;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);  // both CTAs' epilogue threads (leader's copy is used)
    }
    fence_barrier_init();
    tma_prefetch(&ta);
    tma_prefetch(&tb);
  }
  if (warp == 1) tmem_alloc2(tslot, TCOLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();  // predecessor's outputs (our inputs / output buffers) are final

  auto tile_of = [&](int t, int& m0, int& n0, int& split, int& kt0, int& kt1) {
    const int mn = tiles_m * tiles_n;
    split = t / mn;
    const int rem = t - split * mn;
    const int mb = rem / tiles_n;
    m0 = mb * 2 * kBM;
    n0 = (rem - mb * tiles_n) * BN;
    kt0 = split * args.k_tiles_per_split;
    kt1 = min(args.k_tiles_total, kt0 + args.k_tiles_per_split);
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < total; t += ncl) {
        int m0, n0, split, kt0, kt1;
        tile_of(t, m0, n0, split, kt0, kt1);
        const int am = m0 + static_cast<int>(rank) * kBM;
        const int bn0 = n0 + static_cast<int>(rank) * BNH;
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SB;
          uint8_t* sb = sa + A_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * SB);
          if (args.ca.enabled && args.a_mn && args.ca.shift) {
            load_mn_shift<true, BK, ATOM>(sa, &ta, &full[stage], args.ca, am, kBM, kt);
          } else if (args.ca.enabled && args.a_mn) {
            load_b_im2col<true, BK, ATOM>(sa, &ta, &full[stage], args.ca, am, kBM, kt);
          } else if (args.ca.enabled) {
            load_a_im2col<true, ATOM>(sa, &ta, &full[stage], args.ca, am, kt);
          } else {
            load_tile_t<true, BK, ATOM>(sa, &ta, &full[stage], args.a_mn, am, kBM, kt * BK);
          }
          if (args.cb.enabled && args.cb.shift) {
            load_mn_shift<true, BK, ATOM>(sb, &tb, &full[stage], args.cb, bn0, BNH, kt);
          } else if (args.cb.enabled) {
            load_b_im2col<true, BK, ATOM>(sb, &tb, &full[stage], args.cb, bn0, BNH, kt);
          } else {
            load_tile_t<true, BK, ATOM>(sb, &tb, &full[stage], args.b_mn, bn0, BNH, kt * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();  // all of this CTA's loads are issued: the next kernel may launch
    }
  } else if (warp == 1) {
    if (rank == 0) {  // leader's whole warp: warp-uniform loop, one elected issuer
      constexpr uint32_t fmt = MATH == kMathBF16 ? 1u : 2u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                             (static_cast<uint32_t>(args.a_mn) << 15) |
                             (static_cast<uint32_t>(args.b_mn) << 16) |
                             (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>((2 * kBM) >> 4) << 24);
      const uint32_t a_lbo = args.a_mn ? BK * 128 : 16;
      const uint32_t b_lbo = args.b_mn ? BK * 128 : 16;
      const uint32_t a_sbo = (ES == 4 && args.a_mn) ? 512 : 1024;
      const uint32_t b_sbo = (ES == 4 && args.b_mn) ? 512 : 1024;
      const uint32_t a_lay = (ES == 4 && args.a_mn) ? 1 : 2;
      const uint32_t b_lay = (ES == 4 && args.b_mn) ? 1 : 2;
      const uint32_t a_kstep = args.a_mn ? UK * 128 : UK * ES;
      const uint32_t b_kstep = args.b_mn ? UK * 128 : UK * ES;
      const uint32_t ahi = umma_desc_hi(a_sbo, a_lay), bhi = umma_desc_hi(b_sbo, b_lay);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = cid; t < total; t += ncl, ++local) {
        int m0, n0, split, kt0, kt1;
        tile_of(t, m0, n0, split, kt0, kt1);
        const int buf = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(&tempty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(buf) * ACOLS;
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * SB);
          const uint32_t sb = sa + A_BYTES;
          const uint32_t alo = (sa >> 4) | ((a_lbo >> 4) << 16), blo = (sb >> 4) | ((b_lbo >> 4) << 16);
          // one elected thread issues the stage's MMAs back to back (descriptors
          // in uniform registers; bf16 hi words are immediates) and the commit
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
              const uint32_t acc = (kt > kt0 || k > 0) ? 1u : 0u;
              if (MATH == kMathBF16) {
                constexpr uint64_t H = umma_desc_hi(1024, 2);
                mma_f16_2sm_lo<H, H>(d, alo + k * (a_kstep >> 4), blo + k * (b_kstep >> 4), idesc, acc);
              } else {
                mma_2sm_lohi<true>(d, alo + k * (a_kstep >> 4), ahi, blo + k * (b_kstep >> 4), bhi, idesc, acc);
              }
            }
            mma_commit_2sm(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) mma_commit_2sm(&tfull[buf]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const uint32_t tempty_leader[2] = {mapa(smem_u32(&tempty[0]), 0), mapa(smem_u32(&tempty[1]), 0)};
    const float* sbias = epi_stage_bias(args, reinterpret_cast<float*>(smem + STAGES * SB + 256));
    int local = 0;
    for (int t = cid; t < total; t += ncl, ++local) {
      int m0, n0, split, kt0, kt1;
      tile_of(t, m0, n0, split, kt0, kt1);
      const int buf = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      float* stg = reinterpret_cast<float*>(smem + STAGES * SB + 256) + q * 32 * kEpiLd;
      const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf) * ACOLS;
      int mrow[8], mself;
      epi_rows(args, m0 + static_cast<int>(rank) * kBM + q * 32, mrow, mself);
      MaskPre mcur, mnext;
      epi_mask_load(args, mself, n0, mcur);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(base + static_cast<uint32_t>(c), r);
        if (c + 32 < BN) epi_mask_load(args, mself, n0 + c + 32, mnext);
        tmem_ld_wait();
        if (c + 32 >= BN) {
          tc_fence_before();
          mbar_arrive_cluster(tempty_leader[buf]);
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (n0 + c < args.N)
          epi_chunk(args, m0 + static_cast<int>(rank) * kBM + q * 32, n0 + c, split, v, stg, mrow, mself, sbias, &mcur);
        mcur = mnext;
      }
    }
  }
  pdl_trigger();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, TCOLS);
  }
}

// ---------------------------------------------------------------- shift conv
// See conv_shift_plan (gemm.cuh). Warp roles as gemm2_kernel; per tile the
// K loop is (channel block cb) x (tap r, s): one halo TMA per cb (both CTAs,
// own 128 rows + halo), one weight-tile TMA per (tap, cb), 4 MMAs per tap whose
// A descriptor starts (r*wq + s) rows into the halo.
constexpr uint32_t kHaloBytes = 256u * 128u;
// halo ring depth (dev knob): 3 measured no different from 2 on the step
// (conv1 fprop, 2 channel blocks per tile, is not waiting on its halos)
#ifndef HP_SHIFT_HALOS
#define HP_SHIFT_HALOS 2
#endif
constexpr int kShiftHalos = HP_SHIFT_HALOS;
#ifndef HP_SHIFT_CAP
#define HP_SHIFT_CAP 12
#endif
__host__ __device__ constexpr uint32_t shift_b_bytes(int bn) { return static_cast<uint32_t>(bn / 2) * 128u; }
__host__ __device__ constexpr int shift_stages(int bn) {
  return static_cast<int>((kMaxDynSmem - 2304u - kEpiSmemBytes - kShiftHalos * kHaloBytes) / shift_b_bytes(bn)) >
                 HP_SHIFT_CAP
             ? HP_SHIFT_CAP
             : static_cast<int>((kMaxDynSmem - 2304u - kEpiSmemBytes - kShiftHalos * kHaloBytes) / shift_b_bytes(bn));
}
// barrier words (full/empty per stage + 8) and the TMEM slot, rounded to 128 B
__host__ __device__ constexpr uint32_t shift_bar_bytes(int bn) {
  return ((static_cast<uint32_t>(2 * shift_stages(bn) + 2 * kShiftHalos + 4) * 8u + 4u) + 127u) & ~127u;
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    conv_shift_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      const GemmArgs args) {
  constexpr int BNH = BN / 2;
  constexpr uint32_t B_BYTES = shift_b_bytes(BN);
  constexpr int STAGES = shift_stages(BN);
  constexpr uint32_t ACOLS = tmem_cols(BN);
  constexpr uint32_t TCOLS = ACOLS * 2;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* halo = smem;                                 // [kShiftHalos][256 rows][128 B]
  uint8_t* bst = smem + kShiftHalos * kHaloBytes;       // [STAGES][BNH rows][128 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(bst + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* hfull = empty + STAGES;         // [kShiftHalos]
  uint64_t* hempty = hfull + kShiftHalos;   // [kShiftHalos]
  uint64_t* tfull = hempty + kShiftHalos;   // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stg_base = reinterpret_cast<float*>(bst + STAGES * B_BYTES + shift_bar_bytes(BN));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1;
  const int ncl = gridDim.x >> 1;
  const int tiles_m = (args.M + 2 * kBM - 1) / (2 * kBM);
  const int tiles_n = (args.N + BN - 1) / BN;
  const int total = tiles_m * tiles_n;
  const int cblocks = args.sh_C / 64;
  const int taps = args.sh_R * args.sh_S;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < kShiftHalos; ++i) {
      mbar_init(&hfull[i], 1);
      mbar_init(&hempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);  // both CTAs' epilogue threads (leader's copy is used)
    }
    fence_barrier_init();
    tma_prefetch(&ta);
    tma_prefetch(&tb);
  }
  if (warp == 1) tmem_alloc2(tslot, TCOLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();  // predecessor's outputs (our inputs / output buffers) are final

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0, hb = 0;
      uint32_t phase = 0, hphase = 0;
      const uint32_t halo_tx = static_cast<uint32_t>(args.sh_halo) * 128u;
      for (int t = cid; t < total; t += ncl) {
        const int mb = t / tiles_n;
        const int m0 = mb * 2 * kBM, n0 = (t - mb * tiles_n) * BN;
        const int am = m0 + static_cast<int>(rank) * kBM;
        const int bn0 = n0 + static_cast<int>(rank) * BNH;
        for (int cb = 0; cb < cblocks; ++cb) {
          mbar_wait(&hempty[hb], hphase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&hfull[hb], 2 * halo_tx);
          tma_load_2d_2sm(halo + hb * kHaloBytes, &ta, &hfull[hb], cb * 64, am);
          if (++hb == kShiftHalos) {
            hb = 0;
            hphase ^= 1;
          }
          for (int tap = 0; tap < taps; ++tap) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * B_BYTES);
            tma_load_2d_2sm(bst + stage * B_BYTES, &tb, &full[stage], tap * args.sh_C + cb * 64, bn0);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      pdl_trigger();  // all of this CTA's loads are issued: the next kernel may launch
    }
  } else if (warp == 1) {
    if (rank == 0) {  // leader's whole warp: warp-uniform loop, one elected issuer
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                             (static_cast<uint32_t>((2 * kBM) >> 4) << 24);
      int stage = 0, hb = 0, local = 0;
      uint32_t phase = 0, hphase = 0;
      const uint32_t halo0 = smem_u32(halo);
      constexpr uint32_t hi0 = umma_desc_hi(1024, 2);
      for (int t = cid; t < total; t += ncl, ++local) {
        const int buf = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(&tempty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(buf) * ACOLS;
        uint32_t acc = 0;
        for (int cb = 0; cb < cblocks; ++cb) {
          mbar_wait(&hfull[hb], hphase);
          tc_fence_after();
          const uint32_t hbase = halo0 + static_cast<uint32_t>(hb) * kHaloBytes;
          for (int r = 0; r < args.sh_R; ++r)
            for (int sx = 0; sx < args.sh_S; ++sx) {
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              const uint32_t a0 = hbase + static_cast<uint32_t>(r * args.sh_wq + sx) * 128u;
              const uint32_t sb = smem_u32(bst + stage * B_BYTES);
              // The 128B swizzle is a function of the ABSOLUTE smem address bits
              // (TMA wrote the halo 1024-aligned), so a descriptor starting any
              // whole row into the halo reads rows a0.. correctly with the
              // descriptor base offset left 0 (measured: setting it to
              // (a0 >> 7) & 7 double-applies the phase).
              const uint32_t alo = (a0 >> 4) | (1u << 16), blo = (sb >> 4) | (1u << 16);
              if (elect_one()) {  // the tap's MMAs back to back, then the commit
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_f16_2sm_lo<hi0, hi0>(d, alo + 2 * k, blo + 2 * k, idesc, acc | (k > 0));
                mma_commit_2sm(&empty[stage]);
              }
              __syncwarp();
              acc = 1;
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
          if (elect_one()) mma_commit_2sm(&hempty[hb]);
          __syncwarp();
          if (++hb == kShiftHalos) {
            hb = 0;
            hphase ^= 1;
          }
        }
        if (elect_one()) mma_commit_2sm(&tfull[buf]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const uint32_t tempty_leader[2] = {mapa(smem_u32(&tempty[0]), 0), mapa(smem_u32(&tempty[1]), 0)};
    float* stg = stg_base + q * 32 * kEpiLd;
    const float* sbias = epi_stage_bias(args, stg_base);
    int local = 0;
    for (int t = cid; t < total; t += ncl, ++local) {
      const int mb = t / tiles_n;
      const int m0 = mb * 2 * kBM, n0 = (t - mb * tiles_n) * BN;
      const int buf = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf) * ACOLS;
      int mrow[8], mself;
      epi_rows(args, m0 + static_cast<int>(rank) * kBM + q * 32, mrow, mself);
      MaskPre mcur, mnext;
      epi_mask_load(args, mself, n0, mcur);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(base + static_cast<uint32_t>(c), r);
        if (c + 32 < BN) epi_mask_load(args, mself, n0 + c + 32, mnext);
        tmem_ld_wait();
        if (c + 32 >= BN) {
          tc_fence_before();
          mbar_arrive_cluster(tempty_leader[buf]);
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (n0 + c < args.N)
          epi_chunk(args, m0 + static_cast<int>(rank) * kBM + q * 32, n0 + c, 0, v, stg, mrow, mself, sbias, &mcur);
        mcur = mnext;
      }
    }
  }
  pdl_trigger();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, TCOLS);
  }
}

// One fp32 4-vector (m, n..n+3) through the epilogue (vectorised epi_elem).
__device__ __forceinline__ void epi_vec4(const Epi& e, int m, int n, float4 x) {
  const int gm = m;  // GEMM row (per-row bias)
  n = map_col(e.cols, n);  // (4-column groups never straddle a 64-column block)
  m = map_row(e.rows, m);
  if (m < 0) return;
  const long long off = static_cast<long long>(m) * e.ldc + n;
  x.x *= e.alpha;
  x.y *= e.alpha;
  x.z *= e.alpha;
  x.w *= e.alpha;
  if (e.beta) {
    const float4 o = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.c) + off);
    x.x += o.x;
    x.y += o.y;
    x.z += o.z;
    x.w += o.w;
  }
  if (e.sgd_w) {
    float4 w4 = *reinterpret_cast<const float4*>(e.sgd_w + off);
    float4 m4 = *reinterpret_cast<const float4*>(e.sgd_m + off);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float g = f4get(x, j);
      if (e.sgd_has_gscale) g = __fmul_rn(g, e.sgd_gscale);
      float d = __fmul_rn(f4get(m4, j), e.sgd_mu);
      d = __fadd_rn(d, __fmul_rn(e.sgd_s1, g));
      d = __fadd_rn(d, __fmul_rn(e.sgd_s2, f4get(w4, j)));
      f4set(m4, j, d);
      f4set(w4, j, __fadd_rn(f4get(w4, j), d));
    }
    *reinterpret_cast<float4*>(e.sgd_w + off) = w4;
    *reinterpret_cast<float4*>(e.sgd_m + off) = m4;
    if (e.sgd_copy) st_bf16x4(e.sgd_copy, off, w4);
    return;
  }
  if (e.bias_mode == 1) {
    const float bm = e.bias[gm];
    x.x += bm;
    x.y += bm;
    x.z += bm;
    x.w += bm;
  } else if (e.bias_mode == 2) {
    const float4 bb = *reinterpret_cast<const float4*>(e.bias + n);
    x.x += bb.x;
    x.y += bb.y;
    x.z += bb.z;
    x.w += bb.w;
  }
  if (e.relu) {
    x.x = x.x > 0.f ? x.x : 0.f;
    x.y = x.y > 0.f ? x.y : 0.f;
    x.z = x.z > 0.f ? x.z : 0.f;
    x.w = x.w > 0.f ? x.w : 0.f;
  }
  if (e.mask) {
    const long long mo = static_cast<long long>(m) * e.ldmask + n;
    const float4 k = e.mask_type == kBF16 ? ld_bf16x4(e.mask, mo)
                                          : *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.mask) + mo);
    if (!(k.x > 0.f)) x.x = 0.f;
    if (!(k.y > 0.f)) x.y = 0.f;
    if (!(k.z > 0.f)) x.z = 0.f;
    if (!(k.w > 0.f)) x.w = 0.f;
  }
  if (e.c_type == kF32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(e.c) + off) = x;
  } else {
    st_bf16x4(e.c, off, x);
  }
}

// Split-K reduce (ascending split order) + epilogue. vec: 4 columns per
// thread (N, ldc, ldmask multiples of 4, untransposed); else one element.
__global__ void epi_apply_kernel(const float* __restrict__ ws, int splits, int M, int N, const Epi e, int vec) {
  pdl_wait();
  const long long mn = static_cast<long long>(M) * N;
  if (vec) {
    const int n4 = N >> 2;
    const long long total = mn >> 2;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
      float4 acc = reinterpret_cast<const float4*>(ws)[i];
      for (int s = 1; s < splits; ++s) {
        const float4 v = reinterpret_cast<const float4*>(ws + s * mn)[i];
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      const int m = static_cast<int>(i / n4);
      epi_vec4(e, m, 4 * static_cast<int>(i - static_cast<long long>(m) * n4), acc);
    }
    return;
  }
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < mn;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float acc = ws[i];
    for (int s = 1; s < splits; ++s) acc += ws[s * mn + i];
    const int m = static_cast<int>(i / N);
    const int n = static_cast<int>(i - static_cast<long long>(m) * N);
    epi_elem(e, m, n, acc);
  }
}

// ------------------------------------------------------------------ host side

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr) {
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    }
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

CUtensorMap make_map(const void* ptr, int es, long long inner, long long outer, long long ld,
                     int box_inner, int box_outer, CUtensorMapSwizzle swz) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) {
    throw std::runtime_error("gemm: operand base not 16-byte aligned");
  }
  if ((ld * es) % 16 != 0) throw std::runtime_error("gemm: leading dimension not 16-byte aligned");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * es)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) +
                             ")");
  }
  return m;
}

PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr) {
      throw std::runtime_error("cuTensorMapEncodeIm2col unavailable");
    }
    fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  }
  return fn;
}

// im2col view of an NHWC tensor: dims {C, W, H, N}; the bounding box of base
// pixels runs from -pad to (extent + pad - filter) (WHD order, as CUTLASS's
// make_im2col_tma_copy_desc); `pixels` output pixels x ATOM channels per load.
CUtensorMap im2col_map(const void* ptr, int es, const Im2col& g, int pixels, bool mn_major) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) throw std::runtime_error("im2col: base not 16-byte aligned");
  const int atom = 128 / es;
  if (g.C % atom != 0) throw std::runtime_error("im2col: channels must be a multiple of 128 bytes");
  CUtensorMap m;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.C), static_cast<cuuint64_t>(g.W),
                        static_cast<cuuint64_t>(g.H), static_cast<cuuint64_t>(g.N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.C) * es, static_cast<cuuint64_t>(g.W) * g.C * es,
                           static_cast<cuuint64_t>(g.H) * g.W * g.C * es};
  int lower[2] = {-g.pad, -g.pad};                    // {W, H}
  int upper[2] = {g.pad - (g.S - 1), g.pad - (g.R - 1)};
  if (g.corners) {
    lower[0] = lower[1] = g.lo;
    upper[0] = upper[1] = g.hi;
  }
  const int sh = g.stride_h > 0 ? g.stride_h : g.stride;
  cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(g.stride), static_cast<cuuint32_t>(sh), 1};
  CUresult r = encode_im2col_fn()(&m, es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                  4, const_cast<void*>(ptr), dims, strides, lower, upper,
                                  static_cast<cuuint32_t>(atom), static_cast<cuuint32_t>(pixels), estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  (mn_major && es == 4) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                                        : CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw std::runtime_error("cuTensorMapEncodeIm2col failed (" + std::to_string(static_cast<int>(r)) + ")");
  }
  return m;
}

ConvArgs conv_args(const Im2col& g) {
  ConvArgs c{};
  c.enabled = g.enabled;
  c.C = g.C;
  c.S = g.S;
  c.OH = g.OH;
  c.OW = g.OW;
  c.stride = g.stride;
  c.stride_h = g.stride_h > 0 ? g.stride_h : g.stride;
  c.halo = g.halo;
  c.halo_rows = g.halo ? (64 + g.S - 1 + 7) / 8 * 8 : 0;
  c.lo_w = g.corners ? g.lo : -g.pad;
  c.lo_h = g.corners ? g.lo : -g.pad;
  c.shift = g.shift;
  c.wq = g.W;
  c.base_off = -(g.pad * g.W + g.pad);
  return c;
}

CUtensorMap operand_map(const GemmOperand& o, const void* ptr, int es, int rows, int K, int box_rows) {
  const int BK = 128 / es;
  const int ATOM = 128 / es;
  if (!o.mn_major) return make_map(ptr, es, K, rows, o.ld, BK, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
  return make_map(ptr, es, rows, K, o.ld, ATOM, BK,
                  es == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
}

// Kernel launch, optionally with programmatic stream serialization (see
// pdl_wait / pdl_trigger; both are no-ops without the attribute).
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // Opt-in (HP_DEV_PDL=1): measured 74.1k -> 72.4k img/s with it on (bench.py,
  // 2x2 runs) -- the early-resident dependent CTAs cost more than the hidden
  // launch/prologue latency -- so launches stay plainly stream-ordered.
  static const bool on = getenv("HP_DEV_PDL") != nullptr;
  cfg.attrs = attr;
  cfg.numAttrs = on ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm launch: ") + cudaGetErrorString(e));
}

template <int BN, int MATH>
void launch_inst2(const GemmPlan& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm2_kernel<BN, MATH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(p.smem));
    attr = true;
  }
  launch_pdl(gemm2_kernel<BN, MATH>, p.grid, dim3(192), p.smem, s, p.ta, p.tb, p.args);
}

template <int BN, int MATH, bool LIGHT>
void launch_inst(const GemmPlan& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel<BN, MATH, LIGHT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kMaxDynSmem));
    attr = true;
  }
  launch_pdl(gemm_kernel<BN, MATH, LIGHT>, p.grid, dim3(192), p.smem, s, p.ta, p.tb, p.args);
}

template <int MATH>
void launch_math(const GemmPlan& p, cudaStream_t s) {
  if (p.cta2) {
    if constexpr (MATH != kMathF32x3) {
      switch (p.bn) {
        case 64: launch_inst2<64, MATH>(p, s); return;
        case 128: launch_inst2<128, MATH>(p, s); return;
        case 192: launch_inst2<192, MATH>(p, s); return;
        case 256: launch_inst2<256, MATH>(p, s); return;
        default: break;
      }
    }
    throw std::runtime_error("gemm: unsupported 2-CTA configuration");
  }
  if (p.light) {
    if constexpr (MATH != kMathF32x3) {
      if (p.bn == 128) {
        launch_inst<128, MATH, true>(p, s);
        return;
      }
    }
    throw std::runtime_error("gemm: unsupported light configuration");
  }
  switch (p.bn) {
    case 64: launch_inst<64, MATH, false>(p, s); break;
    case 128: launch_inst<128, MATH, false>(p, s); break;
    case 192: launch_inst<192, MATH, false>(p, s); break;
    case 256: launch_inst<256, MATH, false>(p, s); break;
    default: throw std::runtime_error("gemm: unsupported BN");
  }
}

int cdiv(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace

int gemm_choose_bn(int M, int N) {
  const int mt = cdiv(M, kBM);
  const int cands[4] = {256, 192, 128, 64};
  int best = 64;
  double best_score = -1.0;
  for (int bn : cands) {
    const int nt = cdiv(N, bn);
    const double fill = static_cast<double>(N) / (static_cast<double>(nt) * bn);
    const int tiles = mt * nt;
    const int waves = cdiv(tiles, 148);
    const double wave_eff = static_cast<double>(tiles) / (waves * 148.0);
    // Prefer wide tiles (fewer smem bytes per MMA flop) unless they waste work.
    const double width = bn >= 128 ? 1.0 : 0.8;
    const double score = fill * (tiles >= 148 ? wave_eff : 1.0) * width;
    if (score > best_score + 1e-9) {
      best_score = score;
      best = bn;
    }
  }
  return best;
}

// Split-K factor when the tile grid underfills the machine: minimise the
// critical path, waves x (k-tiles per split + a fixed per-unit cost of ~4
// k-tiles: pipeline fill, epilogue, partial-sum write), keeping >= 8 k-tiles
// per split; more splits must win by >3% (partial-sum traffic). Measured on
// the FC shapes (tests/dev/fc_bench.py): fc6/fc7 fwd pick 4, fc8 8.
static int split_for_waves(int tiles, int kt, int slots) {
  if (tiles >= slots * 4 / 5 || kt < 16) return 1;
  int best = 1;
  double best_cost = static_cast<double>(cdiv(tiles, slots)) * (kt + 4);
  for (int s = 2; s <= std::min(64, kt / 8); ++s) {
    const int kps = cdiv(kt, s);
    const int real = cdiv(kt, kps);
    const double cost = static_cast<double>(cdiv(tiles * real, slots)) * (kps + 4);
    if (cost < best_cost * 0.97) {  // >3% better: more splits cost partial-sum traffic
      best_cost = cost;
      best = real;
    }
  }
  return best;
}

int gemm_choose_splits(int math, int M, int N, int K, int bn) {
  if (bn <= 0) bn = gemm_choose_bn(M, N);
  const int es = math == kMathBF16 ? 2 : 4;
  const int kt = cdiv(K, 128 / es);
  const int tiles = cdiv(M, kBM) * cdiv(N, bn);
  if (math == kMathF32x3) {
    // Parity mode: the tensor core accumulates with round-toward-zero, so the
    // error grows with the accumulation chain. Bound each chain to 4 k-tiles
    // (128 tf32 products); the split partials are summed in fp32 (RN).
    const int splits = std::max(1, std::min(cdiv(kt, 4), 512));
    const int kps = cdiv(kt, splits);
    return cdiv(kt, kps);
  }
  return split_for_waves(tiles, kt, 148);
}

static bool g_cta2_default = true;
static int g_force_cta2 = -1, g_force_bn = 0, g_dbg_flags = 0;
void gemm_debug_flags(int flags) { g_dbg_flags = flags; }
void gemm_set_cta2_default(bool on) { g_cta2_default = on; }
void gemm_force_config(int cta2, int bn) {
  g_force_cta2 = cta2;
  g_force_bn = bn;
}

// Tile choice from measured per-SM efficiency of each kernel shape (bf16,
// 8192^3: pair/256 1403 TF/s, single/256 1235, single/192 1047, pair/128 805,
// single/128 852) times N-tile fill and wave quantisation.
struct TileChoice {
  bool cta2;
  int bn;
};
static TileChoice choose_tile(int math, const GemmOperand& b, int M, int N) {
  struct Cand {
    bool cta2;
    int bn;
    double base;
  };
  const Cand cands[] = {{true, 256, 1.0}, {true, 192, 0.93}, {false, 256, 0.88}, {false, 192, 0.80},
                        {true, 128, 0.60}, {false, 128, 0.62}, {true, 64, 0.45}, {false, 64, 0.40}};
  TileChoice best{false, 128};
  double best_score = -1.0;
  for (const Cand& c : cands) {
    if (c.cta2 && (math == kMathF32x3 || !g_cta2_default || M < 256)) continue;
    if (c.cta2 && b.mn_major && (c.bn / 2) % (128 / (math == kMathBF16 ? 2 : 4)) != 0) continue;
    const int mt = c.cta2 ? cdiv(M, 2 * kBM) : cdiv(M, kBM);
    const int nt = cdiv(N, c.bn);
    const double nfill = static_cast<double>(N) / (static_cast<double>(nt) * c.bn);
    const double mfill = static_cast<double>(M) / (static_cast<double>(mt) * (c.cta2 ? 2 * kBM : kBM));
    const int units = mt * nt;                  // tiles (pairs count as one on two SMs)
    const int slots = c.cta2 ? 74 : 148;
    const int waves = cdiv(units, slots);
    const double wave = units >= slots ? static_cast<double>(units) / (waves * slots) : 1.0;
    // (ties -- e.g. pair/192 at 2/3 fill vs 128 at full fill for N = 128 -- go to
    // the tile that wastes less: measured 87.0 vs 84.6 us on conv1's pixel pairs)
    const double score = c.base * nfill * mfill * wave + 1e-3 * nfill * mfill;
    if (score > best_score + 1e-9) {
      best_score = score;
      best = {c.cta2, c.bn};
    }
  }
  return best;
}

static bool light_ok(int math, int kt, int splits) { return math != kMathF32x3 && kt <= 4 && splits == 1; }

GemmPlan gemm_plan(int math, const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
                   const Epi& epi, int splits, float* ws, int bn, int cta2, const TapPairs* tp) {
  if (M <= 0 || N <= 0 || K <= 0) throw std::runtime_error("gemm: empty problem");
  GemmPlan p;
  p.math = math;
  const int es = math == kMathBF16 ? 2 : 4;
  const int BK = 128 / es;
  const int kt = cdiv(K, BK);
  if (cta2 == -1 && g_force_cta2 >= 0) cta2 = g_force_cta2;
  if (bn <= 0 && g_force_bn > 0) bn = g_force_bn;
  if (cta2 == 1 && math == kMathF32x3) throw std::runtime_error("gemm: 3xTF32 has no 2-CTA kernel");
  bool use2;
  if (cta2 == -1 && bn <= 0 && light_ok(math, kt, 1)) {
    use2 = false;  // light single-CTA kernel (below)
  } else if (cta2 == -1 && bn <= 0) {
    const TileChoice tc = choose_tile(math, b, M, N);
    use2 = tc.cta2;
    bn = tc.bn;
  } else {
    use2 = math != kMathF32x3 && (cta2 == 1 || (cta2 == -1 && g_cta2_default && M >= 256));
  }
  if (use2 && b.mn_major && bn == 192) bn = 256;  // MN-major B halves must be whole 128-byte atoms
  p.cta2 = use2;
  if (use2) {
    p.bn = (bn == 64 || bn == 128 || bn == 192 || bn == 256) ? bn : 256;
    if (splits <= 0) {
      const int tiles2 = cdiv(M, 2 * kBM) * cdiv(N, p.bn);
      splits = split_for_waves(tiles2, kt, 74);
    }
  } else {
    p.bn = bn > 0 ? bn : gemm_choose_bn(M, N);
    if (splits <= 0) splits = gemm_choose_splits(math, M, N, K, p.bn);
    // short K (FC wgrad, K = n): the epilogue (gradient store or fused SGD
    // update) is the work -> the 2-CTA/SM light kernel
    p.light = light_ok(math, kt, splits) && cta2 != 1 && (bn <= 0 || bn == 128);
    if (p.light) p.bn = 128;
  }
  const int kps = cdiv(kt, splits);
  splits = cdiv(kt, kps);
  p.splits = splits;
  p.args.M = M;
  p.args.N = N;
  p.args.K = K;
  p.args.k_tiles_total = kt;
  p.args.k_tiles_per_split = kps;
  p.args.a_mn = a.mn_major;
  p.args.b_mn = b.mn_major;
  // (halo B / tap-pair A: the GEMM writes raw partials and epi_apply applies the maps)
  p.args.raw_partial = splits > 1 || (b.conv.enabled && b.conv.halo) || tp ? 1 : 0;
  p.args.dbg = g_dbg_flags;
  p.args.ws = ws;
  p.args.epi = epi;
  if (p.args.raw_partial && ws == nullptr) throw std::runtime_error("gemm: split-K needs a workspace");
  const int b_rows = use2 ? p.bn / 2 : p.bn;
  if (tp) {
    if (!a.conv.enabled || !a.conv.shift || !a.mn_major || use2 || es != 2 || tp->n * kBM != M || tp->n > 16)
      throw std::runtime_error("gemm: tap-pair A needs a bf16 MN-major shift operand on 1-CTA tiles");
    int dmax = 1;
    for (int i = 0; i < tp->n; ++i) dmax = std::max(dmax, tp->d[i]);
    p.args.tp = *tp;
    p.args.tp_rows = (64 + dmax + 7) / 8 * 8;
    p.ta = make_map(a.ptr, es, a.conv.C, static_cast<long long>(a.conv.N) * a.conv.H * a.conv.W, a.conv.C, 64,
                    p.args.tp_rows, CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (a.conv.enabled) {
    // K-major: rows = output pixels (fprop / dgrad); MN-major: K = output
    // pixels, M = (tap, channel) (wgrad as im2col(x)^T . dY)
    if (a.conv.shift) {
      if (!a.mn_major) throw std::runtime_error("gemm: shift-mode A must be MN-major");
      p.ta = make_map(a.ptr, es, a.conv.C, static_cast<long long>(a.conv.N) * a.conv.H * a.conv.W, a.conv.C, 128 / es,
                      BK, es == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
      p.ta = a.mn_major ? im2col_map(a.ptr, es, a.conv, BK, true) : im2col_map(a.ptr, es, a.conv, kBM, false);
    }
  } else {
    p.ta = operand_map(a, a.ptr, es, M, K, kBM);
  }
  if (b.conv.enabled && b.conv.halo) {
    if (!b.mn_major || !b.conv.shift || use2 || p.bn != 64 * b.conv.S || b.conv.C % 64 != 0 || es != 2)
      throw std::runtime_error("gemm: halo B needs a bf16 MN-major shift operand, 1-CTA tiles of S*64 columns");
    p.tb = make_map(b.ptr, es, b.conv.C, static_cast<long long>(b.conv.N) * b.conv.H * b.conv.W, b.conv.C, 64,
                    (64 + b.conv.S - 1 + 7) / 8 * 8, CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (b.conv.enabled && b.conv.shift) {
    if (!b.mn_major) throw std::runtime_error("gemm: shift-mode B must be MN-major");
    p.tb = make_map(b.ptr, es, b.conv.C, static_cast<long long>(b.conv.N) * b.conv.H * b.conv.W, b.conv.C, 128 / es,
                    BK, es == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (b.conv.enabled) {
    if (!b.mn_major) throw std::runtime_error("gemm: im2col B must be MN-major");
    p.tb = im2col_map(b.ptr, es, b.conv, BK, true);
  } else {
    p.tb = operand_map(b, b.ptr, es, N, K, b_rows);
  }
  p.args.ca = conv_args(a.conv);
  p.args.cb = conv_args(b.conv);
  if (use2) {
    const int total = cdiv(M, 2 * kBM) * cdiv(N, p.bn) * splits;
    p.grid = dim3(2 * std::min(total, 74));
    p.smem = static_cast<size_t>(num_stages2(p.bn)) * stage_bytes2(p.bn) + 1024 + 256 + kEpiSmemBytes;
  } else {
    const int total = cdiv(M, kBM) * cdiv(N, p.bn) * splits;
    p.grid = dim3(math == kMathF32x3 ? total : std::min(total, p.light ? 148 * HP_LIGHT_CTAS : 148));
    p.smem = static_cast<size_t>(p.light ? HP_LIGHT_STAGES : num_stages(p.bn, math)) * stage_bytes(p.bn, math) + 1024 + 256 +
             kEpiSmemBytes;
  }
  p.valid = true;
  return p;
}

void epi_apply_launch(const float* ws, int splits, int M, int N, const Epi& e, cudaStream_t s) {
  const bool vec = (N & 3) == 0 && !e.c_trans && !e.mask_trans && (e.ldc & 3) == 0 &&
                   (!e.mask || (e.ldmask & 3) == 0) && (!e.beta || e.c_type == kF32) &&
                   (!e.sgd_w || e.c_type == kF32);
  const long long total = static_cast<long long>(M) * N / (vec ? 4 : 1);
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<long long>((total + threads - 1) / threads, 148LL * 8));
  launch_pdl(epi_apply_kernel, dim3(blocks), dim3(threads), 0, s, ws, splits, M, N, e, vec ? 1 : 0);
}


bool conv_shift_supported(int C, int R, int S, int wq, int N) {
  return C % 64 == 0 && R >= 1 && S >= 1 && 128 + (R - 1) * wq + (S - 1) <= 256 && N >= 16;
}

GemmPlan conv_shift_plan(const void* x, long long rows, int C, int R, int S, int wq, const void* w, long long ldw,
                         int N, const Epi& epi, int boff_mode) {
  GemmPlan p;
  if (!conv_shift_supported(C, R, S, wq, N) || rows >= (1LL << 31)) return p;
  p.math = kMathBF16;
  p.shift = true;
  p.cta2 = true;
  // N tile: minimise rounds of pair tiles on the 74 pairs x the tile's cost
  // (MMA time ~ BN plus a fixed per-tap share), preferring wider tiles on ties
  static const int force_bn = getenv("HP_DEV_SHIFT_BN") ? atoi(getenv("HP_DEV_SHIFT_BN")) : 0;
  int best = 256;
  double best_cost = 1e30;
  const long long mt = (rows + 2 * kBM - 1) / (2 * kBM);
  for (int bn : {256, 192, 128, 64}) {
    const long long tiles = mt * cdiv(N, bn);
    const double cost = static_cast<double>((tiles + 73) / 74) * (bn + 64);
    if (cost < best_cost * 0.97) {
      best_cost = cost;
      best = bn;
    }
  }
  if (force_bn) best = force_bn;
  p.bn = best;
  p.splits = 1;
  const int halo = 128 + (R - 1) * wq + (S - 1);
  p.args.M = static_cast<int>(rows);
  p.args.N = N;
  p.args.K = R * S * C;
  p.args.k_tiles_total = R * S * (C / 64);
  p.args.k_tiles_per_split = p.args.k_tiles_total;
  p.args.epi = epi;
  p.args.sh_R = R;
  p.args.sh_S = S;
  p.args.sh_wq = wq;
  p.args.sh_C = C;
  p.args.sh_halo = halo;
  p.args.sh_boff = boff_mode;
  p.args.dbg = g_dbg_flags;
  p.ta = make_map(x, 2, C, rows, C, 64, halo, CU_TENSOR_MAP_SWIZZLE_128B);
  p.tb = make_map(w, 2, static_cast<long long>(R) * S * C, N, ldw, 64, p.bn / 2, CU_TENSOR_MAP_SWIZZLE_128B);
  const int total = cdiv(rows, 2 * kBM) * cdiv(N, p.bn);
  p.grid = dim3(2 * std::min(total, 74));
  p.smem = kShiftHalos * kHaloBytes + static_cast<size_t>(shift_stages(p.bn)) * shift_b_bytes(p.bn) + 1024 +
           shift_bar_bytes(p.bn) + kEpiSmemBytes;
  p.valid = true;
  return p;
}

template <int BN>
void launch_shift(const GemmPlan& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv_shift_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kMaxDynSmem));
    attr = true;
  }
  launch_pdl(conv_shift_kernel<BN>, p.grid, dim3(192), p.smem, s, p.ta, p.tb, p.args);
}

void gemm_launch(const GemmPlan& p, cudaStream_t s) {
  if (!p.valid) throw std::runtime_error("gemm: invalid plan");
  if (p.shift) {
    switch (p.bn) {
      case 64: launch_shift<64>(p, s); break;
      case 128: launch_shift<128>(p, s); break;
      case 192: launch_shift<192>(p, s); break;
      case 256: launch_shift<256>(p, s); break;
      default: throw std::runtime_error("conv_shift: unsupported BN");
    }
    return;
  }
  switch (p.math) {
    case kMathBF16: launch_math<kMathBF16>(p, s); break;
    case kMathTF32: launch_math<kMathTF32>(p, s); break;
    case kMathF32x3: launch_math<kMathF32x3>(p, s); break;
    default: throw std::runtime_error("gemm: bad math mode");
  }
  if (p.args.raw_partial) epi_apply_launch(p.args.ws, p.splits, p.args.M, p.args.N, p.args.epi, s);
}

}  // namespace hp
