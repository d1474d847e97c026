// Memory-bound kernels of the step (HBM-bound; coalesced, 16-byte vectorised
// where the layout allows). Activations are NHWC; `T` is the activation /
// GEMM-operand storage type (bf16 in bf16 mode, fp32 in tf32 / 3xTF32 modes).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace hp {

// Where a pooling kernel stores its per-pixel output: an H x W grid of rows with
// the image at offset (p, p) (q-layout, see RowMap in gemm.cuh). {0,0,0}: the
// dense output grid.
struct OutLayout {
  int H = 0, W = 0, p = 0;
};

using bf16 = __nv_bfloat16;

// Reference batch layout NCHW fp32 -> device NHWC T.
template <class T>
void launch_nchw_to_nhwc(const float* x, T* y, int B, int C, int H, int W, cudaStream_t s);

// im2col: x [B][H][W][C] -> col [B*OH*OW][ldk], column k = (r*S + s)*C + c.
template <class T>
void launch_im2col(const T* x, T* col, int B, int H, int W, int C, int R, int S, int stride,
                   int pad, int OH, int OW, long long ldk, cudaStream_t st);

// col2im (gather, deterministic): dcol [B*OH*OW][ldk] fp32 -> dx [B][H][W][C].
// Optional ReLU-backward mask (keep where mask > 0, mask NHWC like dx).
template <class TO, class TM>
void launch_col2im(const float* dcol, TO* dx, const TM* mask, int B, int H, int W, int C, int R,
                   int S, int stride, int pad, int OH, int OW, long long ldk, cudaStream_t st);

// Overlapping max-pool, floor mode. idx = argmax plane index h*W+w.
template <class T>
void launch_maxpool_fwd(const T* x, T* y, int32_t* idx, int B, int H, int W, int C, int k, int s,
                        int OH, int OW, cudaStream_t st);
// Gather backward: dx = sum over windows whose argmax is this input.
template <class TO, class TM>
void launch_maxpool_bwd(const float* gy, const int32_t* idx, TO* gx, const TM* mask, int B, int H,
                        int W, int C, int k, int s, int OH, int OW, cudaStream_t st);

// Cross-channel LRN (Krizhevsky 2012; alpha not divided by n).
template <class T>
void launch_lrn_fwd(const T* a, T* b, float* d, long long P, int C, int n, float alpha, float beta,
                    float k, cudaStream_t st);
template <class TO, class TA>
void launch_lrn_bwd(const TA* a, const float* d, const float* gb, TO* ga, long long P, int C, int n,
                    float alpha, float beta, int relu_mask, cudaStream_t st);

// Column sums of x [M][ldx] over rows -> out [N] (ascending row blocks).
template <class T>
void launch_colsum(const T* x, long long M, int N, long long ldx, float* out, float* ws,
                   cudaStream_t st);
size_t colsum_ws_floats(long long M, int N);

// Row sums of x [R][ldx] (first n columns) -> out [R]; beta: out += sum.
template <class T>
void launch_rowsum(const T* x, int R, int n, long long ldx, float* out, int beta, cudaStream_t st);

// Logistic cross-entropy on a feature-major logit shard z [Ls][n] (fp32):
// targets t [n][L] (columns c0..c0+Ls), grad -> dz [Ls][ldz], per-block
// double loss partials -> partial[nblocks]. relu_mask: zero the gradient where
// the (post-ReLU) logit is not > 0. blocks <= 0: xent_blocks(Ls, n); callers
// that combine partials across ranks pass one count for all (every entry of
// partial[0..blocks) is rewritten). Returns nblocks.
template <class TO>
int launch_xent(const float* z, long long ldzin, const float* t, int L, int c0, int Ls, int n,
                TO* dz, long long ldz, double* partial, int* bad_target, int relu_mask, int blocks,
                cudaStream_t st);
int xent_blocks(int Ls, int n);

// Debug marker: a 1-thread kernel carrying an integer tag (graph-structure tests).
// tl: optional dev timeline buffer (see marker_kernel), cap entries.
void launch_marker(int tag, cudaStream_t st, unsigned long long* tl = nullptr, int cap = 0);
bool is_marker_kernel(const void* func);
// Device-resident targets: bad |= any t outside [0,1] (logistic_xent's
// DomainError, tensor.cpp:600-603, checked before a step changes any state).
void launch_target_check(const float* t, long long n, int* bad, cudaStream_t st);

// Momentum SGD over a list of tensors (optimizer.cpp:19-31, float storage:
// scalars rounded to float once, four separate rounded passes, no FMA).
struct SgdTensor {
  float* w;
  float* mom;
  const float* g;
  void* copy;  // optional: updated w cast to the operand type (bf16 mode)
  long long n;
  float gscale;  // grad pre-scale (1/K mean, 1/num_sub): applied as a rounded multiply
  int has_gscale;
};
constexpr int kMaxSgdTensors = 24;
void launch_sgd(const SgdTensor* ts, int nt, int copy_type, double lr, double momentum,
                double weight_decay, cudaStream_t st);

template <class T>
void launch_cast(const float* in, T* out, long long n, cudaStream_t st);

// Logical-transport reductions over K local workers (ascending worker order,
// the reference's order, cluster.cpp:568-576 / 293-295).
constexpr int kMaxLocal = 16;
struct PtrList {
  const float* p[kMaxLocal];
};
struct MutPtrList {
  float* p[kMaxLocal];
};
// out = sum_w in[w] (+ offset), cast to TO, optional scale.
template <class TO>
void launch_sum_k(PtrList in, int K, TO* out, long long n, float alpha, cudaStream_t st);
// bufs[w] = sum_w bufs[w] for all w.
void launch_allreduce_k(MutPtrList bufs, int K, long long n, cudaStream_t st);

// Strided 2D copy helper: rows of `bytes` from src (stride sp) to dst (stride dp).
void copy2d(void* dst, long long dp, const void* src, long long sp, long long bytes, long long rows,
            cudaStream_t st);

// out = (mask == nullptr || mask > 0) ? g : 0, cast to TO (ReLU backward).
template <class TO, class TM>
void launch_mask_cast(const float* g, const TM* mask, TO* out, long long n, cudaStream_t st);

// im2col straight from the reference's NCHW fp32 batch (first layer, C not a
// multiple of 128 bytes): col [B*OH*OW][ldk] in T, k = (r*S+s)*C + c, columns
// [R*S*C, ldk) zero.
template <class T>
void launch_im2col_nchw(const float* x, T* col, int B, int C, int H, int W, int R, int S,
                        int stride, int pad, int OH, int OW, long long ldk, cudaStream_t st);

// Transposed im2col straight from the NCHW fp32 batch: colT [K][P] (pixels
// contiguous, row stride ldp >= P), k = (r*S+s)*C + c. Consumed as an MN-major A
// (fprop) / K-major B (wgrad) operand.
template <class T>
void launch_im2col_t_nchw(const float* x, T* colT, int B, int C, int H, int W, int R, int S,
                          int stride, int pad, int OH, int OW, long long ldp, cudaStream_t st);

// Fused cross-channel LRN + overlapping max-pool forward (conv1/conv2 of
// AlexNet): y = maxpool(lrn(a)); the LRN output and its scale are never
// written (recomputed in backward). widx = argmax window offset r*k+q.
template <class T>
void launch_lrn_pool_fwd(const T* a, T* y, uint8_t* widx, int B, int H, int W, int C, int n,
                         float alpha, float beta, float kk, int pk, int ps, int PH, int PW,
                         cudaStream_t st, OutLayout yl = {});
// Fused backward: dz = relu_mask(a) * lrn_bwd(a, pool_bwd(gy, widx)).
template <class TA>
void launch_lrn_pool_bwd(const float* gy, const uint8_t* widx, const TA* a, TA* dz, int B, int H,
                         int W, int C, int n, float alpha, float beta, float kk, int pk, int ps,
                         int PH, int PW, int relu_mask, cudaStream_t st, OutLayout zl = {});
// Max-pool forward / backward with window-offset argmax (no LRN).
template <class T>
void launch_maxpool_fwd_w(const T* x, T* y, uint8_t* widx, int B, int H, int W, int C, int k, int s,
                          int OH, int OW, cudaStream_t st, OutLayout yl = {});
template <class TO, class TM>
void launch_maxpool_bwd_w(const float* gy, const uint8_t* widx, TO* gx, const TM* mask, int B, int H,
                          int W, int C, int k, int s, int OH, int OW, cudaStream_t st, OutLayout zl = {});

// wrot[c][r][s][f] = w[f][R-1-r][S-1-s][c] (w rows of stride ldk), cast to T:
// the stride-1 dgrad as a convolution over dY.
template <class T>
void launch_rotate_weights(const float* w, long long ldk, T* wrot, int F, int C, int R, int S,
                           cudaStream_t st);
// The same for up to 8 layers in one launch (the step's post-update rotations).
struct RotateTensor {
  const float* w;
  long long ldk;
  void* wrot;
  int F, C, R, S;
};
template <class T>
void launch_rotate_weights_multi(const RotateTensor* ts, int n, cudaStream_t st);

// Space-to-depth for a strided first layer (AlexNet conv1, stride s): the
// stride-s RxS conv over the NCHW fp32 batch equals a stride-1 Rq x Rq conv
// (Rq = ceil(R/s)) over z[b][i][j][ch], ch = (dr*s + dc)*C + c < s*s*C (zero up
// to Cz), z = xpad[b][c][s*i + dr][s*j + dc] (xpad: x shifted by pad, zero
// outside). Zh x Zw = (OH + Rq - 1) x (OW + Rq - 1). The implicit-GEMM path
// then runs conv1 like any other layer (TMA im2col over z, no col buffer).
template <class T>
void launch_s2d_input(const float* x, T* z, int B, int C, int H, int W, int s, int pad, int Zh, int Zw,
                      int Cz, cudaStream_t st);
// wz[f][(a*Rq + b)*Cz + ch] = w[f][((s*a+dr)*S + (s*b+dc))*C + c] (zero where
// s*a+dr >= R, s*b+dc >= S or ch >= s*s*C); w rows of stride ldk.
// bias2 != nullptr: the pixel-pair layout instead -- one GEMM row per pair of
// horizontally adjacent output pixels (2u, 2u+1), N = 2F output columns, taps
// (a, b') with b' in [0, Rq]: wz[p*F + f][(a*(Rq+1) + b')*Cz + ch] = the s2d
// weight at tap (a, b' - p) (zero outside [0, Rq)), and bias2[p*F + f] = bias[f].
template <class T>
void launch_s2d_weights(const float* w, long long ldk, T* wz, int F, int C, int R, int S, int s, int Rq,
                        int Cz, cudaStream_t st, const float* bias = nullptr, float* bias2 = nullptr);
// Inverse map of the s2d weight gradient back to the reference layout:
// dw[f][(r*S + q)*C + c] = dwz[f][((r/s)*Rq + q/s)*Cz + ((r%s)*s + q%s)*C + c].
// pairs: dwz is the pixel-pair gradient [2F][Rq][Rq+1][Cz]; the two pixel
// parities are summed (even + odd, rounded once).
void launch_s2d_wgrad_gather(const float* dwz, float* dw, long long ldk, int F, int C, int R, int S, int s,
                             int Rq, int Cz, cudaStream_t st, int pairs = 0);

// Cluster::set_skip_sync_broadcast negative control (cluster.cpp:306-314): after
// the all-reduce (g = sum over workers), worker-owned entries -- reference flat
// index (kernels [F][C][R][S] then bias, per layer from `base`) inside
// [own_b, own_e) -- become sum * inv_k; every other entry reverts to the
// worker's local gradient. Device layout of one layer: kernels [F][ldk] with
// k = (r*S + s)*C + c, then bias[F].
void launch_skip_sync_fixup(float* g, const float* local, int F, int C, int R, int S, long long ldk,
                            long long base, long long own_b, long long own_e, float inv_k, cudaStream_t st);

// Scale in place (fp32).
void launch_scale(float* x, long long n, float s, cudaStream_t st);

}  // namespace hp
