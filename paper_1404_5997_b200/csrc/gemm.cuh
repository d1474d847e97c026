// tcgen05 GEMM: D[M,N] = sum_k A[m,k] * B[n,k], fp32 accumulation in TMEM.
//
// Operands are staged by TMA into 128B-swizzled shared memory. Each operand
// can be K-major (row-major [rows][K]) or MN-major (row-major [K][rows]); the
// UMMA descriptors take either, so no transposes are ever materialised.
// Inputs are bf16 (kind::f16), fp32 read as tf32 (kind::tf32), or fp32 split
// into hi/lo tf32 pairs (3xTF32, near-fp32 accuracy).
//
// The epilogue (TMEM -> registers -> global) fuses the elementwise work that
// follows each GEMM in the reference step: scale, accumulate (beta=1), bias
// (per row or per column), ReLU, and a ReLU-backward mask.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace hp {

enum DType : int { kF32 = 0, kBF16 = 1 };

enum MathMode : int {
  kMathBF16 = 0,   // bf16 operands, fp32 accumulate
  kMathTF32 = 1,   // fp32 operands read as tf32
  kMathF32x3 = 2,  // fp32 operands, 3xTF32 hi/lo split
};

// Epilogue row remap (im2col / q-layout outputs). GEMM row m is the pixel
// (b, y, x) of a source grid sH x sW (m = (b*sH + y)*sW + x); it is stored
// only if y < vH && x < vW, at row (b*dH + y + dp)*dW + x + dp of the output
// (and of the mask). q-layout: an HxW image with pad p stored as (H+p) x (W+p)
// row slots per image, pixel (h, w) at slot (h+p, w+p), zeros elsewhere -- the
// zero border of one row/image doubles as the next one's, so a stride-1 conv
// reads it as a flat shift of the row index.
struct RowMap {
  int enabled = 0;
  int sH = 0, sW = 0, vH = 0, vW = 0, dH = 0, dW = 0, dp = 0;
};

// Epilogue column permutation (the halo wgrad's N order, see Im2col::halo):
// GEMM column n = ((r * (C/64) + cb) * S + s) * 64 + c_lo is output column
// k = (r * S + s) * C + cb * 64 + c_lo. Applied by epi_apply (split-K reduce).
struct ColMap {
  int enabled = 0;
  int S = 0, C = 0;
};

// Epilogue row-block map for transposed (c_trans) outputs: GEMM row m is
// output row blk[m / 64] + m % 64 (blk < 0: dropped). The tap-pair wgrad's
// M order (see TapPairs); applied by epi_apply.
struct RowBlk {
  int enabled = 0;
  int blk[32] = {};
};

struct Epi {
  void* c = nullptr;  // output
  long long ldc = 0;
  int c_type = kF32;
  int c_trans = 0;    // 1: element (m,n) stored at c[n*ldc + m]
  float alpha = 1.f;
  int beta = 0;       // 1: c += result (fp32 output only)
  const float* bias = nullptr;
  int bias_mode = 0;  // 0 none, 1 per row (m), 2 per column (n)
  int relu = 0;
  const void* mask = nullptr;  // keep value where mask(m,n) > 0 (ReLU backward)
  long long ldmask = 0;
  int mask_type = kF32;
  int mask_trans = 0;
  // Fused momentum SGD (optimizer.cpp:19-31, float storage: four rounded
  // passes, no FMA). When sgd_w is set the (accumulated) result is the
  // gradient g of the parameters at the same offsets as c (ldc, row-major);
  // w and the momentum are updated in place and the gradient is not stored:
  //   g := g * gscale (if has_gscale);  d := mu d + s1 g + s2 w;  w := w + d
  float* sgd_w = nullptr;
  float* sgd_m = nullptr;
  void* sgd_copy = nullptr;  // optional bf16 operand copy of w (same offsets)
  float sgd_mu = 0.f, sgd_s1 = 0.f, sgd_s2 = 0.f, sgd_gscale = 1.f;
  int sgd_has_gscale = 0;
  RowMap rows;  // rows.enabled: remap output (and mask) rows; not with c_trans / sgd
  ColMap cols;  // cols.enabled: remap output columns (epi_apply only; the GEMM writes raw partials)
  RowBlk rblk;  // rblk.enabled: remap output rows by 64-row blocks (c_trans, epi_apply only)
};

// Tap-pair A operand (the swapped stride-1 wgrad, M = (tap, channel)): M tile t
// is two 64-channel atoms -- taps t0, t1 of channel block cb -- whose x rows
// differ by a fixed shift d (two neighbouring taps of a kernel row: d = 1; the
// leftover last taps of two kernel rows: d = wq). Both atoms come from ONE TMA
// box of 64 + d rows and the UMMA descriptor steps between them by d rows
// (LBO = d * 128 B), halving the A bytes of the per-tap boxes. A tile with a
// single tap uses d = 1 and a dropped second atom.
struct TapPairs {
  int n = 0;                 // M tiles
  int off[16] = {}, d[16] = {}, cb[16] = {};  // first atom's row shift, atom spacing (rows), channel block
};

// Implicit-GEMM convolution operand: the matrix is the im2col view of an NHWC
// activation tensor, gathered by TMA im2col loads (no im2col buffer).
//   as A (K-major, fprop / stride-1 dgrad): rows = output pixels (n,oh,ow),
//       K = (r, s, c) with c fastest;
//   as B (MN-major, wgrad): K = output pixels, N = (r, s, c).
// Requires C % (128 bytes / element size) == 0.
struct Im2col {
  int enabled = 0;
  int N = 0, H = 0, W = 0, C = 0;  // activation tensor
  int R = 0, S = 0, stride = 1, pad = 0;
  int OH = 0, OW = 0;              // output pixels enumerated by the GEMM
  // corners != 0: explicit im2col bounding box (both spatial dims) instead of
  // the one implied by pad: base pixels lo .. extent-1+hi (stride 1). Used on
  // zero-bordered "q-layout" tensors (see RowMap), where the padding is in
  // memory and the box walks either the valid outputs (lo 0, hi -p) or every
  // stored position (lo -p, hi -p).
  int corners = 0, lo = 0, hi = 0;
  // shift = 1 (MN-major operands, wgrad): x is a plain [N*H*W][C] q-layout
  // matrix and the K index is a stored q position; the (tap r, s) column block
  // of k-tile kt is the tiled TMA box at rows kt*BK + r*W + s - (pad*W + pad)
  // (zero fill outside) -- plain tiled loads instead of TMA im2col.
  int shift = 0;
  // vertical traversal stride when it differs from `stride` (0: same). The
  // s2d conv1 pixel-pair GEMM walks W with stride 2 (one row per output pixel
  // pair) and H with stride 1.
  int stride_h = 0;
  // halo = 1 (with shift, MN-major B of a stride-1 wgrad, S*64 <= 256): the
  // GEMM's N index is permuted to n = ((r * C/64 + cb) * S + s) * 64 + c_lo so
  // that an N tile of S*64 columns is the S taps (r, 0..S-1) of one 64-channel
  // block. Those taps read the same x rows shifted by 0..S-1, so the tile's B
  // is ONE box of 64 + S - 1 rows (rounded up to 8) and the UMMA descriptor
  // steps between its S atoms by one row (LBO = 128 B) instead of by a whole
  // atom: each x line crosses L2 -> SM once per tile, not once per tap.
  // The output columns come back through Epi::cols (ColMap).
  int halo = 0;
};



struct GemmOperand {
  const void* ptr = nullptr;
  int mn_major = 0;          // 0: [rows][K] (ld >= K); 1: [K][rows] (ld >= rows)
  long long ld = 0;          // elements
  Im2col conv;               // conv.enabled: ptr is the NHWC activation, ld unused
};

struct ConvArgs {            // device-side im2col bookkeeping (see Im2col)
  int enabled, C, S, OH, OW, stride, lo_w, lo_h;
  int shift, wq, base_off;   // Im2col::shift mode
  int stride_h;              // vertical stride (Im2col::stride_h, resolved)
  int halo, halo_rows;       // Im2col::halo: B tile = one box of halo_rows rows
};

struct GemmArgs {
  int M, N, K;
  int k_tiles_total;
  int k_tiles_per_split;
  int a_mn, b_mn;
  int raw_partial;  // 1: write fp32 partials to ws[split][M][N]; epilogue applied by reduce
  float* ws;
  Epi epi;
  ConvArgs ca, cb;  // im2col bookkeeping for A / B
  // shift conv (conv_shift_plan): taps R x S, flat row shift r*wq + s, C
  // channels per tap (64-channel blocks), halo rows per CTA, base-offset mode
  int sh_R, sh_S, sh_wq, sh_C, sh_halo, sh_boff;
  int dbg;  // dev flags (gemm_debug_flags): bit 0 = skip the epilogue's global traffic
  TapPairs tp;  // tp.n > 0: tap-pair A (MN-major shift operand, 1-CTA kernel)
  int tp_rows;  // rows of the tap-pair A box
};

// A fully prepared GEMM launch (tensor maps encoded once, reused every step).
struct GemmPlan {
  CUtensorMap ta, tb;
  GemmArgs args{};
  int math = kMathBF16;
  int bn = 128;
  int splits = 1;
  bool cta2 = false;  // CTA-pair kernel (M=256 tiles, cta_group::2)
  bool light = false; // 2-stage, 1-accumulator, 2-CTA/SM kernel (short K, fused SGD epilogue)
  bool shift = false; // stride-1 conv as flat row shifts of one smem halo per channel block
  dim3 grid;
  size_t smem = 0;
  bool valid = false;
};

// Builds a plan. `splits` <= 0 picks a split-K factor from the tile count.
// `ws` must hold splits*M*N floats when splits > 1 (query with gemm_ws_floats).
GemmPlan gemm_plan(int math, const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
                   const Epi& epi, int splits, float* ws, int bn = 0, int cta2 = -1,
                   const TapPairs* tp = nullptr);
// cta2: -1 auto (pairs for M >= 256 outside 3xTF32), 0 never, 1 force.
void gemm_set_cta2_default(bool on);
// Dev hook: force every later auto-configured plan to (cta2, bn); -1/0 = auto.
void gemm_force_config(int cta2, int bn);
// Dev hook: flags copied into every later plan (GemmArgs::dbg).
void gemm_debug_flags(int flags);
int gemm_choose_splits(int math, int M, int N, int K, int bn = 0);
int gemm_choose_bn(int M, int N);
void gemm_launch(const GemmPlan& p, cudaStream_t s);

// Stride-1 convolution as a flat-shift implicit GEMM (bf16, CTA pairs): the
// input x is a [rows][C] bf16 matrix in which output row o reads rows
// o + r*wq + s for the R x S taps (q-layout or a pad-free grid such as conv1's
// space-to-depth input). Per 64-channel block each CTA stages ONE halo of
// 128 + (R-1)*wq + (S-1) rows (<= 256) in swizzled smem and every tap's A
// operand is a row-shifted UMMA descriptor into it (no per-tap re-load). B is
// the [N][R*S*C] K-major kernel matrix (k = (r*S+s)*C + c). Output rows are the
// M = rows positions (the epilogue's RowMap drops the border / garbage rows);
// w rows have stride ldw >= R*S*C.
// Returns an invalid plan (valid = false) when the shape is unsupported.
GemmPlan conv_shift_plan(const void* x, long long rows, int C, int R, int S, int wq, const void* w, long long ldw,
                         int N, const Epi& epi, int boff_mode = 0);
bool conv_shift_supported(int C, int R, int S, int wq, int N);

// Applies an Epi elementwise to a fp32 [M][N] source (used after split-K and
// by the kernel tests).
void epi_apply_launch(const float* ws, int splits, int M, int N, const Epi& e, cudaStream_t s);

}  // namespace hp
