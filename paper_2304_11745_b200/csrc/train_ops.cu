// train_ops.cu -- sm_100a kernels of the training tenant's CUDA-core steps
// (include/gacer_train.h).
//
// All of these are HBM-bound streaming passes over NHWC bf16 activations
// ([M][C] row-major) or fp32 vectors: 16-byte loads/stores, 8 channels per
// thread, grids sized in multiples of the SM count.  Reductions are
// deterministic: each block sums a fixed row range in row order (fp32), the
// blocks' partials are combined in block order in fp64 -- no atomics.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/gacer.h"
#include "../../include/gacer_train.h"
#include "train_dev.cuh"
#include <cstring>

namespace gacer {
int set_error(int code, const char* msg);
}

namespace {

using gacer::VArgs;
using gacer::VG_THREADS;
using gacer::vg_grid_for;
using namespace gacer;   // VFn

// The one standalone kernel of the training operators: block b of an
// nvb-block grid runs virtual block b of operator fn (train_dev.cuh) -- the
// same device function, thread count and block decomposition the
// executor's DK_VGRID items use, so both paths give identical bits.
__global__ void __launch_bounds__(VG_THREADS) vgrid_kernel(int fn, VArgs a) {
  __shared__ __align__(16) uint8_t smem[gacer::VG_SMEM_BYTES];
  gacer::run_vgrid(fn, a, blockIdx.x, gridDim.x, threadIdx.x, blockDim.x, smem);
}

VArgs vargs() {
  VArgs a;
  memset(&a, 0, sizeof a);
  return a;
}

cudaError_t vlaunch(int fn, const VArgs& a, int nvb, cudaStream_t s) {
  if (nvb < 1) return cudaSuccess;
  vgrid_kernel<<<nvb, VG_THREADS, 0, s>>>(fn, a);
  return cudaGetLastError();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int launched(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    return gacer::set_error(GACER_E_CUDA, buf);
  }
  return GACER_OK;
}

int bad(int code, const char* msg) { return gacer::set_error(code, msg); }

}  // namespace

namespace gacer {
// GEMM-operand staging used by host.cpp's standalone conv calls
cudaError_t launch_dgrad_filter(const float* w, int Cout, int Cin, int KH, int KW, int cread, int Kpad, int rows,
                                void* out, cudaStream_t s) {
  VArgs a = vargs();
  a.p[0] = w; a.p[1] = out;
  a.i[0] = Cout; a.i[1] = Cin; a.i[2] = KH; a.i[3] = KW; a.i[4] = cread; a.i[5] = Kpad; a.i[6] = rows; a.i[7] = 0;
  return vlaunch(VF_FILTER, a, vg_grid_for(static_cast<int64_t>(rows) * Kpad), s);
}

cudaError_t launch_fwd_filter(const float* w, int Cout, int Cin, int KH, int KW, int cread, int Kpad, int rows,
                              void* out, cudaStream_t s, int block_bn) {
  VArgs a = vargs();
  a.p[0] = w; a.p[1] = out;
  a.i[0] = Cout; a.i[1] = Cin; a.i[2] = KH; a.i[3] = KW; a.i[4] = cread; a.i[5] = Kpad; a.i[6] = rows; a.i[7] = 1;
  a.i[8] = block_bn;
  return vlaunch(VF_FILTER, a, vg_grid_for(static_cast<int64_t>(rows) * Kpad), s);
}

cudaError_t launch_dgrad_phase_filter(const float* w, int Cout, int Cin, int KI, int KJ, int cread, int Kpad, int rows,
                                      int S, int pa, int pb, int KH, int KW, void* out, cudaStream_t s) {
  VArgs a = vargs();
  a.p[0] = w; a.p[1] = out;
  a.i[0] = Cout; a.i[1] = Cin; a.i[2] = KI; a.i[3] = KJ; a.i[4] = cread; a.i[5] = Kpad; a.i[6] = rows; a.i[7] = 0;
  a.i[9] = S; a.i[10] = pa; a.i[11] = pb; a.i[12] = KH; a.i[13] = KW;
  return vlaunch(VF_FILTER, a, vg_grid_for(static_cast<int64_t>(rows) * Kpad), s);
}

cudaError_t launch_phase_scatter(const void* const* phase_out, int N, int H, int W, int C, int S, int ph, int pw,
                                 int KH, int KW, void* dx, cudaStream_t s) {
  VArgs a = vargs();
  for (int i = 0; i < S * S && i < 4; ++i) a.p[i] = phase_out[i];
  a.p[4] = dx;
  a.n[0] = static_cast<int64_t>(N) * H * W * (C / 8);
  a.i[0] = N; a.i[1] = H; a.i[2] = W; a.i[3] = C; a.i[4] = S; a.i[5] = ph; a.i[6] = pw; a.i[7] = KH; a.i[8] = KW;
  return vlaunch(VF_PHASE_SCATTER, a, vg_grid_for(a.n[0]), s);
}

cudaError_t launch_dilate(const void* dy, int N, int Hd, int Wd, int C, int S, int Hdd, int Wdd, void* out,
                          cudaStream_t s) {
  VArgs a = vargs();
  a.p[0] = dy; a.p[1] = out;
  a.i[0] = N; a.i[1] = Hd; a.i[2] = Wd; a.i[3] = C; a.i[4] = S; a.i[5] = Hdd; a.i[6] = Wdd;
  return vlaunch(VF_DILATE, a, vg_grid_for(static_cast<int64_t>(N) * Hdd * Wdd * (C / 8)), s);
}

VArgs transpose_args(const void* x, int N, int H, int W, int C, int Ho, int Wo, int KH, int KW, int S, int ph, int pw,
                     int64_t M, int Kpad, void* out) {
  VArgs a = vargs();
  a.p[0] = x; a.p[1] = out;
  a.n[0] = M;
  a.i[0] = N; a.i[1] = H; a.i[2] = W; a.i[3] = C; a.i[4] = Ho; a.i[5] = Wo; a.i[6] = KW; a.i[7] = S;
  a.i[8] = ph; a.i[9] = pw; a.i[10] = Kpad; a.i[11] = KH;
  return a;
}

int transpose_blocks(int C, int KH, int KW, int Kpad) { return vg_transpose_blocks(C, KH, KW, Kpad); }

cudaError_t launch_transpose_im2col(const void* x, int N, int H, int W, int C, int Ho, int Wo, int KH, int KW, int S,
                                    int ph, int pw, int64_t M, int Kpad, void* out, cudaStream_t s) {
  return vlaunch(VF_TRANSPOSE_IM2COL, transpose_args(x, N, H, W, C, Ho, Wo, KH, KW, S, ph, pw, M, Kpad, out),
                 transpose_blocks(C, KH, KW, Kpad), s);
}

cudaError_t launch_wgrad_reduce(const float* part, int Cout, int Cin, int KH, int KW, int bn, int tiles_n, int split,
                                float* dw, cudaStream_t s) {
  VArgs a = vargs();
  a.p[0] = part; a.p[1] = dw;
  a.i[0] = Cout; a.i[1] = Cin; a.i[2] = KH; a.i[3] = KW; a.i[4] = bn; a.i[5] = tiles_n; a.i[6] = split;
  return vlaunch(VF_WGRAD_REDUCE, a, vg_grid_for(static_cast<int64_t>((KH * KW * Cin + 3) / 4) * Cout), s);
}

cudaError_t launch_wgrad_permute(const float* g, int Cout, int Cin, int KH, int KW, float* dw, cudaStream_t s) {
  VArgs a = vargs();
  a.p[0] = g; a.p[1] = dw;
  a.i[0] = Cout; a.i[1] = Cin; a.i[2] = KH; a.i[3] = KW;
  return vlaunch(VF_WGRAD_PERMUTE, a, vg_grid_for(static_cast<int64_t>(Cout) * Cin * KH * KW), s);
}

__global__ void fill_kernel(float* p, int n, float v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

cudaError_t launch_fill(float* p, int n, float v, cudaStream_t s) {
  fill_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, n, v);
  return cudaGetLastError();
}
}  // namespace gacer

extern "C" {

int32_t gacer_bn_partials(int64_t M, int32_t C) {
  (void)C;
  return M < 1 ? 0 : gacer::vg_bn_partials(M);
}

int32_t gacer_bn_train_fwd(const void* x_dev, int64_t M, int32_t C, const float* gamma_dev, const float* beta_dev,
                           float eps, int32_t relu, void* y_dev, float* mean_dev, float* var_dev, float* scratch_dev,
                           void* stream) {
  if (M < 1 || C < 8 || C % 8 || C > VG_MAX_BN_C)
    return bad(GACER_E_SHAPE, "bn_train_fwd: need M >= 1, C % 8 == 0 and C <= 2048");
  if (!x_dev || !y_dev || !gamma_dev || !beta_dev || !mean_dev || !var_dev || !scratch_dev ||
      !aligned16(x_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "bn_train_fwd: null or misaligned pointer");
  auto s = static_cast<cudaStream_t>(stream);
  const int P = gacer::vg_bn_partials(M);
  float* coef = scratch_dev + static_cast<size_t>(P) * 2 * C;
  VArgs a = vargs();
  a.p[0] = x_dev; a.p[5] = scratch_dev; a.n[0] = M; a.i[0] = 0; a.i[1] = C;
  vlaunch(VF_BN_PARTIAL, a, P, s);
  VArgs f = vargs();
  f.p[0] = scratch_dev; f.p[1] = gamma_dev; f.p[2] = beta_dev; f.p[3] = x_dev; f.p[5] = mean_dev; f.p[6] = var_dev;
  f.p[7] = coef; f.n[0] = M; f.i[0] = 0; f.i[1] = C; f.i[2] = P; f.f[0] = eps;
  vlaunch(VF_BN_FINALIZE, f, (C + 31) / 32, s);
  VArgs e = vargs();
  e.p[0] = x_dev; e.p[3] = coef; e.p[4] = y_dev; e.n[0] = M; e.i[0] = 0; e.i[1] = C; e.i[2] = relu;
  vlaunch(VF_BN_APPLY, e, gacer::vg_apply_blocks(M * (C / 8)), s);
  return launched("bn_train_fwd");
}

int32_t gacer_bn_train_bwd(const void* x_dev, const void* dy_dev, const void* relu_y_dev, int64_t M, int32_t C,
                           const float* gamma_dev, const float* mean_dev, const float* var_dev, float eps, void* dx_dev,
                           float* dgamma_dev, float* dbeta_dev, float* scratch_dev, void* stream) {
  if (M < 1 || C < 8 || C % 8 || C > VG_MAX_BN_C)
    return bad(GACER_E_SHAPE, "bn_train_bwd: need M >= 1, C % 8 == 0 and C <= 2048");
  if (!x_dev || !dy_dev || !dx_dev || !gamma_dev || !mean_dev || !var_dev || !dgamma_dev || !dbeta_dev ||
      !scratch_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev) ||
      (relu_y_dev && !aligned16(relu_y_dev)))
    return bad(GACER_E_INVALID_ARG, "bn_train_bwd: null or misaligned pointer");
  auto s = static_cast<cudaStream_t>(stream);
  const int P = gacer::vg_bn_partials(M);
  float* coef = scratch_dev + static_cast<size_t>(P) * 2 * C;
  VArgs a = vargs();
  a.p[0] = x_dev; a.p[1] = dy_dev; a.p[2] = relu_y_dev; a.p[3] = mean_dev; a.p[4] = var_dev; a.p[5] = scratch_dev;
  a.n[0] = M; a.i[0] = 1; a.i[1] = C; a.f[0] = eps;
  vlaunch(VF_BN_PARTIAL, a, P, s);
  VArgs f = vargs();
  f.p[0] = scratch_dev; f.p[1] = gamma_dev; f.p[3] = mean_dev; f.p[4] = var_dev; f.p[5] = dgamma_dev;
  f.p[6] = dbeta_dev; f.p[7] = coef; f.n[0] = M; f.i[0] = 1; f.i[1] = C; f.i[2] = P; f.f[0] = eps;
  vlaunch(VF_BN_FINALIZE, f, (C + 31) / 32, s);
  VArgs e = vargs();
  e.p[0] = x_dev; e.p[1] = dy_dev; e.p[2] = relu_y_dev; e.p[3] = coef; e.p[4] = dx_dev; e.n[0] = M; e.i[0] = 1;
  e.i[1] = C;
  vlaunch(VF_BN_APPLY, e, gacer::vg_apply_blocks(M * (C / 8)), s);
  return launched("bn_train_bwd");
}

int32_t gacer_relu_bwd(const void* x_dev, const void* dy_dev, int64_t n, int32_t six, void* dx_dev, void* stream) {
  if (n < 0 || n % 8) return bad(GACER_E_SHAPE, "relu_bwd: n % 8 != 0");
  if (!x_dev || !dy_dev || !dx_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev))
    return bad(GACER_E_INVALID_ARG, "relu_bwd: null or misaligned pointer");
  if (n == 0) return GACER_OK;
  VArgs a = vargs();
  a.p[0] = x_dev; a.p[1] = dy_dev; a.p[2] = dx_dev; a.n[0] = n / 8; a.i[0] = six;
  vlaunch(VF_RELU_BWD, a, vg_grid_for(n / 8), static_cast<cudaStream_t>(stream));
  return launched("relu_bwd");
}

namespace {
VArgs pool_args(const void* p0, const void* p1, const void* p2, int N, int H, int W, int C, int KH, int KW, int S,
                int ph, int pw, int Ho, int Wo) {
  VArgs a = vargs();
  a.p[0] = p0; a.p[1] = p1; a.p[2] = p2;
  a.i[0] = N; a.i[1] = H; a.i[2] = W; a.i[3] = C; a.i[4] = KH; a.i[5] = KW; a.i[6] = S; a.i[7] = ph; a.i[8] = pw;
  a.i[9] = Ho; a.i[10] = Wo;
  return a;
}
}  // namespace

int32_t gacer_maxpool_bwd(const void* x_dev, const void* dy_dev, int32_t N, int32_t H, int32_t W, int32_t C,
                          int32_t KH, int32_t KW, int32_t stride, int32_t ph, int32_t pw, int32_t Ho, int32_t Wo,
                          void* dx_dev, void* scratch_dev, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || KH < 1 || KW < 1 || KH * KW > 255 || stride < 1 || ph < 0 ||
      pw < 0 || Ho != (H + 2 * ph - KH) / stride + 1 || Wo != (W + 2 * pw - KW) / stride + 1 || Ho < 1 || Wo < 1)
    return bad(GACER_E_SHAPE, "maxpool_bwd: inconsistent shape");
  if (!x_dev || !dy_dev || !dx_dev || !scratch_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev) ||
      (reinterpret_cast<uintptr_t>(scratch_dev) & 7u))
    return bad(GACER_E_INVALID_ARG, "maxpool_bwd: null or misaligned pointer");
  auto s = static_cast<cudaStream_t>(stream);
  vlaunch(VF_MAXPOOL_ARGMAX, pool_args(x_dev, scratch_dev, nullptr, N, H, W, C, KH, KW, stride, ph, pw, Ho, Wo),
          vg_grid_for(static_cast<int64_t>(N) * Ho * Wo * (C / 8)), s);
  vlaunch(VF_MAXPOOL_BWD, pool_args(scratch_dev, dy_dev, dx_dev, N, H, W, C, KH, KW, stride, ph, pw, Ho, Wo),
          vg_grid_for(static_cast<int64_t>(N) * H * W * (C / 8)), s);
  return launched("maxpool_bwd");
}

int32_t gacer_gap_bwd(const float* dy_dev, int32_t N, int32_t HW, int32_t C, void* dx_dev, void* stream) {
  if (N < 1 || HW < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "gap_bwd: need C % 8 == 0");
  if (!dy_dev || !dx_dev || !aligned16(dx_dev)) return bad(GACER_E_INVALID_ARG, "gap_bwd: null or misaligned pointer");
  VArgs a = vargs();
  a.p[0] = dy_dev; a.p[1] = dx_dev; a.i[0] = N; a.i[1] = HW; a.i[2] = C;
  vlaunch(VF_GAP_BWD, a, vg_grid_for(static_cast<int64_t>(N) * HW * (C / 8)), static_cast<cudaStream_t>(stream));
  return launched("gap_bwd");
}

int32_t gacer_maxpool_fwd(const void* x_dev, int32_t N, int32_t H, int32_t W, int32_t C, int32_t KH, int32_t KW,
                          int32_t stride, int32_t ph, int32_t pw, int32_t Ho, int32_t Wo, void* y_dev, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || KH < 1 || KW < 1 || stride < 1 || ph < 0 || pw < 0 ||
      Ho != (H + 2 * ph - KH) / stride + 1 || Wo != (W + 2 * pw - KW) / stride + 1 || Ho < 1 || Wo < 1)
    return bad(GACER_E_SHAPE, "maxpool_fwd: inconsistent shape");
  if (!x_dev || !y_dev || !aligned16(x_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "maxpool_fwd: null or misaligned pointer");
  vlaunch(VF_MAXPOOL_FWD, pool_args(x_dev, y_dev, nullptr, N, H, W, C, KH, KW, stride, ph, pw, Ho, Wo),
          vg_grid_for(static_cast<int64_t>(N) * Ho * Wo * (C / 8)), static_cast<cudaStream_t>(stream));
  return launched("maxpool_fwd");
}

int32_t gacer_add(const void* a_dev, const void* b_dev, int64_t n, int32_t relu, void* y_dev, void* stream) {
  if (n < 0 || n % 8) return bad(GACER_E_SHAPE, "add: n % 8 != 0");
  if (!a_dev || !b_dev || !y_dev || !aligned16(a_dev) || !aligned16(b_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "add: null or misaligned pointer");
  if (n == 0) return GACER_OK;
  VArgs a = vargs();
  a.p[0] = a_dev; a.p[1] = b_dev; a.p[2] = y_dev; a.n[0] = n / 8; a.i[0] = relu;
  vlaunch(VF_ADD, a, vg_grid_for(n / 8), static_cast<cudaStream_t>(stream));
  return launched("add");
}

int32_t gacer_gap_fwd(const void* x_dev, int32_t N, int32_t HW, int32_t C, void* y_dev, void* stream) {
  if (N < 1 || HW < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "gap_fwd: need C % 8 == 0");
  if (!x_dev || !y_dev || !aligned16(x_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "gap_fwd: null or misaligned pointer");
  VArgs a = vargs();
  a.p[0] = x_dev; a.p[1] = y_dev; a.i[0] = N; a.i[1] = HW; a.i[2] = C;
  vlaunch(VF_GAP_FWD, a, vg_grid_for(static_cast<int64_t>(N) * (C / 8)), static_cast<cudaStream_t>(stream));
  return launched("gap_fwd");
}

int32_t gacer_linear_fwd(const void* x_dev, const float* w_dev, const float* b_dev, int32_t N, int32_t K, int32_t O,
                         float* z_dev, void* stream) {
  if (N < 1 || K < 1 || O < 1) return bad(GACER_E_SHAPE, "linear_fwd: need N, K, O >= 1");
  if (!x_dev || !w_dev || !z_dev) return bad(GACER_E_INVALID_ARG, "linear_fwd: null pointer");
  VArgs a = vargs();
  a.p[0] = x_dev; a.p[1] = w_dev; a.p[2] = b_dev; a.p[3] = z_dev; a.i[0] = N; a.i[1] = K; a.i[2] = O;
  vlaunch(VF_LINEAR_FWD, a, vg_grid_for(static_cast<int64_t>(N) * ((O + 3) / 4) * 32), static_cast<cudaStream_t>(stream));
  return launched("linear_fwd");
}

int32_t gacer_linear_bwd(const void* x_dev, const float* w_dev, const float* dy_dev, int32_t N, int32_t K, int32_t O,
                         float* dx_dev, float* dw_dev, float* db_dev, void* stream) {
  if (N < 1 || K < 1 || O < 1) return bad(GACER_E_SHAPE, "linear_bwd: need N, K, O >= 1");
  if (!x_dev || !w_dev || !dy_dev || !dw_dev) return bad(GACER_E_INVALID_ARG, "linear_bwd: null pointer");
  auto s = static_cast<cudaStream_t>(stream);
  if (dx_dev) {
    VArgs a = vargs();
    a.p[0] = w_dev; a.p[1] = dy_dev; a.p[2] = dx_dev; a.i[0] = N; a.i[1] = K; a.i[2] = O;
    vlaunch(VF_LINEAR_DX, a, vg_grid_for(static_cast<int64_t>((N + 3) / 4) * K), s);
  }
  VArgs a = vargs();
  a.p[0] = x_dev; a.p[1] = dy_dev; a.p[2] = dw_dev; a.p[3] = db_dev; a.i[0] = N; a.i[1] = K; a.i[2] = O;
  vlaunch(VF_LINEAR_DW, a, vg_grid_for(static_cast<int64_t>((O + 3) / 4) * K), s);
  return launched("linear_bwd");
}

int32_t gacer_softmax_ce(const float* z_dev, const int32_t* labels_dev, int32_t N, int32_t Cls, float* loss_dev,
                         float* dz_dev, float* scratch_dev, void* stream) {
  if (N < 1 || Cls < 1) return bad(GACER_E_SHAPE, "softmax_ce: need N, Cls >= 1");
  if (!z_dev || !labels_dev || !loss_dev || !dz_dev || !scratch_dev)
    return bad(GACER_E_INVALID_ARG, "softmax_ce: null pointer");
  auto s = static_cast<cudaStream_t>(stream);
  VArgs a = vargs();
  a.p[0] = z_dev; a.p[1] = labels_dev; a.p[2] = dz_dev; a.p[3] = scratch_dev; a.i[0] = N; a.i[1] = Cls;
  vlaunch(VF_SOFTMAX_CE, a, N, s);
  VArgs m = vargs();
  m.p[0] = scratch_dev; m.p[1] = loss_dev; m.i[0] = N;
  vlaunch(VF_MEAN, m, 1, s);
  return launched("softmax_ce");
}

int32_t gacer_sgd_momentum(float* w_dev, const float* g_dev, float* buf_dev, int64_t n, float lr, float momentum,
                           int32_t first, void* stream) {
  if (n < 0) return bad(GACER_E_SHAPE, "sgd_momentum: n < 0");
  if (!w_dev || !g_dev || !buf_dev) return bad(GACER_E_INVALID_ARG, "sgd_momentum: null pointer");
  if (n == 0) return GACER_OK;
  VArgs a = vargs();
  a.p[0] = w_dev; a.p[1] = g_dev; a.p[2] = buf_dev; a.n[0] = n; a.i[0] = first; a.f[0] = lr; a.f[1] = momentum;
  vlaunch(VF_SGD, a, vg_grid_for(n), static_cast<cudaStream_t>(stream));
  return launched("sgd_momentum");
}

}  // extern "C"
