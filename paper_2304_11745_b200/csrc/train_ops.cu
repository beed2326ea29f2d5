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

namespace gacer {
int set_error(int code, const char* msg);
}

namespace {

constexpr int kThreads = 256;
constexpr int kMaxPartials = 148 * 4;   // row blocks of a BN reduction (4 waves of CTAs on 148 SMs)
constexpr int kRowsPerBlockMin = 32;

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  return make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
}

int num_partials(int64_t M) {
  int64_t p = (M + kRowsPerBlockMin - 1) / kRowsPerBlockMin;
  return static_cast<int>(p < kMaxPartials ? (p < 1 ? 1 : p) : kMaxPartials);
}

// ---------------------------------------------------------------- BN reductions
// Per-channel sums over a row block.  MODE 0: (sum x, sum x^2);
// MODE 1: (sum dy, sum dy * xhat) with xhat = (x - mean) * invstd.
// Thread layout: thread t owns 8-channel group g = t % G and row phase
// t / G (RP phases), for channel groups g, g + G, ... when C / 8 > 256.
template <int MODE>
__global__ void __launch_bounds__(kThreads) bn_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ dy, int64_t M, int C,
                                                              const float* __restrict__ mean,
                                                              const float* __restrict__ var, float eps,
                                                              float* __restrict__ part) {
  __shared__ float red[2][kThreads * 8];
  const int G8 = C / 8;
  const int G = G8 < kThreads ? G8 : kThreads;
  const int RP = kThreads / G;
  const int t = threadIdx.x;
  const int gl = t % G, ph = t / G;
  const int P = gridDim.x;
  const int64_t rows = (M + P - 1) / P;
  const int64_t r0 = blockIdx.x * rows;
  const int64_t r1 = r0 + rows < M ? r0 + rows : M;
  for (int gbase = 0; gbase < G8; gbase += G) {
    const int g = gbase + gl;
    float s1[8] = {0, 0, 0, 0, 0, 0, 0, 0}, s2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float mu[8], is[8];
    if (MODE == 1 && ph < RP && g < G8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        mu[j] = mean[g * 8 + j];
        is[j] = rsqrtf(var[g * 8 + j] + eps);
      }
    }
    if (ph < RP && g < G8) {
      for (int64_t r = r0 + ph; r < r1; r += RP) {
        float a[8];
        unpack8(*reinterpret_cast<const uint4*>(x + r * C + g * 8), a);
        if (MODE == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            s1[j] += a[j];
            s2[j] = fmaf(a[j], a[j], s2[j]);
          }
        } else {
          float d[8];
          unpack8(*reinterpret_cast<const uint4*>(dy + r * C + g * 8), d);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            s1[j] += d[j];
            s2[j] = fmaf(d[j], (a[j] - mu[j]) * is[j], s2[j]);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      red[0][t * 8 + j] = s1[j];
      red[1][t * 8 + j] = s2[j];
    }
    __syncthreads();
    if (ph == 0 && g < G8) {          // combine the row phases in phase order
      for (int q = 1; q < RP; ++q)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s1[j] += red[0][(q * G + gl) * 8 + j];
          s2[j] += red[1][(q * G + gl) * 8 + j];
        }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        part[(static_cast<size_t>(blockIdx.x) * 2 + 0) * C + g * 8 + j] = s1[j];
        part[(static_cast<size_t>(blockIdx.x) * 2 + 1) * C + g * 8 + j] = s2[j];
      }
    }
    __syncthreads();
  }
}

// Combine the P partials of every channel in block order (fp64).
// MODE 0 -> mean, biased var; MODE 1 -> dbeta = sum dy, dgamma = sum dy*xhat.
template <int MODE>
__global__ void bn_finalize_kernel(const float* __restrict__ part, int P, int64_t M, int C, float* __restrict__ o1,
                                   float* __restrict__ o2) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double a = 0.0, b = 0.0;
  for (int p = 0; p < P; ++p) {
    a += part[(static_cast<size_t>(p) * 2 + 0) * C + c];
    b += part[(static_cast<size_t>(p) * 2 + 1) * C + c];
  }
  if (MODE == 0) {
    const double mu = a / static_cast<double>(M);
    double v = b / static_cast<double>(M) - mu * mu;
    o1[c] = static_cast<float>(mu);
    o2[c] = static_cast<float>(v > 0.0 ? v : 0.0);
  } else {
    o1[c] = static_cast<float>(b);   // dgamma
    o2[c] = static_cast<float>(a);   // dbeta
  }
}

// y = act(gamma (x - mean) invstd + beta)
__global__ void __launch_bounds__(kThreads) bn_apply_kernel(const __nv_bfloat16* x, int64_t M, int C,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ beta,
                                                            const float* __restrict__ mean,
                                                            const float* __restrict__ var, float eps, int relu,
                                                            __nv_bfloat16* y) {
  const int G8 = C / 8;
  const int64_t n8 = M * G8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % G8) * 8;
    float a[8];
    unpack8(reinterpret_cast<const uint4*>(x)[i], a);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float is = rsqrtf(var[c0 + j] + eps);
      float v = fmaf(gamma[c0 + j] * is, a[j] - mean[c0 + j], beta[c0 + j]);
      a[j] = relu ? fmaxf(v, 0.0f) : v;
    }
    reinterpret_cast<uint4*>(y)[i] = pack8(a);
  }
}

// dx = gamma invstd (dy - dbeta/M - xhat dgamma/M)
__global__ void __launch_bounds__(kThreads) bn_bwd_apply_kernel(
    const __nv_bfloat16* x, const __nv_bfloat16* dy, int64_t M, int C,  // dx may alias dy (same-thread element)
    const float* __restrict__ gamma, const float* __restrict__ mean, const float* __restrict__ var, float eps,
    const float* __restrict__ dgamma, const float* __restrict__ dbeta, __nv_bfloat16* dx) {
  const int G8 = C / 8;
  const int64_t n8 = M * G8;
  const float invM = 1.0f / static_cast<float>(M);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % G8) * 8;
    float a[8], d[8];
    unpack8(reinterpret_cast<const uint4*>(x)[i], a);
    unpack8(reinterpret_cast<const uint4*>(dy)[i], d);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      const float is = rsqrtf(var[c] + eps);
      const float xh = (a[j] - mean[c]) * is;
      a[j] = gamma[c] * is * (d[j] - dbeta[c] * invM - xh * dgamma[c] * invM);
    }
    reinterpret_cast<uint4*>(dx)[i] = pack8(a);
  }
}

__global__ void __launch_bounds__(kThreads) relu_bwd_kernel(const __nv_bfloat16* x,
                                                            const __nv_bfloat16* dy, int64_t n8,
                                                            int six, __nv_bfloat16* dx) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float a[8], d[8];
    unpack8(reinterpret_cast<const uint4*>(x)[i], a);
    unpack8(reinterpret_cast<const uint4*>(dy)[i], d);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = (a[j] > 0.0f && (!six || a[j] < 6.0f)) ? d[j] : 0.0f;
    reinterpret_cast<uint4*>(dx)[i] = pack8(d);
  }
}

// One thread per (input pixel, 8-channel group): gathers the gradients of the
// windows that cover it and whose first maximum it is, in (ho, wo) order.
__global__ void __launch_bounds__(kThreads) maxpool_bwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ dy, int N, int H,
                                                               int W, int C, int KH, int KW, int S, int ph, int pw,
                                                               int Ho, int Wo, __nv_bfloat16* __restrict__ dx) {
  const int G8 = C / 8;
  const int64_t total = static_cast<int64_t>(N) * H * W * G8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int wi = static_cast<int>(pix % W), hi = static_cast<int>((pix / W) % H), n = static_cast<int>(pix / (static_cast<int64_t>(W) * H));
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // windows with ho*S - ph <= hi <= ho*S - ph + KH - 1
    int ho0 = hi + ph - KH + 1;
    ho0 = ho0 <= 0 ? 0 : (ho0 + S - 1) / S;
    int ho1 = (hi + ph) / S;
    ho1 = ho1 < Ho - 1 ? ho1 : Ho - 1;
    int wo0 = wi + pw - KW + 1;
    wo0 = wo0 <= 0 ? 0 : (wo0 + S - 1) / S;
    int wo1 = (wi + pw) / S;
    wo1 = wo1 < Wo - 1 ? wo1 : Wo - 1;
    for (int ho = ho0; ho <= ho1; ++ho)
      for (int wo = wo0; wo <= wo1; ++wo) {
        float best[8];
        int arg[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) { best[j] = -INFINITY; arg[j] = -1; }
        for (int r = 0; r < KH; ++r) {
          const int hh = ho * S - ph + r;
          if (hh < 0 || hh >= H) continue;
          for (int s = 0; s < KW; ++s) {
            const int ww = wo * S - pw + s;
            if (ww < 0 || ww >= W) continue;
            float v[8];
            unpack8(*reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hh) * W + ww) * C + g * 8), v);
            const int id = hh * W + ww;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (arg[j] < 0 || v[j] > best[j]) { best[j] = v[j]; arg[j] = id; }
          }
        }
        float d[8];
        unpack8(*reinterpret_cast<const uint4*>(dy + ((static_cast<int64_t>(n) * Ho + ho) * Wo + wo) * C + g * 8), d);
        const int me = hi * W + wi;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (arg[j] == me) acc[j] += d[j];
      }
    reinterpret_cast<uint4*>(dx)[i] = pack8(acc);
  }
}

__global__ void __launch_bounds__(kThreads) gap_bwd_kernel(const float* __restrict__ dy, int N, int HW, int C,
                                                           __nv_bfloat16* __restrict__ dx) {
  const int G8 = C / 8;
  const int64_t total = static_cast<int64_t>(N) * HW * G8;
  const float inv = 1.0f / static_cast<float>(HW);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % G8);
    const int n = static_cast<int>(i / (static_cast<int64_t>(HW) * G8));
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = dy[static_cast<int64_t>(n) * C + g * 8 + j] * inv;
    reinterpret_cast<uint4*>(dx)[i] = pack8(v);
  }
}

// one block per row: fixed-order tree reductions for the max and the sum
__global__ void __launch_bounds__(kThreads) softmax_ce_kernel(const float* z,
                                                              const int32_t* __restrict__ labels, int N, int Cls,
                                                              float* dz, float* __restrict__ rowloss) {
  __shared__ float red[kThreads];
  const int n = blockIdx.x, t = threadIdx.x;
  const float* zr = z + static_cast<int64_t>(n) * Cls;
  float m = -INFINITY;
  for (int j = t; j < Cls; j += kThreads) m = fmaxf(m, zr[j]);
  red[t] = m;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (t < s) red[t] = fmaxf(red[t], red[t + s]);
    __syncthreads();
  }
  m = red[0];
  __syncthreads();
  float sum = 0.0f;
  for (int j = t; j < Cls; j += kThreads) sum += expf(zr[j] - m);
  red[t] = sum;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (t < s) red[t] += red[t + s];
    __syncthreads();
  }
  sum = red[0];
  const int lab = labels[n];
  const bool ok = lab >= 0 && lab < Cls;
  const float zl = ok ? zr[lab] : 0.0f;   // read before dz (which may alias z) is written
  __syncthreads();
  const float invN = 1.0f / static_cast<float>(N);
  for (int j = t; j < Cls; j += kThreads)
    dz[static_cast<int64_t>(n) * Cls + j] = (expf(zr[j] - m) / sum - (j == lab ? 1.0f : 0.0f)) * invN;
  if (t == 0) rowloss[n] = ok ? (logf(sum) + m) - zl : NAN;
}

__global__ void mean_kernel(const float* __restrict__ v, int N, float* __restrict__ out) {
  double a = 0.0;
  for (int i = 0; i < N; ++i) a += v[i];
  *out = static_cast<float>(a / N);
}

__global__ void __launch_bounds__(kThreads) sgd_kernel(float* __restrict__ w, const float* __restrict__ g,
                                                       float* __restrict__ buf, int64_t n, float lr, float mom,
                                                       int first) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float b = first ? g[i] : fmaf(mom, buf[i], g[i]);
    buf[i] = b;
    w[i] = fmaf(-lr, b, w[i]);
  }
}

int grid_for(int64_t work) {
  int64_t b = (work + kThreads - 1) / kThreads;
  const int64_t cap = 148 * 8;   // 8 resident 256-thread CTAs per SM
  return static_cast<int>(b < cap ? (b < 1 ? 1 : b) : cap);
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

extern "C" {

int32_t gacer_bn_partials(int64_t M, int32_t C) {
  (void)C;
  return M < 1 ? 0 : num_partials(M);
}

int32_t gacer_bn_train_fwd(const void* x_dev, int64_t M, int32_t C, const float* gamma_dev, const float* beta_dev,
                           float eps, int32_t relu, void* y_dev, float* mean_dev, float* var_dev, float* scratch_dev,
                           void* stream) {
  if (M < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "bn_train_fwd: need M >= 1 and C % 8 == 0");
  if (!x_dev || !y_dev || !gamma_dev || !beta_dev || !mean_dev || !var_dev || !scratch_dev ||
      !aligned16(x_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "bn_train_fwd: null or misaligned pointer");
  auto s = static_cast<cudaStream_t>(stream);
  const int P = num_partials(M);
  const auto* x = static_cast<const __nv_bfloat16*>(x_dev);
  bn_partial_kernel<0><<<P, kThreads, 0, s>>>(x, nullptr, M, C, nullptr, nullptr, 0.0f, scratch_dev);
  bn_finalize_kernel<0><<<(C + 127) / 128, 128, 0, s>>>(scratch_dev, P, M, C, mean_dev, var_dev);
  bn_apply_kernel<<<grid_for(M * (C / 8)), kThreads, 0, s>>>(x, M, C, gamma_dev, beta_dev, mean_dev, var_dev, eps,
                                                             relu, static_cast<__nv_bfloat16*>(y_dev));
  return launched("bn_train_fwd");
}

int32_t gacer_bn_train_bwd(const void* x_dev, const void* dy_dev, int64_t M, int32_t C, const float* gamma_dev,
                           const float* mean_dev, const float* var_dev, float eps, void* dx_dev, float* dgamma_dev,
                           float* dbeta_dev, float* scratch_dev, void* stream) {
  if (M < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "bn_train_bwd: need M >= 1 and C % 8 == 0");
  if (!x_dev || !dy_dev || !dx_dev || !gamma_dev || !mean_dev || !var_dev || !dgamma_dev || !dbeta_dev ||
      !scratch_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev))
    return bad(GACER_E_INVALID_ARG, "bn_train_bwd: null or misaligned pointer");
  auto s = static_cast<cudaStream_t>(stream);
  const int P = num_partials(M);
  const auto* x = static_cast<const __nv_bfloat16*>(x_dev);
  const auto* dy = static_cast<const __nv_bfloat16*>(dy_dev);
  bn_partial_kernel<1><<<P, kThreads, 0, s>>>(x, dy, M, C, mean_dev, var_dev, eps, scratch_dev);
  bn_finalize_kernel<1><<<(C + 127) / 128, 128, 0, s>>>(scratch_dev, P, M, C, dgamma_dev, dbeta_dev);
  bn_bwd_apply_kernel<<<grid_for(M * (C / 8)), kThreads, 0, s>>>(x, dy, M, C, gamma_dev, mean_dev, var_dev, eps,
                                                                 dgamma_dev, dbeta_dev,
                                                                 static_cast<__nv_bfloat16*>(dx_dev));
  return launched("bn_train_bwd");
}

int32_t gacer_relu_bwd(const void* x_dev, const void* dy_dev, int64_t n, int32_t six, void* dx_dev, void* stream) {
  if (n < 0 || n % 8) return bad(GACER_E_SHAPE, "relu_bwd: n % 8 != 0");
  if (!x_dev || !dy_dev || !dx_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev))
    return bad(GACER_E_INVALID_ARG, "relu_bwd: null or misaligned pointer");
  if (n == 0) return GACER_OK;
  relu_bwd_kernel<<<grid_for(n / 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x_dev), static_cast<const __nv_bfloat16*>(dy_dev), n / 8, six,
      static_cast<__nv_bfloat16*>(dx_dev));
  return launched("relu_bwd");
}

int32_t gacer_maxpool_bwd(const void* x_dev, const void* dy_dev, int32_t N, int32_t H, int32_t W, int32_t C,
                          int32_t KH, int32_t KW, int32_t stride, int32_t ph, int32_t pw, int32_t Ho, int32_t Wo,
                          void* dx_dev, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || KH < 1 || KW < 1 || stride < 1 || ph < 0 || pw < 0 ||
      Ho != (H + 2 * ph - KH) / stride + 1 || Wo != (W + 2 * pw - KW) / stride + 1 || Ho < 1 || Wo < 1)
    return bad(GACER_E_SHAPE, "maxpool_bwd: inconsistent shape");
  if (!x_dev || !dy_dev || !dx_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev))
    return bad(GACER_E_INVALID_ARG, "maxpool_bwd: null or misaligned pointer");
  maxpool_bwd_kernel<<<grid_for(static_cast<int64_t>(N) * H * W * (C / 8)), kThreads, 0,
                       static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x_dev), static_cast<const __nv_bfloat16*>(dy_dev), N, H, W, C, KH, KW,
      stride, ph, pw, Ho, Wo, static_cast<__nv_bfloat16*>(dx_dev));
  return launched("maxpool_bwd");
}

int32_t gacer_gap_bwd(const float* dy_dev, int32_t N, int32_t HW, int32_t C, void* dx_dev, void* stream) {
  if (N < 1 || HW < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "gap_bwd: need C % 8 == 0");
  if (!dy_dev || !dx_dev || !aligned16(dx_dev)) return bad(GACER_E_INVALID_ARG, "gap_bwd: null or misaligned pointer");
  gap_bwd_kernel<<<grid_for(static_cast<int64_t>(N) * HW * (C / 8)), kThreads, 0,
                   static_cast<cudaStream_t>(stream)>>>(dy_dev, N, HW, C, static_cast<__nv_bfloat16*>(dx_dev));
  return launched("gap_bwd");
}

int32_t gacer_softmax_ce(const float* z_dev, const int32_t* labels_dev, int32_t N, int32_t Cls, float* loss_dev,
                         float* dz_dev, float* scratch_dev, void* stream) {
  if (N < 1 || Cls < 1) return bad(GACER_E_SHAPE, "softmax_ce: need N, Cls >= 1");
  if (!z_dev || !labels_dev || !loss_dev || !dz_dev || !scratch_dev)
    return bad(GACER_E_INVALID_ARG, "softmax_ce: null pointer");
  auto s = static_cast<cudaStream_t>(stream);
  softmax_ce_kernel<<<N, kThreads, 0, s>>>(z_dev, labels_dev, N, Cls, dz_dev, scratch_dev);
  mean_kernel<<<1, 1, 0, s>>>(scratch_dev, N, loss_dev);
  return launched("softmax_ce");
}

int32_t gacer_sgd_momentum(float* w_dev, const float* g_dev, float* buf_dev, int64_t n, float lr, float momentum,
                           int32_t first, void* stream) {
  if (n < 0) return bad(GACER_E_SHAPE, "sgd_momentum: n < 0");
  if (!w_dev || !g_dev || !buf_dev) return bad(GACER_E_INVALID_ARG, "sgd_momentum: null pointer");
  if (n == 0) return GACER_OK;
  sgd_kernel<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(w_dev, g_dev, buf_dev, n, lr, momentum,
                                                                              first);
  return launched("sgd_momentum");
}

}  // extern "C"
