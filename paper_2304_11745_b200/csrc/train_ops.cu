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
// Four rows per thread are loaded before they are summed (16-byte loads in
// flight: 4 x 4 KB per CTA); each thread still sums its rows in row order.
constexpr int kUnroll = 4;

template <int MODE>
__global__ void __launch_bounds__(kThreads) bn_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ dy,
                                                              const __nv_bfloat16* __restrict__ ym, int64_t M, int C,
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
      for (int64_t r = r0 + ph; r < r1; r += kUnroll * RP) {
        uint4 va[kUnroll], vd[kUnroll], vm[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t rr = r + u * RP;
          va[u] = rr < r1 ? __ldcs(reinterpret_cast<const uint4*>(x + rr * C + g * 8)) : make_uint4(0, 0, 0, 0);
          if (MODE == 1) {
            vd[u] = rr < r1 ? __ldcs(reinterpret_cast<const uint4*>(dy + rr * C + g * 8)) : make_uint4(0, 0, 0, 0);
            vm[u] = (ym && rr < r1) ? __ldcs(reinterpret_cast<const uint4*>(ym + rr * C + g * 8)) : make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          if (r + u * RP >= r1) break;
          float a[8];
          unpack8(va[u], a);
          if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              s1[j] += a[j];
              s2[j] = fmaf(a[j], a[j], s2[j]);
            }
          } else {
            float d[8];
            unpack8(vd[u], d);
            if (ym) {                        // fused ReLU backward: the mask of the BN's ReLU output
              float mk[8];
              unpack8(vm[u], mk);
#pragma unroll
              for (int j = 0; j < 8; ++j) d[j] = mk[j] > 0.0f ? d[j] : 0.0f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              s1[j] += d[j];
              s2[j] = fmaf(d[j], (a[j] - mu[j]) * is[j], s2[j]);
            }
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

// Combine the P partials of every channel in block order (fp64), then fold
// the per-channel constants of the apply pass into `coef` (fp32 [k][C]):
//   MODE 0 -> mean, biased var; coef = (scale, shift): y = x * scale + shift
//   MODE 1 -> dgamma = sum dy*xhat, dbeta = sum dy; coef = (a, b, c):
//             dx = a * dy + b * x + c  (the BN-backward formula expanded in x)
template <int MODE>
__global__ void bn_finalize_kernel(const float* __restrict__ part, int P, int64_t M, int C,
                                   const float* __restrict__ gamma, const float* __restrict__ beta,
                                   const float* __restrict__ mean_in, const float* __restrict__ var_in, float eps,
                                   float* __restrict__ o1, float* __restrict__ o2, float* __restrict__ coef) {
  // 32 channels per CTA, lane = channel (coalesced rows of the partials);
  // warp w sums the partials p = w, w+8, ... in order, then warp 0 adds the
  // eight warp sums in warp order (the same order on every run)
  __shared__ double red[2][8][32];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double a = 0.0, b = 0.0;
  if (c < C) {
    int p = wp;
    for (; p + 24 < P; p += 32) {     // four partials' loads in flight, summed in order
      float x0[4], x1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = part[(static_cast<size_t>(p + 8 * u) * 2 + 0) * C + c];
        x1[u] = part[(static_cast<size_t>(p + 8 * u) * 2 + 1) * C + c];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a += x0[u];
        b += x1[u];
      }
    }
    for (; p < P; p += 8) {
      a += part[(static_cast<size_t>(p) * 2 + 0) * C + c];
      b += part[(static_cast<size_t>(p) * 2 + 1) * C + c];
    }
  }
  red[0][wp][lane] = a;
  red[1][wp][lane] = b;
  __syncthreads();
  if (wp != 0 || c >= C) return;
  a = red[0][0][lane];
  b = red[1][0][lane];
  for (int q = 1; q < 8; ++q) {
    a += red[0][q][lane];
    b += red[1][q][lane];
  }
  const double Md = static_cast<double>(M);
  if (MODE == 0) {
    const double mu = a / Md;
    double v = b / Md - mu * mu;
    v = v > 0.0 ? v : 0.0;
    o1[c] = static_cast<float>(mu);
    o2[c] = static_cast<float>(v);
    const double sc = gamma[c] / sqrt(static_cast<double>(static_cast<float>(v)) + eps);
    coef[c] = static_cast<float>(sc);
    coef[C + c] = static_cast<float>(beta[c] - static_cast<double>(static_cast<float>(mu)) * sc);
  } else {
    o1[c] = static_cast<float>(b);   // dgamma
    o2[c] = static_cast<float>(a);   // dbeta
    const double is = 1.0 / sqrt(static_cast<double>(var_in[c]) + eps);
    const double gi = gamma[c] * is;
    const double k = gi * is * static_cast<double>(static_cast<float>(b)) / Md;
    coef[c] = static_cast<float>(gi);
    coef[C + c] = static_cast<float>(-k);
    coef[2 * C + c] = static_cast<float>(-gi * static_cast<double>(static_cast<float>(a)) / Md + k * mean_in[c]);
  }
}

// y = act(x * scale + shift); dx = a * dy + b * x + c.  Grid-stride over
// 8-channel groups; the stride is a multiple of C/8 whenever C/8 divides 256
// (every ResNet width), so a thread's channels are fixed and its constants
// stay in registers.
template <int MODE>
__global__ void __launch_bounds__(kThreads) bn_elementwise_kernel(const __nv_bfloat16* x, const __nv_bfloat16* dy,
                                                                  const __nv_bfloat16* ym,
                                                                  int64_t M, int C, const float* __restrict__ coef,
                                                                  int relu, __nv_bfloat16* out) {
  const int G8 = C / 8;
  const int64_t n8 = M * G8;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool fixed = (stride % G8) == 0;
  float k0[8], k1[8], k2[8];
  int c0 = -1;
  for (; i < n8; i += stride) {
    const int c = (fixed && c0 >= 0) ? c0 : static_cast<int>(i % G8) * 8;
    if (c != c0) {
      c0 = c;
      const float4* q0 = reinterpret_cast<const float4*>(coef + c);
      const float4* q1 = reinterpret_cast<const float4*>(coef + C + c);
      float4 u = q0[0], v = q0[1], w = q1[0], z = q1[1];
      k0[0] = u.x; k0[1] = u.y; k0[2] = u.z; k0[3] = u.w; k0[4] = v.x; k0[5] = v.y; k0[6] = v.z; k0[7] = v.w;
      k1[0] = w.x; k1[1] = w.y; k1[2] = w.z; k1[3] = w.w; k1[4] = z.x; k1[5] = z.y; k1[6] = z.z; k1[7] = z.w;
      if (MODE == 1) {
        const float4* q2 = reinterpret_cast<const float4*>(coef + 2 * C + c);
        float4 p = q2[0], q = q2[1];
        k2[0] = p.x; k2[1] = p.y; k2[2] = p.z; k2[3] = p.w; k2[4] = q.x; k2[5] = q.y; k2[6] = q.z; k2[7] = q.w;
      }
    }
    float a[8];
    unpack8(__ldcs(reinterpret_cast<const uint4*>(x) + i), a);
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float v = fmaf(a[j], k0[j], k1[j]);
        a[j] = relu ? fmaxf(v, 0.0f) : v;
      }
    } else {
      float d[8];
      unpack8(__ldcs(reinterpret_cast<const uint4*>(dy) + i), d);
      if (ym) {
        float mk[8];
        unpack8(__ldcs(reinterpret_cast<const uint4*>(ym) + i), mk);
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = mk[j] > 0.0f ? d[j] : 0.0f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(k0[j], d[j], fmaf(k1[j], a[j], k2[j]));
    }
    __stcs(reinterpret_cast<uint4*>(out) + i, pack8(a));
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

// Max-pool backward in two passes.  Pass 1, one thread per (output window,
// 8-channel group): the window's first maximum per channel (row-major tap
// order, padded taps skipped) as a tap index byte.  Pass 2, one thread per
// (input pixel, 8-channel group): gathers dy of the windows covering the
// pixel whose recorded tap is this pixel, in (ho, wo) order -- no atomics.
__global__ void __launch_bounds__(kThreads) maxpool_argmax_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                                  int W, int C, int KH, int KW, int S, int ph, int pw,
                                                                  int Ho, int Wo, uint8_t* __restrict__ arg) {
  const int G8 = C / 8;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * G8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int wo = static_cast<int>(pix % Wo), ho = static_cast<int>((pix / Wo) % Ho);
    const int n = static_cast<int>(pix / (static_cast<int64_t>(Wo) * Ho));
    float best[8];
    uint32_t tap[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { best[j] = -INFINITY; tap[j] = 255u; }
    for (int r = 0; r < KH; ++r) {
      const int hh = ho * S - ph + r;
      if (hh < 0 || hh >= H) continue;
      for (int q = 0; q < KW; ++q) {
        const int ww = wo * S - pw + q;
        if (ww < 0 || ww >= W) continue;
        float v[8];
        unpack8(*reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hh) * W + ww) * C + g * 8), v);
        const uint32_t id = static_cast<uint32_t>(r * KW + q);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (tap[j] == 255u || v[j] > best[j]) { best[j] = v[j]; tap[j] = id; }
      }
    }
    uint2 o;
    o.x = tap[0] | (tap[1] << 8) | (tap[2] << 16) | (tap[3] << 24);
    o.y = tap[4] | (tap[5] << 8) | (tap[6] << 16) | (tap[7] << 24);
    reinterpret_cast<uint2*>(arg)[i] = o;
  }
}

__global__ void __launch_bounds__(kThreads) maxpool_bwd_kernel(const uint8_t* __restrict__ arg,
                                                               const __nv_bfloat16* __restrict__ dy, int N, int H,
                                                               int W, int C, int KH, int KW, int S, int ph, int pw,
                                                               int Ho, int Wo, __nv_bfloat16* __restrict__ dx) {
  const int G8 = C / 8;
  const int64_t total = static_cast<int64_t>(N) * H * W * G8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int wi = static_cast<int>(pix % W), hi = static_cast<int>((pix / W) % H);
    const int n = static_cast<int>(pix / (static_cast<int64_t>(W) * H));
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
        const int64_t o = ((static_cast<int64_t>(n) * Ho + ho) * Wo + wo) * G8 + g;
        const uint2 t = reinterpret_cast<const uint2*>(arg)[o];
        const uint32_t me = static_cast<uint32_t>((hi - (ho * S - ph)) * KW + (wi - (wo * S - pw)));
        const uint32_t tt[8] = {t.x & 255u, (t.x >> 8) & 255u, (t.x >> 16) & 255u, t.x >> 24,
                                t.y & 255u, (t.y >> 8) & 255u, (t.y >> 16) & 255u, t.y >> 24};
        bool any = false;
#pragma unroll
        for (int j = 0; j < 8; ++j) any |= tt[j] == me;
        if (!any) continue;
        float d[8];
        unpack8(reinterpret_cast<const uint4*>(dy)[o], d);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (tt[j] == me) acc[j] += d[j];
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

// ---------------------------------------------------------------- forward
// (the training step's non-GEMM forward ops; the inference executor fuses
//  these into its work items, the training step still runs them per op)
__global__ void __launch_bounds__(kThreads) maxpool_fwd_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                               int W, int C, int KH, int KW, int S, int ph, int pw,
                                                               int Ho, int Wo, __nv_bfloat16* __restrict__ y) {
  const int G8 = C / 8;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * G8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int wo = static_cast<int>(pix % Wo), ho = static_cast<int>((pix / Wo) % Ho);
    const int n = static_cast<int>(pix / (static_cast<int64_t>(Wo) * Ho));
    float best[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) best[j] = -INFINITY;
    for (int r = 0; r < KH; ++r) {
      const int hh = ho * S - ph + r;
      if (hh < 0 || hh >= H) continue;
      for (int q = 0; q < KW; ++q) {
        const int ww = wo * S - pw + q;
        if (ww < 0 || ww >= W) continue;
        float v[8];
        unpack8(*reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hh) * W + ww) * C + g * 8), v);
#pragma unroll
        for (int j = 0; j < 8; ++j) best[j] = fmaxf(best[j], v[j]);
      }
    }
    reinterpret_cast<uint4*>(y)[i] = pack8(best);
  }
}

// y = a + b (then ReLU when relu != 0), bf16 [n], n % 8 == 0
__global__ void __launch_bounds__(kThreads) add_kernel(const __nv_bfloat16* a, const __nv_bfloat16* b, int64_t n8,
                                                       int relu, __nv_bfloat16* y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float u[8], v[8];
    unpack8(reinterpret_cast<const uint4*>(a)[i], u);
    unpack8(reinterpret_cast<const uint4*>(b)[i], v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float t = u[j] + v[j];
      u[j] = relu ? fmaxf(t, 0.0f) : t;
    }
    reinterpret_cast<uint4*>(y)[i] = pack8(u);
  }
}

// y[n][c] = (1/HW) sum_p x[n][p][c], summed in pixel order (fp32), bf16 out
__global__ void __launch_bounds__(kThreads) gap_fwd_kernel(const __nv_bfloat16* __restrict__ x, int N, int HW, int C,
                                                           __nv_bfloat16* __restrict__ y) {
  const int G8 = C / 8;
  const int64_t total = static_cast<int64_t>(N) * G8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % G8), n = static_cast<int>(i / G8);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < HW; ++p) {
      float v[8];
      unpack8(*reinterpret_cast<const uint4*>(x + (static_cast<int64_t>(n) * HW + p) * C + g * 8), v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += v[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] /= static_cast<float>(HW);
    reinterpret_cast<uint4*>(y)[i] = pack8(acc);
  }
}

// z[n][o] = b[o] + sum_k w[o][k] x[n][k] (x bf16, w fp32): one warp per
// output, lane l sums k = l, l+32, ... (coalesced rows of w and x), then a
// fixed xor-butterfly combines the lanes (deterministic)
__global__ void __launch_bounds__(kThreads) linear_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const float* __restrict__ w, const float* __restrict__ b,
                                                              int N, int K, int O, float* __restrict__ z) {
  const int64_t wid = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= static_cast<int64_t>(N) * O) return;
  const int n = static_cast<int>(wid / O), o = static_cast<int>(wid % O);
  const __nv_bfloat16* xr = x + static_cast<int64_t>(n) * K;
  const float* wr = w + static_cast<int64_t>(o) * K;
  float a = 0.0f;
  for (int k = lane; k < K; k += 32) a = fmaf(__bfloat162float(xr[k]), wr[k], a);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
  if (lane == 0) z[wid] = a + (b ? b[o] : 0.0f);
}

// FC backward: one output element per thread, reductions in index order
__global__ void __launch_bounds__(kThreads) linear_dx_kernel(const float* __restrict__ w, const float* __restrict__ dy,
                                                             int N, int K, int O, float* __restrict__ dx) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(N) * K) return;
  const int n = static_cast<int>(i / K), k = static_cast<int>(i % K);
  float a = 0.0f;
  for (int o = 0; o < O; ++o) a = fmaf(dy[static_cast<int64_t>(n) * O + o], w[static_cast<int64_t>(o) * K + k], a);
  dx[i] = a;
}

__global__ void __launch_bounds__(kThreads) linear_dw_kernel(const __nv_bfloat16* __restrict__ x,
                                                             const float* __restrict__ dy, int N, int K, int O,
                                                             float* __restrict__ dw, float* __restrict__ db) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(O) * K) return;
  const int o = static_cast<int>(i / K), k = static_cast<int>(i % K);
  float a = 0.0f;
  for (int n = 0; n < N; ++n)
    a = fmaf(dy[static_cast<int64_t>(n) * O + o], __bfloat162float(x[static_cast<int64_t>(n) * K + k]), a);
  dw[i] = a;
  if (db && k == 0) {
    float b = 0.0f;
    for (int n = 0; n < N; ++n) b += dy[static_cast<int64_t>(n) * O + o];
    db[o] = b;
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

namespace gacer {
// Conv data-gradient filter (stride 1): the forward filter w fp32
// [Cout][Cin][KH][KW] flipped and transposed into the K-major bf16 B operand
// of a forward conv over dy: row ci, column (r*KW + s)*cread + co holds
// w[co][ci][KH-1-r][KW-1-s]; padded rows/columns are zero.
// (forward = 1: the plain forward B operand, row co, column (r*KW + s)*cread + ci
//  holding w[co][ci][r][s])
__global__ void dgrad_filter_kernel(const float* __restrict__ w, int Cout, int Cin, int KH, int KW, int cread,
                                    int Kpad, int rows, int forward, __nv_bfloat16* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(rows) * Kpad;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / Kpad), k = static_cast<int>(i % Kpad);
    const int tap = k / cread, col = k % cread;
    float v = 0.0f;
    if (forward) {
      if (row < Cout && tap < KH * KW && col < Cin)
        v = w[((static_cast<int64_t>(row) * Cin + col) * KH + tap / KW) * KW + tap % KW];
    } else if (row < Cin && tap < KH * KW && col < Cout) {
      const int r = tap / KW, s = tap % KW;
      v = w[((static_cast<int64_t>(col) * Cin + row) * KH + (KH - 1 - r)) * KW + (KW - 1 - s)];
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

cudaError_t launch_dgrad_filter(const float* w, int Cout, int Cin, int KH, int KW, int cread, int Kpad, int rows,
                                void* out, cudaStream_t s) {
  dgrad_filter_kernel<<<grid_for(static_cast<int64_t>(rows) * Kpad), kThreads, 0, s>>>(
      w, Cout, Cin, KH, KW, cread, Kpad, rows, 0, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

cudaError_t launch_fwd_filter(const float* w, int Cout, int Cin, int KH, int KW, int cread, int Kpad, int rows,
                              void* out, cudaStream_t s) {
  dgrad_filter_kernel<<<grid_for(static_cast<int64_t>(rows) * Kpad), kThreads, 0, s>>>(
      w, Cout, Cin, KH, KW, cread, Kpad, rows, 1, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

// Zero-dilated dy for a strided conv's data gradient: dyd[n][hh][ww][c] =
// dy[n][hh/S][ww/S][c] when S divides hh and ww, else 0; Hdd x Wdd output.
__global__ void dilate_kernel(const __nv_bfloat16* __restrict__ dy, int N, int Hd, int Wd, int C, int S, int Hdd,
                              int Wdd, __nv_bfloat16* __restrict__ out) {
  const int G8 = C / 8;
  const int64_t total = static_cast<int64_t>(N) * Hdd * Wdd * G8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int ww = static_cast<int>(pix % Wdd), hh = static_cast<int>((pix / Wdd) % Hdd);
    const int n = static_cast<int>(pix / (static_cast<int64_t>(Wdd) * Hdd));
    uint4 v = make_uint4(0, 0, 0, 0);
    if (hh % S == 0 && ww % S == 0 && hh / S < Hd && ww / S < Wd)
      v = *reinterpret_cast<const uint4*>(dy + ((static_cast<int64_t>(n) * Hd + hh / S) * Wd + ww / S) * C + g * 8);
    reinterpret_cast<uint4*>(out)[i] = v;
  }
}

cudaError_t launch_dilate(const void* dy, int N, int Hd, int Wd, int C, int S, int Hdd, int Wdd, void* out,
                          cudaStream_t s) {
  dilate_kernel<<<grid_for(static_cast<int64_t>(N) * Hdd * Wdd * (C / 8)), kThreads, 0, s>>>(
      static_cast<const __nv_bfloat16*>(dy), N, Hd, Wd, C, S, Hdd, Wdd, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

// Weight-gradient operands: both GEMM operands K-major along the pixel
// index m (the reduction), i.e. the transposes of the NHWC tensors, row
// stride Kpad, zero-filled past M.  64x64 smem tiles keep reads and writes
// coalesced and 16 bytes wide.  Tap t = (r, s) of the im2col operand reads x at
// (ho*S - p + r, wo*S - p + s) (zero outside the image).
__global__ void __launch_bounds__(256) transpose_im2col_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                               int W, int C, int Ho, int Wo, int KW, int S, int ph,
                                                               int pw, int64_t M, int Kpad,
                                                               __nv_bfloat16* __restrict__ out) {
  // 64 pixels x 64 channels per CTA: 16-byte loads along the channels,
  // a transposed smem tile, 16-byte stores along the pixels
  // [channel][pixel] tile, 16-byte pixel blocks XOR-swizzled by the channel
  // octet: the transposing scalar stores of a warp hit 32 distinct banks and
  // the 16-byte row reads stay contiguous
  constexpr int T = 64;
  __shared__ __align__(16) __nv_bfloat16 tile[T * T];
  auto at = [](int c, int i) { return c * T + ((((i >> 3) ^ (c >> 3)) & 7) << 3) + (i & 7); };
  const int t = blockIdx.z;
  const int r = t / KW, q = t % KW;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * T;
  const int c0 = blockIdx.y * T;
  const bool vec = (C % 8) == 0;
  for (int e = threadIdx.x; e < T * (T / 8); e += blockDim.x) {
    const int i = e / (T / 8), cg = (e % (T / 8)) * 8;        // pixel row i, channel group cg
    const int64_t m = m0 + i;
    __nv_bfloat16 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __float2bfloat16_rn(0.0f);
    if (m < M && c0 + cg < C) {
      const uint32_t m32 = static_cast<uint32_t>(m);        // M < 2^30 (checked on the host): 32-bit division
      const uint32_t pq = m32 / static_cast<uint32_t>(Wo);   // (n, ho) of the pixel
      const int wo = static_cast<int>(m32 - pq * static_cast<uint32_t>(Wo));
      const int n = static_cast<int>(pq / static_cast<uint32_t>(Ho));
      const int ho = static_cast<int>(pq - static_cast<uint32_t>(n) * static_cast<uint32_t>(Ho));
      const int hi = ho * S - ph + r, wi = wo * S - pw + q;
      if (hi >= 0 && hi < H && wi >= 0 && wi < W) {
        const __nv_bfloat16* src = x + ((static_cast<int64_t>(n) * H + hi) * W + wi) * C + c0 + cg;
        if (vec) {
          const uint4 u = *reinterpret_cast<const uint4*>(src);
          const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = h[j];
        } else {
          for (int j = 0; j < 8 && c0 + cg + j < C; ++j) v[j] = src[j];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) tile[at(cg + j, i)] = v[j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < T * (T / 8); e += blockDim.x) {
    const int cc = e / (T / 8), mg = (e % (T / 8)) * 8;       // channel row cc, pixel group mg
    const int c = c0 + cc;
    const int64_t m = m0 + mg;
    if (c < C && m < Kpad)                                      // Kpad is a multiple of 64: whole groups
      *reinterpret_cast<uint4*>(out + (static_cast<int64_t>(t) * C + c) * Kpad + m) =
          *reinterpret_cast<const uint4*>(&tile[at(cc, mg)]);
  }
}

cudaError_t launch_transpose_im2col(const void* x, int N, int H, int W, int C, int Ho, int Wo, int KH, int KW, int S,
                                    int ph, int pw, int64_t M, int Kpad, void* out, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>((Kpad + 63) / 64), static_cast<unsigned>((C + 63) / 64),
                  static_cast<unsigned>(KH * KW));
  transpose_im2col_kernel<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), N, H, W, C, Ho, Wo, KW, S, ph,
                                               pw, M, Kpad, static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

// dW from the GEMM's [Cout][(r*KW + s)*Cin + ci] order to the master
// weights' [Cout][Cin][KH][KW] order.
__global__ void wgrad_permute_kernel(const float* __restrict__ g, int Cout, int Cin, int KH, int KW,
                                     float* __restrict__ dw) {
  const int64_t total = static_cast<int64_t>(Cout) * Cin * KH * KW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(i % KW), r = static_cast<int>((i / KW) % KH);
    const int ci = static_cast<int>((i / (KW * KH)) % Cin), co = static_cast<int>(i / (static_cast<int64_t>(KW) * KH * Cin));
    dw[i] = g[static_cast<int64_t>(co) * (KH * KW * Cin) + (r * KW + s) * Cin + ci];
  }
}

// Weight-gradient split-K reduction: the GEMM's per-split partial tiles
// (layout [tile][split][bn/4][128 rows] float4) summed in split order, written
// straight into dW's master [Cout][Cin][KH][KW] layout.  One thread per
// (4-column group, row): consecutive threads read consecutive float4 rows.
__global__ void __launch_bounds__(kThreads) wgrad_reduce_kernel(const float* __restrict__ part, int Cout, int Cin,
                                                                int KH, int KW, int bn, int tiles_n, int split,
                                                                float* __restrict__ dw) {
  const int Ng = KH * KW * Cin;
  const int g4 = (Ng + 3) / 4;
  const int64_t total = static_cast<int64_t>(g4) * Cout;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int co = static_cast<int>(i % Cout), q = static_cast<int>(i / Cout);
    const int n0 = q * 4;
    const int tile = (co / 128) * tiles_n + n0 / bn;
    const int r = co % 128, c4 = (n0 % bn) / 4;
    const float4* src = reinterpret_cast<const float4*>(part) +
                        (static_cast<int64_t>(tile) * split * (bn / 4) + c4) * 128 + r;
    float4 a = src[0];
    for (int ks = 1; ks < split; ++ks) {
      const float4 b = src[static_cast<int64_t>(ks) * (bn / 4) * 128];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    const float v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + j;
      if (n >= Ng) break;
      const int tap = n / Cin, ci = n % Cin;
      dw[((static_cast<int64_t>(co) * Cin + ci) * KH + tap / KW) * KW + tap % KW] = v[j];
    }
  }
}

cudaError_t launch_wgrad_reduce(const float* part, int Cout, int Cin, int KH, int KW, int bn, int tiles_n, int split,
                                float* dw, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>((KH * KW * Cin + 3) / 4) * Cout;
  wgrad_reduce_kernel<<<grid_for(total), kThreads, 0, s>>>(part, Cout, Cin, KH, KW, bn, tiles_n, split, dw);
  return cudaGetLastError();
}

cudaError_t launch_wgrad_permute(const float* g, int Cout, int Cin, int KH, int KW, float* dw, cudaStream_t s) {
  wgrad_permute_kernel<<<grid_for(static_cast<int64_t>(Cout) * Cin * KH * KW), kThreads, 0, s>>>(g, Cout, Cin, KH, KW,
                                                                                                dw);
  return cudaGetLastError();
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
  float* coef = scratch_dev + static_cast<size_t>(P) * 2 * C;
  bn_partial_kernel<0><<<P, kThreads, 0, s>>>(x, nullptr, nullptr, M, C, nullptr, nullptr, 0.0f, scratch_dev);
  bn_finalize_kernel<0><<<(C + 31) / 32, 256, 0, s>>>(scratch_dev, P, M, C, gamma_dev, beta_dev, nullptr, nullptr,
                                                       eps, mean_dev, var_dev, coef);
  bn_elementwise_kernel<0><<<grid_for(M * (C / 8)), kThreads, 0, s>>>(x, nullptr, nullptr, M, C, coef, relu,
                                                                      static_cast<__nv_bfloat16*>(y_dev));
  return launched("bn_train_fwd");
}

int32_t gacer_bn_train_bwd(const void* x_dev, const void* dy_dev, const void* relu_y_dev, int64_t M, int32_t C,
                           const float* gamma_dev, const float* mean_dev, const float* var_dev, float eps, void* dx_dev,
                           float* dgamma_dev, float* dbeta_dev, float* scratch_dev, void* stream) {
  if (M < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "bn_train_bwd: need M >= 1 and C % 8 == 0");
  if (!x_dev || !dy_dev || !dx_dev || !gamma_dev || !mean_dev || !var_dev || !dgamma_dev || !dbeta_dev ||
      !scratch_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev) ||
      (relu_y_dev && !aligned16(relu_y_dev)))
    return bad(GACER_E_INVALID_ARG, "bn_train_bwd: null or misaligned pointer");
  const auto* ym = static_cast<const __nv_bfloat16*>(relu_y_dev);
  auto s = static_cast<cudaStream_t>(stream);
  const int P = num_partials(M);
  const auto* x = static_cast<const __nv_bfloat16*>(x_dev);
  const auto* dy = static_cast<const __nv_bfloat16*>(dy_dev);
  float* coef = scratch_dev + static_cast<size_t>(P) * 2 * C;
  bn_partial_kernel<1><<<P, kThreads, 0, s>>>(x, dy, ym, M, C, mean_dev, var_dev, eps, scratch_dev);
  bn_finalize_kernel<1><<<(C + 31) / 32, 256, 0, s>>>(scratch_dev, P, M, C, gamma_dev, nullptr, mean_dev, var_dev,
                                                       eps, dgamma_dev, dbeta_dev, coef);
  bn_elementwise_kernel<1><<<grid_for(M * (C / 8)), kThreads, 0, s>>>(x, dy, ym, M, C, coef, 0,
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
                          void* dx_dev, void* scratch_dev, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || KH < 1 || KW < 1 || KH * KW > 255 || stride < 1 || ph < 0 ||
      pw < 0 || Ho != (H + 2 * ph - KH) / stride + 1 || Wo != (W + 2 * pw - KW) / stride + 1 || Ho < 1 || Wo < 1)
    return bad(GACER_E_SHAPE, "maxpool_bwd: inconsistent shape");
  if (!x_dev || !dy_dev || !dx_dev || !scratch_dev || !aligned16(x_dev) || !aligned16(dy_dev) || !aligned16(dx_dev) ||
      (reinterpret_cast<uintptr_t>(scratch_dev) & 7u))
    return bad(GACER_E_INVALID_ARG, "maxpool_bwd: null or misaligned pointer");
  auto s = static_cast<cudaStream_t>(stream);
  auto* arg = static_cast<uint8_t*>(scratch_dev);
  maxpool_argmax_kernel<<<grid_for(static_cast<int64_t>(N) * Ho * Wo * (C / 8)), kThreads, 0, s>>>(
      static_cast<const __nv_bfloat16*>(x_dev), N, H, W, C, KH, KW, stride, ph, pw, Ho, Wo, arg);
  maxpool_bwd_kernel<<<grid_for(static_cast<int64_t>(N) * H * W * (C / 8)), kThreads, 0, s>>>(
      arg, static_cast<const __nv_bfloat16*>(dy_dev), N, H, W, C, KH, KW, stride, ph, pw, Ho, Wo,
      static_cast<__nv_bfloat16*>(dx_dev));
  return launched("maxpool_bwd");
}

int32_t gacer_gap_bwd(const float* dy_dev, int32_t N, int32_t HW, int32_t C, void* dx_dev, void* stream) {
  if (N < 1 || HW < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "gap_bwd: need C % 8 == 0");
  if (!dy_dev || !dx_dev || !aligned16(dx_dev)) return bad(GACER_E_INVALID_ARG, "gap_bwd: null or misaligned pointer");
  gap_bwd_kernel<<<grid_for(static_cast<int64_t>(N) * HW * (C / 8)), kThreads, 0,
                   static_cast<cudaStream_t>(stream)>>>(dy_dev, N, HW, C, static_cast<__nv_bfloat16*>(dx_dev));
  return launched("gap_bwd");
}

int32_t gacer_maxpool_fwd(const void* x_dev, int32_t N, int32_t H, int32_t W, int32_t C, int32_t KH, int32_t KW,
                          int32_t stride, int32_t ph, int32_t pw, int32_t Ho, int32_t Wo, void* y_dev, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || KH < 1 || KW < 1 || stride < 1 || ph < 0 || pw < 0 ||
      Ho != (H + 2 * ph - KH) / stride + 1 || Wo != (W + 2 * pw - KW) / stride + 1 || Ho < 1 || Wo < 1)
    return bad(GACER_E_SHAPE, "maxpool_fwd: inconsistent shape");
  if (!x_dev || !y_dev || !aligned16(x_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "maxpool_fwd: null or misaligned pointer");
  maxpool_fwd_kernel<<<grid_for(static_cast<int64_t>(N) * Ho * Wo * (C / 8)), kThreads, 0,
                       static_cast<cudaStream_t>(stream)>>>(static_cast<const __nv_bfloat16*>(x_dev), N, H, W, C, KH,
                                                            KW, stride, ph, pw, Ho, Wo,
                                                            static_cast<__nv_bfloat16*>(y_dev));
  return launched("maxpool_fwd");
}

int32_t gacer_add(const void* a_dev, const void* b_dev, int64_t n, int32_t relu, void* y_dev, void* stream) {
  if (n < 0 || n % 8) return bad(GACER_E_SHAPE, "add: n % 8 != 0");
  if (!a_dev || !b_dev || !y_dev || !aligned16(a_dev) || !aligned16(b_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "add: null or misaligned pointer");
  if (n == 0) return GACER_OK;
  add_kernel<<<grid_for(n / 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(a_dev), static_cast<const __nv_bfloat16*>(b_dev), n / 8, relu,
      static_cast<__nv_bfloat16*>(y_dev));
  return launched("add");
}

int32_t gacer_gap_fwd(const void* x_dev, int32_t N, int32_t HW, int32_t C, void* y_dev, void* stream) {
  if (N < 1 || HW < 1 || C < 8 || C % 8) return bad(GACER_E_SHAPE, "gap_fwd: need C % 8 == 0");
  if (!x_dev || !y_dev || !aligned16(x_dev) || !aligned16(y_dev))
    return bad(GACER_E_INVALID_ARG, "gap_fwd: null or misaligned pointer");
  gap_fwd_kernel<<<grid_for(static_cast<int64_t>(N) * (C / 8)), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x_dev), N, HW, C, static_cast<__nv_bfloat16*>(y_dev));
  return launched("gap_fwd");
}

int32_t gacer_linear_fwd(const void* x_dev, const float* w_dev, const float* b_dev, int32_t N, int32_t K, int32_t O,
                         float* z_dev, void* stream) {
  if (N < 1 || K < 1 || O < 1) return bad(GACER_E_SHAPE, "linear_fwd: need N, K, O >= 1");
  if (!x_dev || !w_dev || !z_dev) return bad(GACER_E_INVALID_ARG, "linear_fwd: null pointer");
  const int64_t n = static_cast<int64_t>(N) * O * 32;   // one warp per output
  linear_fwd_kernel<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0,
                      static_cast<cudaStream_t>(stream)>>>(static_cast<const __nv_bfloat16*>(x_dev), w_dev, b_dev, N,
                                                           K, O, z_dev);
  return launched("linear_fwd");
}

int32_t gacer_linear_bwd(const void* x_dev, const float* w_dev, const float* dy_dev, int32_t N, int32_t K, int32_t O,
                         float* dx_dev, float* dw_dev, float* db_dev, void* stream) {
  if (N < 1 || K < 1 || O < 1) return bad(GACER_E_SHAPE, "linear_bwd: need N, K, O >= 1");
  if (!x_dev || !w_dev || !dy_dev || !dw_dev) return bad(GACER_E_INVALID_ARG, "linear_bwd: null pointer");
  auto s = static_cast<cudaStream_t>(stream);
  if (dx_dev) {
    const int64_t n = static_cast<int64_t>(N) * K;
    linear_dx_kernel<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(w_dev, dy_dev, N, K, O,
                                                                                         dx_dev);
  }
  const int64_t n = static_cast<int64_t>(O) * K;
  linear_dw_kernel<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      static_cast<const __nv_bfloat16*>(x_dev), dy_dev, N, K, O, dw_dev, db_dev);
  return launched("linear_bwd");
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
