// train_dev.cuh -- the training tenant's CUDA-core operators (SURVEY.md §8(a)
// A11) as "virtual grid" device functions, shared by the standalone C-ABI
// calls of include/gacer_train.h (train_ops.cu: one vgrid_kernel launch of
// nvb blocks x VG_THREADS) and by the executor's DK_VGRID work items
// (executor.cu: the worker group runs a range of virtual blocks).  Same code,
// same thread count, same virtual-block decomposition => bit-identical
// results in both paths.
//
// Every function is   f(const VArgs& a, vb, nvb, tid, nthr, smem)
// and behaves like block vb of an nvb-block grid of nthr threads: grid-stride
// loops stride by nvb * nthr; block-level reductions use named barrier 1 over
// nthr threads and the caller's shared-memory scratch (VG_SMEM_BYTES).
// Reductions are deterministic: fixed row ranges per virtual block summed in
// row order (fp32), block partials combined in block order (fp64), no atomics.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "gacer_dev.h"

namespace gacer {

static_assert(VG_THREADS == NWORK, "virtual blocks run on the executor's worker group");
constexpr int VG_SMEM_BYTES = 16384 * 2;      // largest scratch: a transpose tile (>= BN constants 3 x 2048 floats)

// Each operator is its own (non-inlined) function: the executor dispatches
// them from one switch, and inlining would give every operator the register
// allocation of the heaviest one (spills).
#define VG_FN static __device__ __noinline__

__device__ __forceinline__ void vg_bar(int nthr) { asm volatile("bar.sync 1, %0;\n" ::"r"(nthr) : "memory"); }

__device__ __forceinline__ void vg_unpack8(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint32_t vg_pack2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint4 vg_pack8(const float* f) {
  return make_uint4(vg_pack2(f[0], f[1]), vg_pack2(f[2], f[3]), vg_pack2(f[4], f[5]), vg_pack2(f[6], f[7]));
}

#define VG_LOOP(i, total) \
  for (int64_t i = static_cast<int64_t>(vb) * nthr + tid; i < (total); i += static_cast<int64_t>(nvb) * nthr)

// ------------------------------------------------------------------ BN
// BN partial sums over row block vb (of P = nvb blocks).  mode 0 (forward
// statistics): (sum (x - K), sum (x - K)^2) with the per-channel shift K =
// x[0][c] (shifted sums: no cancellation when |mean| >> std); mode 1
// (backward): (sum dy', sum dy' * xhat), dy' = dy masked by the fused ReLU's
// output ym when given, xhat = (x - mean) * rsqrt(var + eps).
// Thread t owns 8-channel group gl = t % G and row phase t / G.
// a: p0 x, p1 dy, p2 ym, p3 mean, p4 var, p5 part [P][2][C] (out); n0 M;
//    i0 mode, i1 C; f0 eps
// BN partial sums over rows r, r + RP, ... < r1 of 8 channels (g): U rows'
// loads in flight, summed in row order.  MODE 0: shifted sums of x - K;
// MODE 1: sum dy' and sum dy' * xhat (dy' = dy masked by the ReLU output ym).
template <int U, int MODE>
__device__ __forceinline__ void bnp_rows(const __nv_bfloat16* x, const __nv_bfloat16* dy, const __nv_bfloat16* ym,
                                         int C, int g, int64_t rbeg, int64_t r1, int RP, const float (&mu)[8],
                                         const float (&is)[8], float (&s1)[8], float (&s2)[8]) {
  for (int64_t r = rbeg; r < r1; r += static_cast<int64_t>(U) * RP) {
    uint4 va[U], vd[MODE ? U : 1], vm[MODE ? U : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t rr = r + u * RP;
      va[u] = rr < r1 ? __ldcs(reinterpret_cast<const uint4*>(x + rr * C + g * 8)) : make_uint4(0, 0, 0, 0);
      if (MODE == 1) {
        vd[u] = rr < r1 ? __ldcs(reinterpret_cast<const uint4*>(dy + rr * C + g * 8)) : make_uint4(0, 0, 0, 0);
        vm[u] = (ym && rr < r1) ? __ldcs(reinterpret_cast<const uint4*>(ym + rr * C + g * 8)) : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (r + u * RP >= r1) break;
      float v[8];
      vg_unpack8(va[u], v);
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = v[j] - mu[j];
          s1[j] += d;
          s2[j] = fmaf(d, d, s2[j]);
        }
      } else {
        float d[8];
        vg_unpack8(vd[MODE ? u : 0], d);
        if (ym) {                        // fused ReLU backward: the mask of the BN's ReLU output
          float mk[8];
          vg_unpack8(vm[MODE ? u : 0], mk);
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] = mk[j] > 0.0f ? d[j] : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s1[j] += d[j];
          s2[j] = fmaf(d[j], (v[j] - mu[j]) * is[j], s2[j]);
        }
      }
    }
  }
}

VG_FN void vg_bn_partial(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t* smem) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.p[0]);
  const __nv_bfloat16* dy = static_cast<const __nv_bfloat16*>(a.p[1]);
  const __nv_bfloat16* ym = static_cast<const __nv_bfloat16*>(a.p[2]);
  const float* mean = static_cast<const float*>(a.p[3]);
  const float* var = static_cast<const float*>(a.p[4]);
  float* part = static_cast<float*>(const_cast<void*>(a.p[5]));
  const int64_t M = a.n[0];
  const int mode = a.i[0], C = a.i[1];
  const float eps = a.f[0];
  float* red = reinterpret_cast<float*>(smem);           // [2][nthr * 8]
  const int G8 = C / 8;
  const int G = G8 < nthr ? G8 : nthr;
  const int RP = nthr / G;
  const int gl = tid % G, ph = tid / G;
  const int64_t rows = (M + nvb - 1) / nvb;
  const int64_t r0 = vb * rows;
  const int64_t r1 = r0 + rows < M ? r0 + rows : M;
  for (int gbase = 0; gbase < G8; gbase += G) {
    const int g = gbase + gl;
    float s1[8] = {0, 0, 0, 0, 0, 0, 0, 0}, s2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float mu[8], is[8];
    const bool active = ph < RP && g < G8;
    if (active) {
      if (mode == 1) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          mu[j] = mean[g * 8 + j];
          is[j] = rsqrtf(var[g * 8 + j] + eps);
        }
      } else {
        vg_unpack8(*reinterpret_cast<const uint4*>(x + g * 8), mu);   // the shift K (row 0)
      }
    }
    if (active) {
      // rows in flight per thread: 16 for the forward statistics (one tensor),
      // 8 for the backward sums (three tensors); each thread still sums its
      // rows r0 + ph, + RP, ... in row order (results independent of it)
      if (mode == 0) bnp_rows<16, 0>(x, dy, ym, C, g, r0 + ph, r1, RP, mu, is, s1, s2);
      else bnp_rows<8, 1>(x, dy, ym, C, g, r0 + ph, r1, RP, mu, is, s1, s2);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      red[tid * 8 + j] = s1[j];
      red[nthr * 8 + tid * 8 + j] = s2[j];
    }
    vg_bar(nthr);
    if (ph == 0 && g < G8) {          // combine the row phases in phase order
      for (int q = 1; q < RP; ++q)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s1[j] += red[(q * G + gl) * 8 + j];
          s2[j] += red[nthr * 8 + (q * G + gl) * 8 + j];
        }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        part[(static_cast<size_t>(vb) * 2 + 0) * C + g * 8 + j] = s1[j];
        part[(static_cast<size_t>(vb) * 2 + 1) * C + g * 8 + j] = s2[j];
      }
    }
    vg_bar(nthr);
  }
}

// Combine the P partials of 32 channels (block vb) in block order (fp64),
// then fold the apply pass's per-channel constants into coef (fp32 [k][C]):
//   mode 0 -> o1 = mean, o2 = biased var; coef = (scale, shift)
//   mode 1 -> o1 = dgamma = sum dy*xhat, o2 = dbeta = sum dy; coef = (a, b, c)
//             with dx = a * dy + b * x + c (BN backward expanded in x)
// Warp w sums partials p = w, w + W, ... (W = nthr / 32 warps) in order, then
// warp 0 adds the W warp sums in warp order.
// a: p0 part, p1 gamma, p2 beta, p3 x (mode 0: the shift rows) / mean_in
//    (mode 1), p4 var_in (mode 1), p5 o1, p6 o2, p7 coef; n0 M; i0 mode,
//    i1 C, i2 P; f0 eps
VG_FN void vg_bn_finalize(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t* smem) {
  (void)nvb;
  const float* part = static_cast<const float*>(a.p[0]);
  const float* gamma = static_cast<const float*>(a.p[1]);
  const float* beta = static_cast<const float*>(a.p[2]);
  const int64_t M = a.n[0];
  const int mode = a.i[0], C = a.i[1], P = a.i[2];
  const float eps = a.f[0];
  float* o1 = static_cast<float*>(const_cast<void*>(a.p[5]));
  float* o2 = static_cast<float*>(const_cast<void*>(a.p[6]));
  float* coef = static_cast<float*>(const_cast<void*>(a.p[7]));
  const int W = nthr >> 5;
  double* red = reinterpret_cast<double*>(smem);        // [2][W][32]
  const int lane = tid & 31, wp = tid >> 5;
  const int c = vb * 32 + lane;
  double s = 0.0, q = 0.0;
  if (c < C && wp < W) {
    int p = wp;
    for (; p + 3 * W < P; p += 4 * W) {     // four partials' loads in flight, summed in order
      float x0[4], x1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = part[(static_cast<size_t>(p + W * u) * 2 + 0) * C + c];
        x1[u] = part[(static_cast<size_t>(p + W * u) * 2 + 1) * C + c];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s += x0[u];
        q += x1[u];
      }
    }
    for (; p < P; p += W) {
      s += part[(static_cast<size_t>(p) * 2 + 0) * C + c];
      q += part[(static_cast<size_t>(p) * 2 + 1) * C + c];
    }
  }
  if (wp < W) {
    red[wp * 32 + lane] = s;
    red[(W + wp) * 32 + lane] = q;
  }
  vg_bar(nthr);
  if (wp == 0 && c < C) {
    s = red[lane];
    q = red[W * 32 + lane];
    for (int w = 1; w < W; ++w) {
      s += red[w * 32 + lane];
      q += red[(W + w) * 32 + lane];
    }
    const double Md = static_cast<double>(M);
    if (mode == 0) {
      const double K = __bfloat162float(static_cast<const __nv_bfloat16*>(a.p[3])[c]);   // the shift
      const double d = s / Md;
      double v = q / Md - d * d;
      v = v > 0.0 ? v : 0.0;
      const double mu = K + d;
      o1[c] = static_cast<float>(mu);
      o2[c] = static_cast<float>(v);
      const double sc = gamma[c] / sqrt(static_cast<double>(static_cast<float>(v)) + eps);
      coef[c] = static_cast<float>(sc);
      coef[C + c] = static_cast<float>(beta[c] - static_cast<double>(static_cast<float>(mu)) * sc);
    } else {
      const float* mean_in = static_cast<const float*>(a.p[3]);
      const float* var_in = static_cast<const float*>(a.p[4]);
      o1[c] = static_cast<float>(q);   // dgamma
      o2[c] = static_cast<float>(s);   // dbeta
      const double is = 1.0 / sqrt(static_cast<double>(var_in[c]) + eps);
      const double gi = gamma[c] * is;
      const double k = gi * is * static_cast<double>(static_cast<float>(q)) / Md;
      coef[c] = static_cast<float>(gi);
      coef[C + c] = static_cast<float>(-k);
      coef[2 * C + c] = static_cast<float>(-gi * static_cast<double>(static_cast<float>(s)) / Md + k * mean_in[c]);
    }
  }
  vg_bar(nthr);   // the scratch is reused by the next virtual block
}

// y = act(x * scale + shift) (mode 0); dx = a * dy + b * x + c (mode 1).
// The host sizes the grid so the stride nvb * nthr is a multiple of C / 8
// (vg_apply_blocks): every thread keeps one 8-channel group and its
// constants in registers; VG_UNROLL 16-byte groups' loads are in flight.
// a: p0 x, p1 dy, p2 ym, p3 coef, p4 out; n0 M; i0 mode, i1 C, i2 relu
constexpr int VG_UNROLL = 8;   // 16-byte groups per thread with loads in flight
template <int MODE>
VG_FN void vg_bn_apply_t(const VArgs& a, int vb, int nvb, int tid, int nthr) {
  constexpr int U = MODE == 0 ? VG_UNROLL : VG_UNROLL / 2;   // (mode 1 streams three tensors)
  const uint4* x = static_cast<const uint4*>(a.p[0]);
  const uint4* dy = static_cast<const uint4*>(a.p[1]);
  const uint4* ym = static_cast<const uint4*>(a.p[2]);
  const float* coef = static_cast<const float*>(a.p[3]);
  uint4* out = static_cast<uint4*>(const_cast<void*>(a.p[4]));
  const int64_t M = a.n[0];
  constexpr int mode = MODE;
  const int C = a.i[1], relu = a.i[2];
  const int G8 = C / 8;
  const int64_t total = M * G8, stride = static_cast<int64_t>(nvb) * nthr;
  const int64_t first = static_cast<int64_t>(vb) * nthr + tid;
  const bool fixed = (stride % G8) == 0;
  float k0[8], k1[8], k2[8];
  int c0 = -1;
  for (int64_t i0 = first; i0 < total; i0 += U * stride) {
    uint4 vx[U], vd[U], vm[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) {
        vx[u] = __ldcs(x + i);
        if (mode == 1) {
          vd[u] = __ldcs(dy + i);
          if (ym) vm[u] = __ldcs(ym + i);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) {
        const int c = (fixed && c0 >= 0) ? c0 : static_cast<int>(i % G8) * 8;
        if (c != c0) {
          c0 = c;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            k0[j] = coef[c + j];
            k1[j] = coef[C + c + j];
            k2[j] = mode == 1 ? coef[2 * C + c + j] : 0.0f;
          }
        }
        float v[8];
        vg_unpack8(vx[u], v);
        if (mode == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float t = fmaf(v[j], k0[j], k1[j]);
            v[j] = relu ? fmaxf(t, 0.0f) : t;
          }
        } else {
          float d[8];
          vg_unpack8(vd[u], d);
          if (ym) {
            float mk[8];
            vg_unpack8(vm[u], mk);
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j] = mk[j] > 0.0f ? d[j] : 0.0f;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = fmaf(k0[j], d[j], fmaf(k1[j], v[j], k2[j]));
        }
        __stcs(out + i, vg_pack8(v));
      }
    }
  }
}

VG_FN void vg_bn_apply(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  if (a.i[0] == 0) vg_bn_apply_t<0>(a, vb, nvb, tid, nthr);
  else vg_bn_apply_t<1>(a, vb, nvb, tid, nthr);
}

// ------------------------------------------------------------------ elementwise
// dx = dy where x > 0 (and x < 6 for ReLU6), else 0.  a: p0 x, p1 dy, p2 dx; n0 n8; i0 six
VG_FN void vg_relu_bwd(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const uint4* x = static_cast<const uint4*>(a.p[0]);
  const uint4* dy = static_cast<const uint4*>(a.p[1]);
  uint4* dx = static_cast<uint4*>(const_cast<void*>(a.p[2]));
  const int six = a.i[0];
  const int64_t total = a.n[0], stride = static_cast<int64_t>(nvb) * nthr;
  for (int64_t i0 = static_cast<int64_t>(vb) * nthr + tid; i0 < total; i0 += VG_UNROLL * stride) {
    uint4 vx[VG_UNROLL], vd[VG_UNROLL];
#pragma unroll
    for (int u = 0; u < VG_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) { vx[u] = x[i]; vd[u] = dy[i]; }
    }
#pragma unroll
    for (int u = 0; u < VG_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) {
        float v[8], d[8];
        vg_unpack8(vx[u], v);
        vg_unpack8(vd[u], d);
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = (v[j] > 0.0f && (!six || v[j] < 6.0f)) ? d[j] : 0.0f;
        dx[i] = vg_pack8(d);
      }
    }
  }
}

// y = a + b (ReLU when relu != 0).  a: p0 a, p1 b, p2 y; n0 n8; i0 relu
VG_FN void vg_add(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const uint4* pa = static_cast<const uint4*>(a.p[0]);
  const uint4* pb = static_cast<const uint4*>(a.p[1]);
  uint4* y = static_cast<uint4*>(const_cast<void*>(a.p[2]));
  const int relu = a.i[0];
  const int64_t total = a.n[0], stride = static_cast<int64_t>(nvb) * nthr;
  for (int64_t i0 = static_cast<int64_t>(vb) * nthr + tid; i0 < total; i0 += VG_UNROLL * stride) {
    uint4 va[VG_UNROLL], vb2[VG_UNROLL];
#pragma unroll
    for (int u = 0; u < VG_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) { va[u] = pa[i]; vb2[u] = pb[i]; }
    }
#pragma unroll
    for (int u = 0; u < VG_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) {
        float p[8], q[8];
        vg_unpack8(va[u], p);
        vg_unpack8(vb2[u], q);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float t = p[j] + q[j];
          p[j] = relu ? fmaxf(t, 0.0f) : t;
        }
        y[i] = vg_pack8(p);
      }
    }
  }
}

// ------------------------------------------------------------------ pooling
// ints: i0 N, i1 H, i2 W, i3 C, i4 KH, i5 KW, i6 S, i7 ph, i8 pw, i9 Ho, i10 Wo
// Max-pool forward.  a: p0 x, p1 y
VG_FN void vg_maxpool_fwd(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.p[0]);
  uint4* y = static_cast<uint4*>(const_cast<void*>(a.p[1]));
  const int N = a.i[0], H = a.i[1], W = a.i[2], C = a.i[3], KH = a.i[4], KW = a.i[5], S = a.i[6], ph = a.i[7],
            pw = a.i[8], Ho = a.i[9], Wo = a.i[10];
  const int G8 = C / 8;
  VG_LOOP(i, static_cast<int64_t>(N) * Ho * Wo * G8) {
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
        vg_unpack8(*reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hh) * W + ww) * C + g * 8), v);
#pragma unroll
        for (int j = 0; j < 8; ++j) best[j] = fmaxf(best[j], v[j]);
      }
    }
    y[i] = vg_pack8(best);
  }
}

// Max-pool backward, pass 1: per (output window, 8-channel group) the first
// maximum per channel (row-major tap order, padded taps skipped, Q14) as a
// tap index byte.  a: p0 x, p1 arg (uint8 [N*Ho*Wo*C])
VG_FN void vg_maxpool_argmax(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.p[0]);
  uint2* arg = static_cast<uint2*>(const_cast<void*>(a.p[1]));
  // p2 (optional): also the pooled output, exactly as vg_maxpool_fwd computes
  // it (the fmaxf chain) -- the executor's training step runs the forward
  // pool and the backward's argmax as this one operator
  uint4* yo = static_cast<uint4*>(const_cast<void*>(a.p[2]));
  const int N = a.i[0], H = a.i[1], W = a.i[2], C = a.i[3], KH = a.i[4], KW = a.i[5], S = a.i[6], ph = a.i[7],
            pw = a.i[8], Ho = a.i[9], Wo = a.i[10];
  const int G8 = C / 8;
  VG_LOOP(i, static_cast<int64_t>(N) * Ho * Wo * G8) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int wo = static_cast<int>(pix % Wo), ho = static_cast<int>((pix / Wo) % Ho);
    const int n = static_cast<int>(pix / (static_cast<int64_t>(Wo) * Ho));
    float best[8];
    uint32_t tap[8];
#pragma unroll
    float mx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { best[j] = -INFINITY; tap[j] = 255u; mx[j] = -INFINITY; }
    for (int r = 0; r < KH; ++r) {
      const int hh = ho * S - ph + r;
      if (hh < 0 || hh >= H) continue;
      for (int q = 0; q < KW; ++q) {
        const int ww = wo * S - pw + q;
        if (ww < 0 || ww >= W) continue;
        float v[8];
        vg_unpack8(*reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + hh) * W + ww) * C + g * 8), v);
        const uint32_t id = static_cast<uint32_t>(r * KW + q);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (tap[j] == 255u || v[j] > best[j]) { best[j] = v[j]; tap[j] = id; }
          mx[j] = fmaxf(mx[j], v[j]);
        }
      }
    }
    uint2 o;
    o.x = tap[0] | (tap[1] << 8) | (tap[2] << 16) | (tap[3] << 24);
    o.y = tap[4] | (tap[5] << 8) | (tap[6] << 16) | (tap[7] << 24);
    arg[i] = o;
    if (yo) yo[i] = vg_pack8(mx);
  }
}

// Max-pool backward, pass 2: per (input pixel, 8-channel group) the sum of dy
// over the windows whose recorded tap is this pixel, in (ho, wo) order.
// a: p0 arg, p1 dy, p2 dx
VG_FN void vg_maxpool_bwd(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const uint2* arg = static_cast<const uint2*>(a.p[0]);
  const uint4* dy = static_cast<const uint4*>(a.p[1]);
  uint4* dx = static_cast<uint4*>(const_cast<void*>(a.p[2]));
  const int N = a.i[0], H = a.i[1], W = a.i[2], C = a.i[3], KH = a.i[4], KW = a.i[5], S = a.i[6], ph = a.i[7],
            pw = a.i[8], Ho = a.i[9], Wo = a.i[10];
  const int G8 = C / 8;
  VG_LOOP(i, static_cast<int64_t>(N) * H * W * G8) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int wi = static_cast<int>(pix % W), hi = static_cast<int>((pix / W) % H);
    const int n = static_cast<int>(pix / (static_cast<int64_t>(W) * H));
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int ho0 = hi + ph - KH + 1;
    ho0 = ho0 <= 0 ? 0 : (ho0 + S - 1) / S;
    int ho1 = (hi + ph) / S;
    ho1 = ho1 < Ho - 1 ? ho1 : Ho - 1;
    int wo0 = wi + pw - KW + 1;
    wo0 = wo0 <= 0 ? 0 : (wo0 + S - 1) / S;
    int wo1 = (wi + pw) / S;
    wo1 = wo1 < Wo - 1 ? wo1 : Wo - 1;
    auto add_window = [&](int ho, int wo, uint2 t, uint4 dv) {
      const uint32_t me = static_cast<uint32_t>((hi - (ho * S - ph)) * KW + (wi - (wo * S - pw)));
      const uint32_t tt[8] = {t.x & 255u, (t.x >> 8) & 255u, (t.x >> 16) & 255u, t.x >> 24,
                              t.y & 255u, (t.y >> 8) & 255u, (t.y >> 16) & 255u, t.y >> 24};
      float d[8];
      vg_unpack8(dv, d);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (tt[j] == me) acc[j] += d[j];
    };
    if (ho1 - ho0 <= 1 && wo1 - wo0 <= 1) {
      // at most 2 x 2 windows (3x3 / stride 2): every window's argmax and dy
      // loaded up front (one round trip instead of two per window); summed
      // in the same (ho, wo) order.  (Two groups per pass, or the 3x3
      // forward / argmax taps loaded together, spilled and ran slower.)
      uint2 t[4];
      uint4 dv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ho = ho0 + (q >> 1), wo = wo0 + (q & 1);
        if (ho <= ho1 && wo <= wo1) {
          const int64_t o = ((static_cast<int64_t>(n) * Ho + ho) * Wo + wo) * G8 + g;
          t[q] = arg[o];
          dv[q] = dy[o];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ho = ho0 + (q >> 1), wo = wo0 + (q & 1);
        if (ho <= ho1 && wo <= wo1) add_window(ho, wo, t[q], dv[q]);
      }
    } else {
      for (int ho = ho0; ho <= ho1; ++ho)
        for (int wo = wo0; wo <= wo1; ++wo) {
          const int64_t o = ((static_cast<int64_t>(n) * Ho + ho) * Wo + wo) * G8 + g;
          add_window(ho, wo, arg[o], dy[o]);
        }
    }
    dx[i] = vg_pack8(acc);
  }
}

// GAP backward: dx[n][p][c] = dy[n][c] / HW.  a: p0 dy (f32 [N][C]), p1 dx; i0 N, i1 HW, i2 C
VG_FN void vg_gap_bwd(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const float* dy = static_cast<const float*>(a.p[0]);
  uint4* dx = static_cast<uint4*>(const_cast<void*>(a.p[1]));
  const int N = a.i[0], HW = a.i[1], C = a.i[2];
  const int G8 = C / 8;
  const float inv = 1.0f / static_cast<float>(HW);
  VG_LOOP(i, static_cast<int64_t>(N) * HW * G8) {
    const int g = static_cast<int>(i % G8);
    const int n = static_cast<int>(i / (static_cast<int64_t>(HW) * G8));
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = dy[static_cast<int64_t>(n) * C + g * 8 + j] * inv;
    dx[i] = vg_pack8(v);
  }
}

// GAP forward: y[n][c] = (1/HW) sum_p x[n][p][c] in pixel order (fp32), bf16.
// a: p0 x, p1 y; i0 N, i1 HW, i2 C
VG_FN void vg_gap_fwd(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.p[0]);
  uint4* y = static_cast<uint4*>(const_cast<void*>(a.p[1]));
  const int N = a.i[0], HW = a.i[1], C = a.i[2];
  const int G8 = C / 8;
  VG_LOOP(i, static_cast<int64_t>(N) * G8) {
    const int g = static_cast<int>(i % G8), n = static_cast<int>(i / G8);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < HW; ++p) {
      float v[8];
      vg_unpack8(*reinterpret_cast<const uint4*>(x + (static_cast<int64_t>(n) * HW + p) * C + g * 8), v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += v[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] /= static_cast<float>(HW);
    y[i] = vg_pack8(acc);
  }
}

// ------------------------------------------------------------------ FC
// z[n][o] = b[o] + sum_k w[o][k] x[n][k]: one warp per output, lane l sums
// k = l, l+32, ..., then a fixed xor butterfly.  a: p0 x (bf16), p1 w (f32),
// p2 b (nullable), p3 z (f32); i0 N, i1 K, i2 O
VG_FN void vg_linear_fwd(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.p[0]);
  const float* w = static_cast<const float*>(a.p[1]);
  const float* b = static_cast<const float*>(a.p[2]);
  float* z = static_cast<float*>(const_cast<void*>(a.p[3]));
  const int N = a.i[0], K = a.i[1], O = a.i[2];
  const int lane = tid & 31;
  // a warp computes 4 outputs (n, o .. o + 3) of one row (N * ceil(O/4)
  // warp units): 4 independent FMA chains sharing the x loads; each output
  // keeps its summation order (lane partials over k = lane, lane + 32, ...,
  // then the xor tree)
  const int O4 = (O + 3) / 4;
  const int64_t nw = static_cast<int64_t>(nvb) * (nthr >> 5);
  for (int64_t wid = static_cast<int64_t>(vb) * (nthr >> 5) + (tid >> 5); wid < static_cast<int64_t>(N) * O4;
       wid += nw) {
    const int n = static_cast<int>(wid / O4), o0 = static_cast<int>(wid % O4) * 4;
    const __nv_bfloat16* xr = x + static_cast<int64_t>(n) * K;
    const float* wr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) wr[u] = w + static_cast<int64_t>(o0 + u < O ? o0 + u : o0) * K;
    float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int k = lane; k < K; k += 32) {
      const float xv = __bfloat162float(xr[k]);
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] = fmaf(xv, wr[u][k], s[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s[u] += __shfl_xor_sync(0xffffffffu, s[u], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (o0 + u < O) z[static_cast<int64_t>(n) * O + o0 + u] = s[u] + (b ? b[o0 + u] : 0.0f);
    }
  }
}
// a: p0 w [O][K] fp32, p1 dy [N][O] fp32, p2 dx [N][K] fp32; i0 N, i1 K, i2 O.
// Unit: 4 rows n0..n0+3 of one column k (the grid covers ceil(N/4) * K
// units): each weight load serves 4 independent FMA chains; every output
// still sums over o in order.
VG_FN void vg_linear_dx(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const float* w = static_cast<const float*>(a.p[0]);
  const float* dy = static_cast<const float*>(a.p[1]);
  float* dx = static_cast<float*>(const_cast<void*>(a.p[2]));
  const int N = a.i[0], K = a.i[1], O = a.i[2];
  const int N4 = (N + 3) / 4;
  VG_LOOP(i, static_cast<int64_t>(N4) * K) {
    const int n0 = static_cast<int>(i / K) * 4, k = static_cast<int>(i % K);
    const float* dyr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) dyr[u] = dy + static_cast<int64_t>(n0 + u < N ? n0 + u : n0) * O;
    float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 4
    for (int o = 0; o < O; ++o) {
      const float wv = w[static_cast<int64_t>(o) * K + k];
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] = fmaf(dyr[u][o], wv, s[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (n0 + u < N) dx[static_cast<int64_t>(n0 + u) * K + k] = s[u];
  }
}

// dw[o][k] = sum_n dy[n][o] x[n][k], db[o] = sum_n dy[n][o] (n order).
// a: p0 x (bf16), p1 dy, p2 dw, p3 db (nullable); i0 N, i1 K, i2 O
// a: p0 x [N][K] bf16, p1 dy [N][O] fp32, p2 dw [O][K], p3 db [O] (or null); i0 N, i1 K, i2 O.
// Unit: 4 outputs o0..o0+3 of one column k (ceil(O/4) * K units): each x
// load serves 4 chains; every output sums over n in order.
VG_FN void vg_linear_dw(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.p[0]);
  const float* dy = static_cast<const float*>(a.p[1]);
  float* dw = static_cast<float*>(const_cast<void*>(a.p[2]));
  float* db = static_cast<float*>(const_cast<void*>(a.p[3]));
  const int N = a.i[0], K = a.i[1], O = a.i[2];
  const int O4 = (O + 3) / 4;
  VG_LOOP(i, static_cast<int64_t>(O4) * K) {
    const int o0 = static_cast<int>(i / K) * 4, k = static_cast<int>(i % K);
    float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 4
    for (int n = 0; n < N; ++n) {
      const float xv = __bfloat162float(x[static_cast<int64_t>(n) * K + k]);
      const float* dyr = dy + static_cast<int64_t>(n) * O + o0;
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] = fmaf(o0 + u < O ? dyr[u] : 0.0f, xv, s[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (o0 + u < O) dw[static_cast<int64_t>(o0 + u) * K + k] = s[u];
    if (db && k == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (o0 + u >= O) break;
        float t = 0.0f;
        for (int n = 0; n < N; ++n) t += dy[static_cast<int64_t>(n) * O + o0 + u];
        db[o0 + u] = t;
      }
    }
  }
}

// Softmax cross-entropy of row vb: fixed-order reductions (max, then sum of
// exp): thread partials over j = tid, tid + nthr, ..., then thread 0 combines
// them in thread order.  dz = (softmax - onehot) / N (may alias z); rowloss[n].
// a: p0 z, p1 labels (int32), p2 dz, p3 rowloss; i0 N, i1 Cls
VG_FN void vg_softmax_ce(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t* smem) {
  (void)nvb;
  const float* z = static_cast<const float*>(a.p[0]);
  const int32_t* labels = static_cast<const int32_t*>(a.p[1]);
  float* dz = static_cast<float*>(const_cast<void*>(a.p[2]));
  float* rowloss = static_cast<float*>(const_cast<void*>(a.p[3]));
  const int N = a.i[0], Cls = a.i[1];
  float* red = reinterpret_cast<float*>(smem);   // [nthr + 2]
  const int n = vb;
  const float* zr = z + static_cast<int64_t>(n) * Cls;
  float m = -INFINITY;
  for (int j = tid; j < Cls; j += nthr) m = fmaxf(m, zr[j]);
  red[tid] = m;
  vg_bar(nthr);
  if (tid == 0) {
    float t = red[0];
    for (int q = 1; q < nthr; ++q) t = fmaxf(t, red[q]);
    red[nthr] = t;
  }
  vg_bar(nthr);
  m = red[nthr];
  float s = 0.0f;
  for (int j = tid; j < Cls; j += nthr) s += expf(zr[j] - m);
  vg_bar(nthr);
  red[tid] = s;
  vg_bar(nthr);
  if (tid == 0) {
    float t = red[0];
    for (int q = 1; q < nthr; ++q) t += red[q];
    red[nthr + 1] = t;
  }
  vg_bar(nthr);
  const float sum = red[nthr + 1];
  const int lab = labels[n];
  const bool ok = lab >= 0 && lab < Cls;
  const float zl = ok ? zr[lab] : 0.0f;   // read before dz (which may alias z) is written
  vg_bar(nthr);
  const float invN = 1.0f / static_cast<float>(N);
  for (int j = tid; j < Cls; j += nthr)
    dz[static_cast<int64_t>(n) * Cls + j] = (expf(zr[j] - m) / sum - (j == lab ? 1.0f : 0.0f)) * invN;
  if (tid == 0) rowloss[n] = ok ? (logf(sum) + m) - zl : NAN;
  vg_bar(nthr);   // the scratch is reused by the next virtual block
}

// out = mean of v[0..N) in index order (fp64).  a: p0 v, p1 out; i0 N
VG_FN void vg_mean(const VArgs& a, int vb, int, int tid, int, uint8_t*) {
  if (vb != 0 || tid != 0) return;
  const float* v = static_cast<const float*>(a.p[0]);
  const int N = a.i[0];
  double s = 0.0;
  for (int i = 0; i < N; ++i) s += v[i];
  *static_cast<float*>(const_cast<void*>(a.p[1])) = static_cast<float>(s / N);
}

// SGD with momentum (PyTorch semantics): buf = mom * buf + g (buf = g on the
// first step: a zero-initialised buf gives exactly that), w -= lr * buf.
// a: p0 w, p1 g, p2 buf; n0 n; i0 first; f0 lr, f1 momentum
VG_FN void vg_sgd(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  float* w = static_cast<float*>(const_cast<void*>(a.p[0]));
  const float* g = static_cast<const float*>(a.p[1]);
  float* buf = static_cast<float*>(const_cast<void*>(a.p[2]));
  const int first = a.i[0];
  const float lr = a.f[0], mom = a.f[1];
  VG_LOOP(i, a.n[0]) {
    const float b = first ? g[i] : fmaf(mom, buf[i], g[i]);
    buf[i] = b;
    w[i] = fmaf(-lr, b, w[i]);
  }
}

// ------------------------------------------------------------------ GEMM operand staging
// Conv filter packing from the fp32 master weights w [Cout][Cin][KH][KW] into
// a K-major bf16 GEMM B operand [rows][Kpad]: forward = 1: row co, column
// (r*KW + s)*cread + ci = w[co][ci][r][s]; forward = 0 (data gradient): row
// ci, column (r*KW + s)*cread + co = w[co][ci][KH-1-r][KW-1-s]; padding 0.
// a: p0 w, p1 out; i0 Cout, i1 Cin, i2 KH, i3 KW, i4 cread, i5 Kpad, i6 rows, i7 forward, i8 block bn,
//    i9 phase stride S (dgrad sub-filter; 0: none), i10/i11 phase (a, b), i12/i13 the full KH, KW
// One packed element i of a filter job (the body of vg_filter / vg_filter_all).
__device__ __forceinline__ void filter_elem(const float* w, __nv_bfloat16* out, const int32_t* ai, int64_t i) {
  const int Cout = ai[0], Cin = ai[1], KH = ai[2], KW = ai[3], cread = ai[4], Kpad = ai[5], forward = ai[7],
            bbn = ai[8];
  const int phS = ai[9], pa = ai[10], pb = ai[11], KHf = ai[12], KWf = ai[13];   // dgrad phase (phS > 0)
  {
    const int row = static_cast<int>(i / Kpad), k = static_cast<int>(i % Kpad);
    // bbn > 0: the A_IM2COL8 block layout -- per (N-tile, K-block) a bn x 64
    // block in the no-swizzle core-matrix layout (same bijection as the
    // inference packing in host.cpp)
    const int64_t dst = bbn > 0 ? (static_cast<int64_t>(row / bbn) * (Kpad / 64) + k / 64) * bbn * 64 +
                                      ((row % bbn) % 8) * 8 + ((row % bbn) / 8) * 64 + (k % 64) % 8 +
                                      ((k % 64) / 8) * bbn * 8
                                : i;
    const int tap = k / cread, col = k % cread;
    float v = 0.0f;
    if (forward) {
      if (row < Cout && tap < KH * KW && col < Cin)
        v = w[((static_cast<int64_t>(row) * Cin + col) * KH + tap / KW) * KW + tap % KW];
    } else if (row < Cin && tap < KH * KW && col < Cout) {
      const int r = tap / KW, s = tap % KW;
      if (phS > 0)   // the phase (pa, pb) sub-filter of a strided conv, flipped: tap (r, s) = full tap
                     // (pa + S (KH - 1 - r), pb + S (KW - 1 - s)) of the KHf x KWf filter
        v = w[((static_cast<int64_t>(col) * Cin + row) * KHf + (pa + phS * (KH - 1 - r))) * KWf +
              (pb + phS * (KW - 1 - s))];
      else
        v = w[((static_cast<int64_t>(col) * Cin + row) * KH + (KH - 1 - r)) * KW + (KW - 1 - s)];
    }
    out[dst] = __float2bfloat16_rn(v);
  }
}

VG_FN void vg_filter(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const float* w = static_cast<const float*>(a.p[0]);
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(const_cast<void*>(a.p[1]));
  VG_LOOP(i, static_cast<int64_t>(a.i[6]) * a.i[5]) filter_elem(w, out, a.i, i);
}

// Every filter job of the step in one operator (one grid over the jobs'
// concatenated outputs; the job of an element by binary search on `start`):
// the same packed values as one vg_filter per conv, without ~100 per-conv
// operators.  a: p0 FilterJob[n], i0 n, n0 total elements
VG_FN void vg_filter_all(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const FilterJob* jobs = static_cast<const FilterJob*>(a.p[0]);
  const int n = a.i[0];
  const int64_t total = a.n[0];
  // 8-element groups: every job is rows x Kpad elements (Kpad a multiple of
  // 64) and cread is a multiple of 8, so a group shares its row and tap and
  // covers 8 consecutive channels -- one set of index divisions and one
  // 16-byte store per group instead of per element (the per-element form ran
  // ~1.2 ms at the head of every ResNet-50 step, ahead of the first GEMM).
  // Same values, same RNE conversions as filter_elem.
  const int64_t tg = total >> 3;
  const int64_t per = (tg + nvb - 1) / nvb;
  const int64_t g0 = vb * per + tid, g1 = (vb + 1) * per < tg ? (vb + 1) * per : tg;
  if (g0 >= g1) return;
  // a thread finds its first job by binary search, then walks the jobs forward
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].start <= g0 * 8) lo = mid; else hi = mid - 1;
  }
  int j = lo;
  int64_t jstart = 0, jnext = 0;
  const float* w = nullptr;
  __nv_bfloat16* out = nullptr;
  int Cout = 0, Cin = 0, KH = 1, KW = 1, cread = 8, Kpad = 64, forward = 1, bbn = 0, phS = 0, pa = 0, pb = 0,
      KHf = 1, KWf = 1;
  auto load_job = [&](int q) {
    const FilterJob& J = jobs[q];
    jstart = J.start;
    jnext = q + 1 < n ? jobs[q + 1].start : total;
    w = J.w;
    out = static_cast<__nv_bfloat16*>(J.out);
    Cout = J.i[0]; Cin = J.i[1]; KH = J.i[2]; KW = J.i[3]; cread = J.i[4]; Kpad = J.i[5];
    forward = J.i[7]; bbn = J.i[8]; phS = J.i[9]; pa = J.i[10]; pb = J.i[11]; KHf = J.i[12]; KWf = J.i[13];
  };
  load_job(j);
  // one group: its 8 source values (loads issued) and its destination
  auto gather = [&](int64_t g, float (&v)[8], __nv_bfloat16*& o, int64_t& dst) {
    const int64_t e = g * 8;
    while (e >= jnext) load_job(++j);
    const int li = static_cast<int>(e - jstart);
    const int row = li / Kpad, k0 = li - row * Kpad;
    const int tap = k0 / cread, col0 = k0 - tap * cread;
    const int r = tap / KW, s_ = tap - r * KW;
    if (forward) {
      const bool ok = row < Cout && tap < KH * KW;
      const int64_t base = ((static_cast<int64_t>(row) * Cin + col0) * KH + r) * KW + s_;
      const int64_t step = static_cast<int64_t>(KH) * KW;
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (ok && col0 + q < Cin) ? w[base + q * step] : 0.0f;
    } else {
      const bool ok = row < Cin && tap < KH * KW;
      int64_t base, step;
      if (phS > 0) {   // the phase (pa, pb) sub-filter of a strided conv, flipped
        base = ((static_cast<int64_t>(col0) * Cin + row) * KHf + (pa + phS * (KH - 1 - r))) * KWf +
               (pb + phS * (KW - 1 - s_));
        step = static_cast<int64_t>(Cin) * KHf * KWf;
      } else {
        base = ((static_cast<int64_t>(col0) * Cin + row) * KH + (KH - 1 - r)) * KW + (KW - 1 - s_);
        step = static_cast<int64_t>(Cin) * KH * KW;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (ok && col0 + q < Cout) ? w[base + q * step] : 0.0f;
    }
    // bbn > 0: the A_IM2COL8 block layout (filter_elem's bijection; the 8
    // channels of a group are 8 consecutive elements there too)
    dst = bbn > 0 ? (static_cast<int64_t>(row / bbn) * (Kpad / 64) + k0 / 64) * bbn * 64 +
                        ((row % bbn) % 8) * 8 + ((row % bbn) / 8) * 64 + ((k0 % 64) / 8) * bbn * 8
                  : e - jstart;
    o = out;
  };
  auto put = [](const float (&v)[8], __nv_bfloat16* o, int64_t dst) {
    __nv_bfloat162 h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) h[q] = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    *reinterpret_cast<uint4*>(o + dst) = *reinterpret_cast<const uint4*>(h);
  };
  // (two groups per pass -- 16 loads in flight per thread -- measured no
  //  faster: 264 -> 282 us for the ResNet-50 step's packing)
  for (int64_t g = g0; g < g1; g += nthr) {
    float v[8];
    __nv_bfloat16* o;
    int64_t dst;
    gather(g, v, o, dst);
    put(v, o, dst);
  }
}

// Phase-decomposed data gradient of a stride-S conv: dx pixel (h, w) of phase
// (a, b) = ((h + ph) mod S, (w + pw) mod S) is element (u - u0_a, v - v0_b)
// of that phase's stride-1 dgrad conv output P_ab [N][n_a][n_b][C] (DgPhase),
// u = (h + ph - a) / S; a phase no tap reaches is 0.  16-byte groups.
// a: p0..p3 P_ab (index a * S + b; null = no taps); n0 total groups; i0 N, i1 H, i2 W, i3 C, i4 S,
//    i5 ph, i6 pw, i7 KH, i8 KW, p4 dx
VG_FN void vg_phase_scatter(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const int N = a.i[0], H = a.i[1], W = a.i[2], C = a.i[3], S = a.i[4], ph = a.i[5], pw = a.i[6], KH = a.i[7],
            KW = a.i[8];
  uint4* dx = static_cast<uint4*>(const_cast<void*>(a.p[4]));
  const int G8 = C / 8;
  (void)N;
  VG_LOOP(i, a.n[0]) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int w = static_cast<int>(pix % W), h = static_cast<int>((pix / W) % H);
    const int64_t n = pix / (static_cast<int64_t>(W) * H);
    const int pa = (h + ph) % S, pb = (w + pw) % S;
    const uint4* src = static_cast<const uint4*>(a.p[pa * S + pb]);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (src) {
      const DgPhase da = dg_phase(pa, KH, S, ph, H), db = dg_phase(pb, KW, S, pw, W);
      const int u = (h + ph - pa) / S - da.u0, q = (w + pw - pb) / S - db.u0;
      v = src[((n * da.n + u) * db.n + q) * G8 + g];
    }
    dx[i] = v;
  }
}

// Zero-dilated dy of a strided conv's data gradient (Hdd x Wdd).
// a: p0 dy, p1 out; i0 N, i1 Hd, i2 Wd, i3 C, i4 S, i5 Hdd, i6 Wdd
VG_FN void vg_dilate(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const __nv_bfloat16* dy = static_cast<const __nv_bfloat16*>(a.p[0]);
  uint4* out = static_cast<uint4*>(const_cast<void*>(a.p[1]));
  const int N = a.i[0], Hd = a.i[1], Wd = a.i[2], C = a.i[3], S = a.i[4], Hdd = a.i[5], Wdd = a.i[6];
  const int G8 = C / 8;
  VG_LOOP(i, static_cast<int64_t>(N) * Hdd * Wdd * G8) {
    const int g = static_cast<int>(i % G8);
    const int64_t pix = i / G8;
    const int ww = static_cast<int>(pix % Wdd), hh = static_cast<int>((pix / Wdd) % Hdd);
    const int n = static_cast<int>(pix / (static_cast<int64_t>(Wdd) * Hdd));
    uint4 v = make_uint4(0, 0, 0, 0);
    if (hh % S == 0 && ww % S == 0 && hh / S < Hd && ww / S < Wd)
      v = *reinterpret_cast<const uint4*>(dy + ((static_cast<int64_t>(n) * Hd + hh / S) * Wd + ww / S) * C + g * 8);
    out[i] = v;
  }
}

// Weight-gradient operand: the transposed im2col of x, K-major along the
// pixel index m (row (t*C + c), column m), TC channels x TP = 16384 / TC
// pixels of one tap t per virtual block (vg_transpose_tc) through a smem
// tile (coalesced 16-byte loads and stores; 64-pixel segments XOR-swizzled by
// the channel octet so the transposing scalar stores hit distinct banks).
// Block vb = (bx, by, bz) over (cdiv(Kpad, TP), cdiv(C, TC), KH*KW).
// a: p0 x, p1 out; n0 M; i0 N, i1 H, i2 W, i3 C, i4 Ho, i5 Wo, i6 KW, i7 S,
//    i8 ph, i9 pw, i10 Kpad, i11 KH
VG_FN void vg_transpose_im2col(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t* smem) {
  (void)nvb;
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.p[0]);
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(const_cast<void*>(a.p[1]));
  const int64_t M = a.n[0];
  const int H = a.i[1], W = a.i[2], C = a.i[3], Ho = a.i[4], Wo = a.i[5], KW = a.i[6], S = a.i[7],
            ph = a.i[8], pw = a.i[9], Kpad = a.i[10];
  const int TC = vg_transpose_tc(C), TP = VG_TRANSPOSE_TILE / TC, GPR = TC / 8;   // channel groups per pixel
  __nv_bfloat16* tile = reinterpret_cast<__nv_bfloat16*>(smem);
  auto at = [TP](int c, int i) { return c * TP + (i & ~63) + ((((i >> 3) ^ (c >> 3)) & 7) << 3) + (i & 7); };
  const int gx = (Kpad + TP - 1) / TP, gy = (C + TC - 1) / TC;
  const int t = vb / (gx * gy);
  const int by = (vb / gx) % gy, bx = vb % gx;
  const int r = t / KW, q = t % KW;
  const int64_t m0 = static_cast<int64_t>(bx) * TP;
  const int c0 = by * TC;
  const bool vec = (C % 8) == 0;
  for (int e = tid; e < TP * GPR; e += nthr) {
    const int i = e / GPR, cg = (e % GPR) * 8;
    const int64_t m = m0 + i;
    __nv_bfloat16 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __float2bfloat16_rn(0.0f);
    if (m < M && c0 + cg < C) {
      const uint32_t m32 = static_cast<uint32_t>(m);
      const uint32_t pq = m32 / static_cast<uint32_t>(Wo);
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
  vg_bar(nthr);
  for (int e = tid; e < TC * (TP / 8); e += nthr) {
    const int cc = e / (TP / 8), mg = (e % (TP / 8)) * 8;
    const int c = c0 + cc;
    const int64_t m = m0 + mg;
    if (c < C && m < Kpad)
      *reinterpret_cast<uint4*>(out + (static_cast<int64_t>(t) * C + c) * Kpad + m) =
          *reinterpret_cast<const uint4*>(&tile[at(cc, mg)]);
  }
  vg_bar(nthr);   // the tile is reused by the next virtual block
}

// dW from the GEMM's [Cout][(r*KW + s)*Cin + ci] order to [Cout][Cin][KH][KW].
// a: p0 g, p1 dw; i0 Cout, i1 Cin, i2 KH, i3 KW
VG_FN void vg_wgrad_permute(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const float* g = static_cast<const float*>(a.p[0]);
  float* dw = static_cast<float*>(const_cast<void*>(a.p[1]));
  const int Cout = a.i[0], Cin = a.i[1], KH = a.i[2], KW = a.i[3];
  VG_LOOP(i, static_cast<int64_t>(Cout) * Cin * KH * KW) {
    const int s = static_cast<int>(i % KW), r = static_cast<int>((i / KW) % KH);
    const int ci = static_cast<int>((i / (KW * KH)) % Cin), co = static_cast<int>(i / (static_cast<int64_t>(KW) * KH * Cin));
    dw[i] = g[static_cast<int64_t>(co) * (KH * KW * Cin) + (r * KW + s) * Cin + ci];
  }
}

// Weight-gradient split-K reduction: per-split partial tiles ([tile][split]
// [bn/4][128 rows] float4) summed in split order straight into dW's
// [Cout][Cin][KH][KW] layout.  a: p0 part, p1 dw; i0 Cout, i1 Cin, i2 KH,
// i3 KW, i4 bn, i5 tiles_n, i6 split
VG_FN void vg_wgrad_reduce(const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t*) {
  const float4* part = static_cast<const float4*>(a.p[0]);
  float* dw = static_cast<float*>(const_cast<void*>(a.p[1]));
  const int Cout = a.i[0], Cin = a.i[1], KH = a.i[2], KW = a.i[3], bn = a.i[4], tiles_n = a.i[5], split = a.i[6];
  const int Ng = KH * KW * Cin;
  const int g4 = (Ng + 3) / 4;
  VG_LOOP(i, static_cast<int64_t>(g4) * Cout) {
    const int co = static_cast<int>(i % Cout), q = static_cast<int>(i / Cout);
    const int n0 = q * 4;
    const int tile = (co / 128) * tiles_n + n0 / bn;
    const int r = co % 128, c4 = (n0 % bn) / 4;
    const float4* src = part + (static_cast<int64_t>(tile) * split * (bn / 4) + c4) * 128 + r;
    float4 s = src[0];
    for (int ks = 1; ks < split; ++ks) {
      const float4 b = src[static_cast<int64_t>(ks) * (bn / 4) * 128];
      s.x += b.x; s.y += b.y; s.z += b.z; s.w += b.w;
    }
    const float v[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + j;
      if (n >= Ng) break;
      const int tap = n / Cin, ci = n % Cin;
      dw[((static_cast<int64_t>(co) * Cin + ci) * KH + tap / KW) * KW + tap % KW] = v[j];
    }
  }
}

// ------------------------------------------------------------------ staged streaming
// The elementwise operators (BN apply, ReLU backward, add, SGD) read and write
// whole tensors once: HBM-bound.  Inside the executor only the 192-thread
// worker group of ONE CTA per SM runs them, so register-held loads cannot
// keep enough bytes in flight (~36 KB per SM measured ~0.9 TB/s chip-wide).
// Staged path: one thread streams the item's contiguous range through shared
// memory with bulk async copies (cp.async.bulk, mbarrier complete_tx), NS
// stages of n_in x 8 KB in flight; the group computes in place and one
// thread writes each chunk back with a bulk store.  Same per-element IEEE
// operations as the register path (results bit-identical); only the
// element -> thread assignment differs.
constexpr int VGS_CH = 512;                   // min 16-byte groups per chunk (8 KB per tensor)
#ifndef GACER_VGS_CH_MAX
#define GACER_VGS_CH_MAX 2048
#endif
constexpr int VGS_CH_MAX = GACER_VGS_CH_MAX;  // max groups per chunk (32 KB per tensor)
constexpr int VGS_MIN_STAGES = 4;
constexpr int VGS_MAX_STAGES = 8;

__device__ __forceinline__ uint32_t vgs_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void vgs_mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(vgs_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void vgs_mbar_inval(uint64_t* b) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(vgs_u32(b)) : "memory");
}
__device__ __forceinline__ void vgs_mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(vgs_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void vgs_mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\nVGS_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra VGS_WAIT;\n}\n" ::"r"(vgs_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void vgs_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(vgs_u32(dst)), "l"(src), "r"(bytes), "r"(vgs_u32(bar)) : "memory");
}
__device__ __forceinline__ void vgs_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
               ::"l"(dst), "r"(vgs_u32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void vgs_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void vgs_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void vgs_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
__device__ __forceinline__ void vgs_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// Operators as staged-stream kernels: in-place compute on the smem chunk.
//   n_in input tensors (16-byte groups), results written over slot out_slot[k]
//   and stored to out[k].  prepare(): per-item constants into `extra` smem.
struct VgsBnApply {   // a: p0 x, p1 dy, p2 ym, p3 coef, p4 out; n0 M; i0 mode, i1 C, i2 relu
  const VArgs& a;
  int n_in, C, G8, mode, relu;
  __device__ explicit VgsBnApply(const VArgs& a_) : a(a_) {
    mode = a.i[0]; C = a.i[1]; G8 = C / 8; relu = a.i[2];
    n_in = mode == 0 ? 1 : (a.p[2] ? 3 : 2);
  }
  __device__ const void* in(int k) const { return a.p[k]; }
  __device__ int n_out() const { return 1; }
  __device__ void* out(int) const { return const_cast<void*>(a.p[4]); }
  __device__ int out_slot(int) const { return 0; }
  __device__ int extra_bytes() const { return (mode == 0 ? 2 : 3) * C * 4; }
  __device__ void prepare(float* ex, int tid, int nthr) const {
    const float* coef = static_cast<const float*>(a.p[3]);
    const int n = (mode == 0 ? 2 : 3) * C;
    for (int i = tid; i < n; i += nthr) ex[i] = coef[i];
  }
  __device__ void apply(uint4* const* sl, int j, int64_t gi, const float* ex) const {
    const int c = static_cast<int>(gi % G8) * 8;
    float v[8];
    vg_unpack8(sl[0][j], v);
    const float4* k0 = reinterpret_cast<const float4*>(ex + c);
    const float4* k1 = reinterpret_cast<const float4*>(ex + C + c);
    const float4 a0 = k0[0], a1 = k0[1], b0 = k1[0], b1 = k1[1];
    const float K0[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float K1[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    if (mode == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float t = fmaf(v[q], K0[q], K1[q]);
        v[q] = relu ? fmaxf(t, 0.0f) : t;
      }
    } else {
      const float4* k2 = reinterpret_cast<const float4*>(ex + 2 * C + c);
      const float4 c0 = k2[0], c1 = k2[1];
      const float K2[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      float d[8];
      vg_unpack8(sl[1][j], d);
      if (n_in == 3) {
        float mk[8];
        vg_unpack8(sl[2][j], mk);
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = mk[q] > 0.0f ? d[q] : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = fmaf(K0[q], d[q], fmaf(K1[q], v[q], K2[q]));
    }
    sl[0][j] = vg_pack8(v);
  }
};
struct VgsReluBwd {   // a: p0 x, p1 dy, p2 dx; n0 n8; i0 six
  const VArgs& a;
  int n_in = 2;
  __device__ explicit VgsReluBwd(const VArgs& a_) : a(a_) {}
  __device__ const void* in(int k) const { return a.p[k]; }
  __device__ int n_out() const { return 1; }
  __device__ void* out(int) const { return const_cast<void*>(a.p[2]); }
  __device__ int out_slot(int) const { return 1; }
  __device__ int extra_bytes() const { return 0; }
  __device__ void prepare(float*, int, int) const {}
  __device__ void apply(uint4* const* sl, int j, int64_t, const float*) const {
    const int six = a.i[0];
    float v[8], d[8];
    vg_unpack8(sl[0][j], v);
    vg_unpack8(sl[1][j], d);
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = (v[q] > 0.0f && (!six || v[q] < 6.0f)) ? d[q] : 0.0f;
    sl[1][j] = vg_pack8(d);
  }
};
struct VgsAdd {       // a: p0 a, p1 b, p2 y; n0 n8; i0 relu
  const VArgs& a;
  int n_in = 2;
  __device__ explicit VgsAdd(const VArgs& a_) : a(a_) {}
  __device__ const void* in(int k) const { return a.p[k]; }
  __device__ int n_out() const { return 1; }
  __device__ void* out(int) const { return const_cast<void*>(a.p[2]); }
  __device__ int out_slot(int) const { return 0; }
  __device__ int extra_bytes() const { return 0; }
  __device__ void prepare(float*, int, int) const {}
  __device__ void apply(uint4* const* sl, int j, int64_t, const float*) const {
    const int relu = a.i[0];
    float p[8], q8[8];
    vg_unpack8(sl[0][j], p);
    vg_unpack8(sl[1][j], q8);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float t = p[q] + q8[q];
      p[q] = relu ? fmaxf(t, 0.0f) : t;
    }
    sl[0][j] = vg_pack8(p);
  }
};
struct VgsSgd {       // fp32 float4 groups.  a: p0 w, p1 g, p2 buf; n0 n; i0 first; f0 lr, f1 momentum
  const VArgs& a;
  int n_in = 3;
  __device__ explicit VgsSgd(const VArgs& a_) : a(a_) {}
  __device__ const void* in(int k) const { return a.p[k]; }
  __device__ int n_out() const { return 2; }
  __device__ void* out(int k) const { return const_cast<void*>(a.p[k == 0 ? 0 : 2]); }
  __device__ int out_slot(int k) const { return k == 0 ? 0 : 2; }
  __device__ int extra_bytes() const { return 0; }
  __device__ void prepare(float*, int, int) const {}
  __device__ void apply(uint4* const* sl, int j, int64_t, const float*) const {
    const int first = a.i[0];
    const float lr = a.f[0], mom = a.f[1];
    float* w = reinterpret_cast<float*>(sl[0] + j);
    const float* g = reinterpret_cast<const float*>(sl[1] + j);
    float* buf = reinterpret_cast<float*>(sl[2] + j);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float b = first ? g[q] : fmaf(mom, buf[q], g[q]);
      buf[q] = b;
      w[q] = fmaf(-lr, b, w[q]);
    }
  }
};

// Stream 16-byte groups [g0, g1) of the operator through `smem` (smem_bytes).
template <class Op>
__device__ void vgs_run(const Op& op, int64_t g0, int64_t g1, int tid, int nthr, uint8_t* smem, int smem_bytes) {
  if (g1 <= g0) return;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                      // [VGS_MAX_STAGES]
  float* extra = reinterpret_cast<float*>(smem + 128);
  const int ex_bytes = (op.extra_bytes() + 127) & ~127;
  uint8_t* stages = smem + 128 + ex_bytes;
  // chunk size: the largest that still gives VGS_MIN_STAGES stages (the
  // per-chunk cost -- barrier, fence, bulk-store issue -- is ~0.6 us, so
  // 8 KB chunks capped a streaming operator at ~12 GB/s per SM)
  int ch = (smem_bytes - 128 - ex_bytes) / (VGS_MIN_STAGES * op.n_in * 16);
  ch = ch > VGS_CH_MAX ? VGS_CH_MAX : (ch < VGS_CH ? VGS_CH : ch);
  ch &= ~31;
  const int stage_bytes = op.n_in * ch * 16;
  int ns = (smem_bytes - 128 - ex_bytes) / stage_bytes;
  ns = ns > VGS_MAX_STAGES ? VGS_MAX_STAGES : ns;
  const int64_t nch = (g1 - g0 + ch - 1) / ch;
  auto chunk_len = [&](int64_t k) -> int {
    const int64_t b = g0 + k * ch, e = b + ch < g1 ? b + ch : g1;
    return static_cast<int>(e - b);
  };
  auto issue_load = [&](int64_t k) {
    const int st = static_cast<int>(k % ns);
    const int len = chunk_len(k);
    const uint32_t bytes = static_cast<uint32_t>(len) * 16u;
    vgs_mbar_expect(&bars[st], bytes * op.n_in);
    for (int t = 0; t < op.n_in; ++t)
      vgs_load(stages + st * stage_bytes + t * ch * 16,
               static_cast<const uint8_t*>(op.in(t)) + (g0 + k * ch) * 16, bytes, &bars[st]);
  };
  if (tid == 0) {
    for (int st = 0; st < ns; ++st) vgs_mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.global;\n" ::: "memory");   // acquired inputs -> the async proxy
    for (int64_t k = 0; k < nch && k < ns; ++k) issue_load(k);
  }
  op.prepare(extra, tid, nthr);
  vg_bar(nthr);
  for (int64_t k = 0; k < nch; ++k) {
    const int st = static_cast<int>(k % ns);
    vgs_mbar_wait(&bars[st], static_cast<uint32_t>((k / ns) & 1));
    uint4* sl[3];
    for (int t = 0; t < 3; ++t)
      sl[t] = reinterpret_cast<uint4*>(stages + st * stage_bytes + (t < op.n_in ? t : 0) * ch * 16);
    const int len = chunk_len(k);
    const int64_t base = g0 + k * ch;
    for (int j = tid; j < len; j += nthr) op.apply(sl, j, base + j, extra);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic smem writes -> bulk store
    vg_bar(nthr);
    if (tid == 0) {
      for (int o = 0; o < op.n_out(); ++o)
        vgs_store(static_cast<uint8_t*>(op.out(o)) + base * 16, sl[op.out_slot(o)], static_cast<uint32_t>(len) * 16u);
      vgs_commit();
      if (ns >= 2) {
        // refill the PREVIOUS chunk's stage: its store (one group back) has
        // long been read out, while waiting for this chunk's store here would
        // stall the single issuing thread once per 8 KB chunk (the streaming
        // operators then ran at ~12 GB/s per SM)
        if (k >= 1 && k - 1 + ns < nch) {
          vgs_wait_read1();
          issue_load(k - 1 + ns);
        }
      } else if (k + ns < nch) {
        vgs_wait_read0();   // the stage's results are read out before it is refilled
        issue_load(k + ns);
      }
    }
  }
  if (tid == 0) {
    vgs_wait0();                                           // results written before the item is released
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    for (int st = 0; st < ns; ++st) vgs_mbar_inval(&bars[st]);
  }
  vg_bar(nthr);
}

__device__ __forceinline__ bool vg_streamable(int fn) {
  return fn == VF_BN_APPLY || fn == VF_RELU_BWD || fn == VF_ADD || fn == VF_SGD;
}

// Virtual blocks [v0, v1) of an nvb-block streaming operator, staged: the
// blocks' 16-byte groups form one contiguous range (block vb owns groups
// [vb * per, (vb + 1) * per)).  SGD's fp32 tail (n % 4) is done by thread 0 of
// the item that owns the last group.
VG_FN void vg_stream_item(int fn, const VArgs& a, int v0, int v1, int nvb, int tid, int nthr, uint8_t* smem,
                          int smem_bytes) {
  int64_t total;
  switch (fn) {
    case VF_BN_APPLY: total = a.n[0] * (a.i[1] / 8); break;
    case VF_SGD: total = a.n[0] / 4; break;
    default: total = a.n[0]; break;
  }
  const int64_t per = (total + nvb - 1) / nvb;
  const int64_t g0 = v0 * per < total ? v0 * per : total;
  const int64_t g1 = v1 * per < total ? v1 * per : total;
  switch (fn) {
    case VF_BN_APPLY: vgs_run(VgsBnApply(a), g0, g1, tid, nthr, smem, smem_bytes); break;
    case VF_RELU_BWD: vgs_run(VgsReluBwd(a), g0, g1, tid, nthr, smem, smem_bytes); break;
    case VF_ADD: vgs_run(VgsAdd(a), g0, g1, tid, nthr, smem, smem_bytes); break;
    case VF_SGD: {
      vgs_run(VgsSgd(a), g0, g1, tid, nthr, smem, smem_bytes);
      if (v1 >= nvb && tid == 0) {   // fp32 tail past the last full float4 group
        float* w = static_cast<float*>(const_cast<void*>(a.p[0]));
        const float* g = static_cast<const float*>(a.p[1]);
        float* buf = static_cast<float*>(const_cast<void*>(a.p[2]));
        for (int64_t i = total * 4; i < a.n[0]; ++i) {
          const float b = a.i[0] ? g[i] : fmaf(a.f[1], buf[i], g[i]);
          buf[i] = b;
          w[i] = fmaf(-a.f[0], b, w[i]);
        }
      }
      break;
    }
    default: break;
  }
}

// ------------------------------------------------------------------ dispatch
__device__ inline void run_vgrid(int fn, const VArgs& a, int vb, int nvb, int tid, int nthr, uint8_t* smem) {
  switch (fn) {
    case VF_BN_PARTIAL: vg_bn_partial(a, vb, nvb, tid, nthr, smem); break;
    case VF_BN_FINALIZE: vg_bn_finalize(a, vb, nvb, tid, nthr, smem); break;
    case VF_BN_APPLY: vg_bn_apply(a, vb, nvb, tid, nthr, smem); break;
    case VF_RELU_BWD: vg_relu_bwd(a, vb, nvb, tid, nthr, smem); break;
    case VF_ADD: vg_add(a, vb, nvb, tid, nthr, smem); break;
    case VF_MAXPOOL_FWD: vg_maxpool_fwd(a, vb, nvb, tid, nthr, smem); break;
    case VF_MAXPOOL_ARGMAX: vg_maxpool_argmax(a, vb, nvb, tid, nthr, smem); break;
    case VF_MAXPOOL_BWD: vg_maxpool_bwd(a, vb, nvb, tid, nthr, smem); break;
    case VF_GAP_FWD: vg_gap_fwd(a, vb, nvb, tid, nthr, smem); break;
    case VF_GAP_BWD: vg_gap_bwd(a, vb, nvb, tid, nthr, smem); break;
    case VF_LINEAR_FWD: vg_linear_fwd(a, vb, nvb, tid, nthr, smem); break;
    case VF_LINEAR_DX: vg_linear_dx(a, vb, nvb, tid, nthr, smem); break;
    case VF_LINEAR_DW: vg_linear_dw(a, vb, nvb, tid, nthr, smem); break;
    case VF_SOFTMAX_CE: vg_softmax_ce(a, vb, nvb, tid, nthr, smem); break;
    case VF_MEAN: vg_mean(a, vb, nvb, tid, nthr, smem); break;
    case VF_SGD: vg_sgd(a, vb, nvb, tid, nthr, smem); break;
    case VF_FILTER: vg_filter(a, vb, nvb, tid, nthr, smem); break;
    case VF_FILTER_ALL: vg_filter_all(a, vb, nvb, tid, nthr, smem); break;
    case VF_DILATE: vg_dilate(a, vb, nvb, tid, nthr, smem); break;
    case VF_PHASE_SCATTER: vg_phase_scatter(a, vb, nvb, tid, nthr, smem); break;
    case VF_TRANSPOSE_IM2COL: vg_transpose_im2col(a, vb, nvb, tid, nthr, smem); break;
    case VF_WGRAD_PERMUTE: vg_wgrad_permute(a, vb, nvb, tid, nthr, smem); break;
    case VF_WGRAD_REDUCE: vg_wgrad_reduce(a, vb, nvb, tid, nthr, smem); break;
    default: break;
  }
}

}  // namespace gacer
