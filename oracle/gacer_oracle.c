/*
 * gacer_oracle.c -- plain fp64 CPU operators for the GACER parity oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header or constant with paper_2304_11745_b200/.
 *
 * GACER (arXiv 2304.11745) is a scheduling method: a regulated multi-tenant
 * round computes, for every tenant n, exactly y_n = M_n(x_n), the result of
 * running the model alone ("without sacrificing model accuracy", PAPER.md
 * §4.2 l.674).  The oracle is therefore the plain definition of each
 * operator of the tenants' DFGs (PyTorch eval-mode semantics, SURVEY.md
 * §8(c) C1), in fp64, NCHW, written as direct loops with no blocking, fusion
 * or reordering.  OpenMP parallelises over independent output elements only;
 * every output is summed in one fixed order.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

/* conv2d (C1): y[n,co,ho,wo] = b[co] + sum_{ci in group(co), r, s}
 *   w[co, ci, r, s] * x[n, g*Cig + ci, ho*stride - ph + r, wo*stride - pw + s],
 * out-of-bounds taps contribute 0.  Dilation 1. */
void oracle_conv2d(const double* x, const double* w, const double* b,
                   int N, int Cin, int H, int W, int Cout, int KH, int KW,
                   int stride, int ph, int pw, int groups,
                   int Ho, int Wo, double* y) {
  const int Cig = Cin / groups, Cog = Cout / groups;
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int co = 0; co < Cout; ++co) {
      const int g = co / Cog;
      for (int ho = 0; ho < Ho; ++ho)
        for (int wo = 0; wo < Wo; ++wo) {
          double acc = b ? b[co] : 0.0;
          for (int ci = 0; ci < Cig; ++ci)
            for (int r = 0; r < KH; ++r) {
              const int hi = ho * stride - ph + r;
              if (hi < 0 || hi >= H) continue;
              for (int s = 0; s < KW; ++s) {
                const int wi = wo * stride - pw + s;
                if (wi < 0 || wi >= W) continue;
                acc += w[(((size_t)co * Cig + ci) * KH + r) * KW + s] *
                       x[(((size_t)n * Cin + g * Cig + ci) * H + hi) * W + wi];
              }
            }
          y[(((size_t)n * Cout + co) * Ho + ho) * Wo + wo] = acc;
        }
    }
}

/* BatchNorm2d inference (C1): gamma * (x - mean) / sqrt(var + eps) + beta */
void oracle_batchnorm(const double* x, int N, int C, int HW,
                      const double* gamma, const double* beta,
                      const double* mean, const double* var, double eps,
                      double* y) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) {
      const double inv = 1.0 / sqrt(var[c] + eps);
      for (int i = 0; i < HW; ++i) {
        const size_t k = ((size_t)n * C + c) * HW + i;
        y[k] = gamma[c] * (x[k] - mean[c]) * inv + beta[c];
      }
    }
}

/* ReLU: max(0,x); ReLU6: min(max(0,x),6) */
void oracle_relu(const double* x, size_t n, int six, double* y) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) {
    double v = x[i] > 0.0 ? x[i] : 0.0;
    if (six && v > 6.0) v = 6.0;
    y[i] = v;
  }
}

/* max-pool, floor mode, implicit -inf padding (C1) */
void oracle_maxpool(const double* x, int N, int C, int H, int W, int KH, int KW,
                    int stride, int ph, int pw, int Ho, int Wo, double* y) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c)
      for (int ho = 0; ho < Ho; ++ho)
        for (int wo = 0; wo < Wo; ++wo) {
          double m = -INFINITY;
          for (int r = 0; r < KH; ++r) {
            const int hi = ho * stride - ph + r;
            if (hi < 0 || hi >= H) continue;
            for (int s = 0; s < KW; ++s) {
              const int wi = wo * stride - pw + s;
              if (wi < 0 || wi >= W) continue;
              const double v = x[(((size_t)n * C + c) * H + hi) * W + wi];
              if (v > m) m = v;
            }
          }
          y[(((size_t)n * C + c) * Ho + ho) * Wo + wo] = m;
        }
}

/* avg-pool, floor mode; count_include_pad => divisor KH*KW, else the number
 * of in-bounds taps (C1: Inception's F.avg_pool2d default is cip = True) */
void oracle_avgpool(const double* x, int N, int C, int H, int W, int KH, int KW,
                    int stride, int ph, int pw, int cip, int Ho, int Wo, double* y) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c)
      for (int ho = 0; ho < Ho; ++ho)
        for (int wo = 0; wo < Wo; ++wo) {
          double acc = 0.0;
          int cnt = 0;
          for (int r = 0; r < KH; ++r) {
            const int hi = ho * stride - ph + r;
            for (int s = 0; s < KW; ++s) {
              const int wi = wo * stride - pw + s;
              /* taps inside the padded frame count when cip */
              if (hi < -ph || hi >= H + ph || wi < -pw || wi >= W + pw) continue;
              if (cip) ++cnt;
              if (hi < 0 || hi >= H || wi < 0 || wi >= W) continue;
              if (!cip) ++cnt;
              acc += x[(((size_t)n * C + c) * H + hi) * W + wi];
            }
          }
          y[(((size_t)n * C + c) * Ho + ho) * Wo + wo] = acc / (double)cnt;
        }
}

/* global average pool: mean over H*W */
void oracle_gap(const double* x, int N, int C, int HW, double* y) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
      for (int i = 0; i < HW; ++i) acc += x[((size_t)n * C + c) * HW + i];
      y[(size_t)n * C + c] = acc / (double)HW;
    }
}

/* linear: y[n,o] = b[o] + sum_k w[o,k] x[n,k] */
void oracle_linear(const double* x, const double* w, const double* b,
                   int N, int K, int O, double* y) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int o = 0; o < O; ++o) {
      double acc = b ? b[o] : 0.0;
      for (int k = 0; k < K; ++k) acc += w[(size_t)o * K + k] * x[(size_t)n * K + k];
      y[(size_t)n * O + o] = acc;
    }
}

/* elementwise add */
void oracle_add(const double* a, const double* b, size_t n, double* y) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) y[i] = a[i] + b[i];
}

/* hardswish (MobileNetV3, PyTorch Hardswish): y = x * relu6(x + 3) / 6 */
void oracle_hardswish(const double* x, size_t n, double* y) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) {
    double t = x[i] + 3.0;
    t = t < 0.0 ? 0.0 : (t > 6.0 ? 6.0 : t);
    y[i] = x[i] * t / 6.0;
  }
}

/* hardsigmoid (PyTorch Hardsigmoid, the SE gate of MobileNetV3):
 * y = relu6(x + 3) / 6 */
void oracle_hardsigmoid(const double* x, size_t n, double* y) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) {
    double t = x[i] + 3.0;
    t = t < 0.0 ? 0.0 : (t > 6.0 ? 6.0 : t);
    y[i] = t / 6.0;
  }
}

/* channel scale (squeeze-and-excitation): y[n,c,p] = x[n,c,p] * s[n,c] */
void oracle_scale_channels(const double* x, const double* s, int N, int C, int HW, double* y) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c)
      for (int p = 0; p < HW; ++p)
        y[((size_t)n * C + c) * HW + p] = x[((size_t)n * C + c) * HW + p] * s[(size_t)n * C + c];
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
