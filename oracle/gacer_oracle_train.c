/*
 * gacer_oracle_train.c -- plain fp64 CPU backward operators and the SGD update
 * for the training tenant (SURVEY.md §8(a) A11, §8(c) "Training").
 *
 * TEST INFRASTRUCTURE ONLY (same rules as gacer_oracle.c): only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library; it shares nothing with paper_2304_11745_b200/.
 *
 * The paper trains with PyTorch defaults (§5.1 l.903-911 names the
 * models; the training step itself is not specified -- SURVEY §8(c): loss =
 * mean softmax cross-entropy, SGD momentum 0.9, lr 0.1, BN in training mode
 * with per-replica batch statistics; all "proposed").  Each function is the
 * textbook derivative of the forward definition in gacer_oracle.c, written as
 * direct loops in fp64, NCHW, one fixed summation order per output.
 */
#include <math.h>
#include <stddef.h>
#include <string.h>

/* conv2d data gradient: y[n,co,ho,wo] = sum w[co,ci,r,s] x[n,g*Cig+ci,hi,wi]
 * with hi = ho*stride - ph + r, wi = wo*stride - pw + s, so
 *   dx[n, g*Cig+ci, hi, wi] = sum_{co in group g, ho, wo, r, s : taps hit (hi,wi)}
 *                              dy[n,co,ho,wo] * w[co,ci,r,s].
 * Written as a scatter over (co, ho, wo, ci, r, s) per sample n; samples are
 * independent (OpenMP over n), the order inside a sample is fixed. */
void oracle_conv2d_bwd_data(const double* dy, const double* w, int N, int Cin, int H, int W,
                            int Cout, int KH, int KW, int stride, int ph, int pw, int groups,
                            int Ho, int Wo, double* dx) {
  const int Cig = Cin / groups, Cog = Cout / groups;
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n) {
    double* dxn = dx + (size_t)n * Cin * H * W;
    memset(dxn, 0, sizeof(double) * (size_t)Cin * H * W);
    for (int co = 0; co < Cout; ++co) {
      const int g = co / Cog;
      for (int ho = 0; ho < Ho; ++ho)
        for (int wo = 0; wo < Wo; ++wo) {
          const double d = dy[(((size_t)n * Cout + co) * Ho + ho) * Wo + wo];
          for (int ci = 0; ci < Cig; ++ci)
            for (int r = 0; r < KH; ++r) {
              const int hi = ho * stride - ph + r;
              if (hi < 0 || hi >= H) continue;
              for (int s = 0; s < KW; ++s) {
                const int wi = wo * stride - pw + s;
                if (wi < 0 || wi >= W) continue;
                dxn[((size_t)(g * Cig + ci) * H + hi) * W + wi] +=
                    d * w[(((size_t)co * Cig + ci) * KH + r) * KW + s];
              }
            }
        }
    }
  }
}

/* conv2d weight / bias gradient:
 *   dw[co,ci,r,s] = sum_{n,ho,wo} dy[n,co,ho,wo] * x[n, g*Cig+ci, hi, wi]  (in-bounds taps)
 *   db[co]        = sum_{n,ho,wo} dy[n,co,ho,wo]                            (db may be NULL) */
void oracle_conv2d_bwd_weight(const double* x, const double* dy, int N, int Cin, int H, int W,
                              int Cout, int KH, int KW, int stride, int ph, int pw, int groups,
                              int Ho, int Wo, double* dw, double* db) {
  const int Cig = Cin / groups, Cog = Cout / groups;
#pragma omp parallel for schedule(static)
  for (int co = 0; co < Cout; ++co) {
    const int g = co / Cog;
    for (int ci = 0; ci < Cig; ++ci)
      for (int r = 0; r < KH; ++r)
        for (int s = 0; s < KW; ++s) {
          double acc = 0.0;
          for (int n = 0; n < N; ++n)
            for (int ho = 0; ho < Ho; ++ho) {
              const int hi = ho * stride - ph + r;
              if (hi < 0 || hi >= H) continue;
              for (int wo = 0; wo < Wo; ++wo) {
                const int wi = wo * stride - pw + s;
                if (wi < 0 || wi >= W) continue;
                acc += dy[(((size_t)n * Cout + co) * Ho + ho) * Wo + wo] *
                       x[(((size_t)n * Cin + g * Cig + ci) * H + hi) * W + wi];
              }
            }
          dw[(((size_t)co * Cig + ci) * KH + r) * KW + s] = acc;
        }
    if (db) {
      double acc = 0.0;
      for (int n = 0; n < N; ++n)
        for (int i = 0; i < Ho * Wo; ++i) acc += dy[((size_t)n * Cout + co) * Ho * Wo + i];
      db[co] = acc;
    }
  }
}

/* BatchNorm, training mode (per-batch statistics over n and the HW
 * positions, M = N*HW values per channel; biased variance in the
 * normalisation, PyTorch semantics):
 *   mean_c = (1/M) sum x,  var_c = (1/M) sum (x - mean_c)^2,
 *   y = gamma_c (x - mean_c) / sqrt(var_c + eps) + beta_c. */
void oracle_bn_train_fwd(const double* x, int N, int C, int HW, const double* gamma,
                         const double* beta, double eps, double* y, double* mean, double* var) {
  const double M = (double)N * HW;
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    double s = 0.0;
    for (int n = 0; n < N; ++n)
      for (int i = 0; i < HW; ++i) s += x[((size_t)n * C + c) * HW + i];
    const double mu = s / M;
    double q = 0.0;
    for (int n = 0; n < N; ++n)
      for (int i = 0; i < HW; ++i) {
        const double d = x[((size_t)n * C + c) * HW + i] - mu;
        q += d * d;
      }
    const double v = q / M;
    const double inv = 1.0 / sqrt(v + eps);
    for (int n = 0; n < N; ++n)
      for (int i = 0; i < HW; ++i) {
        const size_t k = ((size_t)n * C + c) * HW + i;
        y[k] = gamma[c] * (x[k] - mu) * inv + beta[c];
      }
    mean[c] = mu;
    var[c] = v;
  }
}

/* BatchNorm training backward (chain rule through mean and var; xhat =
 * (x - mean)/sqrt(var + eps)):
 *   dbeta_c  = sum dy,   dgamma_c = sum dy * xhat,
 *   dx = gamma_c / sqrt(var_c + eps) * (dy - dbeta_c / M - xhat * dgamma_c / M). */
void oracle_bn_train_bwd(const double* x, const double* dy, int N, int C, int HW,
                         const double* gamma, const double* mean, const double* var, double eps,
                         double* dx, double* dgamma, double* dbeta) {
  const double M = (double)N * HW;
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    const double inv = 1.0 / sqrt(var[c] + eps);
    double sb = 0.0, sg = 0.0;
    for (int n = 0; n < N; ++n)
      for (int i = 0; i < HW; ++i) {
        const size_t k = ((size_t)n * C + c) * HW + i;
        sb += dy[k];
        sg += dy[k] * (x[k] - mean[c]) * inv;
      }
    for (int n = 0; n < N; ++n)
      for (int i = 0; i < HW; ++i) {
        const size_t k = ((size_t)n * C + c) * HW + i;
        const double xh = (x[k] - mean[c]) * inv;
        dx[k] = gamma[c] * inv * (dy[k] - sb / M - xh * sg / M);
      }
    dgamma[c] = sg;
    dbeta[c] = sb;
  }
}

/* ReLU / ReLU6 backward on the forward INPUT x: dx = dy where 0 < x (and
 * x < 6 for ReLU6), else 0 (PyTorch's subgradient 0 at the kinks). */
void oracle_relu_bwd(const double* x, const double* dy, size_t n, int six, double* dx) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) {
    const int pass = x[i] > 0.0 && (!six || x[i] < 6.0);
    dx[i] = pass ? dy[i] : 0.0;
  }
}

/* max-pool backward: each output's gradient goes to the FIRST maximum of its
 * window in row-major (r, s) order; padded taps never win. */
void oracle_maxpool_bwd(const double* x, const double* dy, int N, int C, int H, int W, int KH,
                        int KW, int stride, int ph, int pw, int Ho, int Wo, double* dx) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) {
      const double* xp = x + ((size_t)n * C + c) * H * W;
      double* dxp = dx + ((size_t)n * C + c) * H * W;
      memset(dxp, 0, sizeof(double) * (size_t)H * W);
      for (int ho = 0; ho < Ho; ++ho)
        for (int wo = 0; wo < Wo; ++wo) {
          int best = -1;
          double m = -INFINITY;
          for (int r = 0; r < KH; ++r) {
            const int hi = ho * stride - ph + r;
            if (hi < 0 || hi >= H) continue;
            for (int s = 0; s < KW; ++s) {
              const int wi = wo * stride - pw + s;
              if (wi < 0 || wi >= W) continue;
              if (best < 0 || xp[hi * W + wi] > m) { m = xp[hi * W + wi]; best = hi * W + wi; }
            }
          }
          if (best >= 0) dxp[best] += dy[(((size_t)n * C + c) * Ho + ho) * Wo + wo];
        }
    }
}

/* global average pool backward: dx[n,c,i] = dy[n,c] / HW. */
void oracle_gap_bwd(const double* dy, int N, int C, int HW, double* dx) {
  for (size_t k = 0; k < (size_t)N * C; ++k)
    for (int i = 0; i < HW; ++i) dx[k * HW + i] = dy[k] / HW;
}

/* linear backward, y[n,o] = b[o] + sum_k w[o,k] x[n,k]:
 *   dx[n,k] = sum_o dy[n,o] w[o,k],  dw[o,k] = sum_n dy[n,o] x[n,k],
 *   db[o] = sum_n dy[n,o]  (db may be NULL). */
void oracle_linear_bwd(const double* x, const double* w, const double* dy, int N, int K, int O,
                       double* dx, double* dw, double* db) {
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      double acc = 0.0;
      for (int o = 0; o < O; ++o) acc += dy[(size_t)n * O + o] * w[(size_t)o * K + k];
      dx[(size_t)n * K + k] = acc;
    }
#pragma omp parallel for schedule(static)
  for (int o = 0; o < O; ++o) {
    for (int k = 0; k < K; ++k) {
      double acc = 0.0;
      for (int n = 0; n < N; ++n) acc += dy[(size_t)n * O + o] * x[(size_t)n * K + k];
      dw[(size_t)o * K + k] = acc;
    }
    if (db) {
      double acc = 0.0;
      for (int n = 0; n < N; ++n) acc += dy[(size_t)n * O + o];
      db[o] = acc;
    }
  }
}

/* mean softmax cross-entropy over the batch and its gradient:
 *   loss = (1/N) sum_n [log sum_j exp(z[n,j]) - z[n, label_n]],
 *   dz[n,j] = (softmax(z_n)_j - [j == label_n]) / N.
 * The row maximum is subtracted before exp (an identity of the definition). */
double oracle_softmax_ce(const double* z, const int* labels, int N, int Cls, double* dz) {
  double loss = 0.0;
  for (int n = 0; n < N; ++n) {
    const double* zr = z + (size_t)n * Cls;
    double m = zr[0];
    for (int j = 1; j < Cls; ++j) m = zr[j] > m ? zr[j] : m;
    double s = 0.0;
    for (int j = 0; j < Cls; ++j) s += exp(zr[j] - m);
    loss += (log(s) + m) - zr[labels[n]];
    for (int j = 0; j < Cls; ++j)
      dz[(size_t)n * Cls + j] = (exp(zr[j] - m) / s - (j == labels[n] ? 1.0 : 0.0)) / N;
  }
  return loss / N;
}

/* SGD with momentum (PyTorch semantics, dampening 0, no Nesterov, no weight
 * decay): buf = g on the first step, else buf = momentum * buf + g;
 * w -= lr * buf.  Updates w and buf in place. */
void oracle_sgd_momentum(double* w, const double* g, double* buf, size_t n, double lr,
                         double momentum, int first) {
  for (size_t i = 0; i < n; ++i) {
    buf[i] = first ? g[i] : momentum * buf[i] + g[i];
    w[i] -= lr * buf[i];
  }
}
