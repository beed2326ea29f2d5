/*
 * gacer_train.h -- C ABI of the training tenant's CUDA-core operators
 * (first part).
 *
 * A training tenant's step (SURVEY §8(c) "Training"; the paper trains with
 * PyTorch defaults and states no hyper-parameters, §5.1 l.903-911)
 * is: forward with BatchNorm in TRAINING mode (statistics of the replica's
 * batch), mean softmax cross-entropy, backward, SGD with momentum.  This
 * header exposes the HBM-bound, non-GEMM steps of that step as stream-ordered
 * device calls, each the device twin of a function of the fp64 oracle
 * (oracle/gacer_oracle_train.c) and checked against it per operator, fed the
 * GPU's own bf16 tensors (SURVEY §8(c) C2b reading (1)).  The tensor-core
 * steps (conv dgrad / wgrad as implicit GEMMs on tcgen05) and the
 * integration of the whole step as executor work items are the next step of
 * A11; the FC backward (0.5 GFLOP for ResNet-50's head) runs on CUDA cores.
 *
 * Conventions:
 *   - every tensor argument is a DEVICE pointer owned by the caller; no call
 *     allocates, frees or synchronises; work is enqueued on `stream`
 *     (a cudaStream_t passed as void*, NULL = legacy default stream).
 *   - activations are NHWC bf16, viewed as a row-major [M][C] matrix with
 *     M = N*H*W rows (the executor's layout); C % 8 == 0 and 16-byte aligned
 *     pointers are required (else GACER_E_SHAPE / GACER_E_INVALID_ARG).
 *   - statistics, gradients of parameters, logits and SGD state are fp32.
 *   - every reduction is summed in one fixed order: results are bitwise
 *     reproducible run to run (north_star H4 applied to training).
 *   - return GACER_OK (0) or a negative gacer_status (gacer.h); launch errors
 *     return GACER_E_CUDA.
 */
#ifndef GACER_TRAIN_H_
#define GACER_TRAIN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scratch floats the BN calls need: 2 * C * P partial sums plus 4 * C
 * per-channel constants, with P = gacer_bn_partials(M, C) row blocks. */
int32_t gacer_bn_partials(int64_t M, int32_t C);

/* BatchNorm training forward (oracle_bn_train_fwd):
 *   mean_c = (1/M) sum_m x[m,c],  var_c = (1/M) sum_m (x[m,c] - mean_c)^2 (biased),
 *   y[m,c] = act(gamma_c (x[m,c] - mean_c) / sqrt(var_c + eps) + beta_c),
 * act = ReLU when relu != 0 (the BN -> ReLU pair of a ResNet block), else
 * identity.  x, y: bf16 [M][C] (y may alias x); gamma, beta: fp32 [C];
 * mean, var: fp32 [C] outputs (saved for the backward); scratch: fp32,
 * gacer_bn_partials(M, C) * 2 * C + 4 * C floats.  Per-block partial sums
 * are fp32 in row order, combined across blocks in fp64 in block order. */
int32_t gacer_bn_train_fwd(const void* x_dev, int64_t M, int32_t C, const float* gamma_dev,
                           const float* beta_dev, float eps, int32_t relu, void* y_dev, float* mean_dev,
                           float* var_dev, float* scratch_dev, void* stream);

/* BatchNorm training backward (oracle_bn_train_bwd), xhat = (x - mean)/sqrt(var + eps):
 *   dbeta_c = sum_m dy,  dgamma_c = sum_m dy * xhat,
 *   dx = gamma_c / sqrt(var_c + eps) * (dy - dbeta_c / M - xhat * dgamma_c / M).
 * x: the BN input (bf16 [M][C]), dy: the gradient of the BN output (bf16),
 * mean/var from gacer_bn_train_fwd; outputs dx (bf16 [M][C], may alias dy),
 * dgamma, dbeta (fp32 [C]); scratch as for the forward.  relu_y (may be
 * NULL): the output of a ReLU fused behind this BN (gacer_bn_train_fwd with
 * relu = 1); dy is then the gradient of that ReLU's output and is masked by
 * relu_y > 0 first (the ReLU backward, oracle_relu_bwd, fused in). */
int32_t gacer_bn_train_bwd(const void* x_dev, const void* dy_dev, const void* relu_y_dev, int64_t M, int32_t C,
                           const float* gamma_dev, const float* mean_dev, const float* var_dev, float eps,
                           void* dx_dev, float* dgamma_dev, float* dbeta_dev, float* scratch_dev, void* stream);

/* ReLU / ReLU6 backward on the forward INPUT x (oracle_relu_bwd):
 * dx = dy where x > 0 (and x < 6 when six != 0), else 0.  bf16 [n]
 * (n % 8 == 0); dx may alias dy. */
int32_t gacer_relu_bwd(const void* x_dev, const void* dy_dev, int64_t n, int32_t six, void* dx_dev,
                       void* stream);

/* Max-pool backward, NHWC (oracle_maxpool_bwd): each output's gradient goes
 * to the FIRST maximum of its window in row-major order,
 * padded taps never win; gradients of an input shared by several windows are
 * summed in (ho, wo) order (a gather: no atomics).  x: bf16 [N][H][W][C],
 * dy: bf16 [N][Ho][Wo][C], dx: bf16 [N][H][W][C]; scratch: N*Ho*Wo*C bytes
 * (8-byte aligned) for the windows' argmax tap indices (KH*KW <= 255). */
int32_t gacer_maxpool_bwd(const void* x_dev, const void* dy_dev, int32_t N, int32_t H, int32_t W, int32_t C,
                          int32_t KH, int32_t KW, int32_t stride, int32_t ph, int32_t pw, int32_t Ho, int32_t Wo,
                          void* dx_dev, void* scratch_dev, void* stream);

/* Global-average-pool backward (oracle_gap_bwd): dx[n,p,c] = dy[n,c] / HW.
 * dy: fp32 [N][C], dx: bf16 [N][HW][C]. */
int32_t gacer_gap_bwd(const float* dy_dev, int32_t N, int32_t HW, int32_t C, void* dx_dev, void* stream);

/* Fully-connected layer backward (oracle_linear_bwd), y[n,o] = b[o] + sum_k w[o,k] x[n,k]:
 *   dx[n,k] = sum_o dy[n,o] w[o,k],  dw[o,k] = sum_n dy[n,o] x[n,k],  db[o] = sum_n dy[n,o].
 * x: bf16 [N][K] (the saved forward input), w: fp32 [O][K] (master weights),
 * dy: fp32 [N][O]; outputs dx fp32 [N][K] (may be NULL), dw fp32 [O][K],
 * db fp32 [O] (may be NULL).  CUDA cores, one output per thread, summed in
 * index order (ResNet-50's head: N=64, K=2048, O=1000, 0.5 GFLOP). */
int32_t gacer_linear_bwd(const void* x_dev, const float* w_dev, const float* dy_dev, int32_t N, int32_t K, int32_t O,
                         float* dx_dev, float* dw_dev, float* db_dev, void* stream);

/* Convolution data gradient (oracle_conv2d_bwd_data) on the tcgen05
 * implicit-GEMM path of the executor.  For a forward conv y = conv(x, w,
 * stride S, pad p):
 *   dx[n,ci,h,w] = sum_{co,ho,wo,r,s : ho*S-p+r = h, wo*S-p+s = w} dy[n,co,ho,wo] w[co,ci,r,s]
 *                = conv_stride1(dilate_S(dy), w', pad K-1-p),
 *   w'[ci,co,r,s] = w[co,ci,K-1-r,K-1-s],
 * i.e. a forward conv of dy (zero-dilated by S, plus the (H+2p-K) mod S
 * trailing rows/columns no window reached) with the flipped, transposed
 * filter.  The call packs w' (bf16, K-major) and, for S > 1, the dilated dy
 * into the workspace, then runs one single-op launch of the executor kernel.
 * dy: bf16 NHWC [N][Ho][Wo][Cout] (Ho = (H+2p-KH)/S + 1); w: fp32
 * [Cout][Cin][KH][KW] (the master weights); dx: bf16 NHWC [N][H][W][Cin].
 * Cout % 64 == 0, Cin % 8 == 0, 0 <= pad <= k-1.  Workspace:
 * gacer_conv_dgrad_workspace(...) bytes, 256-byte aligned.  Requires
 * gacer_init on a device.  (S > 1 spends S^2 x the MMA work on the zeros of
 * the dilated dy; a phase-decomposed dgrad is the planned replacement.) */
int64_t gacer_conv_dgrad_workspace(int32_t N, int32_t H, int32_t W, int32_t Cin, int32_t Cout, int32_t KH, int32_t KW,
                                   int32_t stride, int32_t pad_h, int32_t pad_w);
int32_t gacer_conv_dgrad(const void* dy_dev, const float* w_dev, int32_t N, int32_t H, int32_t W, int32_t Cin,
                         int32_t Cout, int32_t KH, int32_t KW, int32_t stride, int32_t pad_h, int32_t pad_w,
                         void* dx_dev, void* ws_dev, int64_t ws_bytes, void* stream);

/* Convolution weight gradient (oracle_conv2d_bwd_weight) on the tcgen05
 * GEMM path:  dw[co,ci,r,s] = sum_{n,ho,wo} dy[n,co,ho,wo] x[n,ci,ho*S-p+r,wo*S-p+s],
 * a GEMM with M = Cout, N = KH*KW*Cin and the reduction over the
 * N*Ho*Wo output pixels.  Both operands are made K-major along the pixel
 * index (dy^T and the transposed im2col of x, zero-padded to a multiple of
 * 64 pixels) in the workspace, the GEMM runs as one single-op launch of the
 * executor kernel with a fixed split-K (partials summed in split order: the
 * result is deterministic), and dw is written fp32 in the master weights'
 * [Cout][Cin][KH][KW] order.  x: bf16 NHWC [N][H][W][Cin] (the saved
 * forward input); dy: bf16 NHWC [N][Ho][Wo][Cout].  Workspace:
 * gacer_conv_wgrad_workspace(...) bytes, 256-byte aligned (it holds the
 * KH*KW-fold im2col; a streamed im2col producer is the planned replacement).
 * Requires gacer_init on a device. */
int64_t gacer_conv_wgrad_workspace(int32_t N, int32_t H, int32_t W, int32_t Cin, int32_t Cout, int32_t KH, int32_t KW,
                                   int32_t stride, int32_t pad_h, int32_t pad_w);
int32_t gacer_conv_wgrad(const void* x_dev, const void* dy_dev, int32_t N, int32_t H, int32_t W, int32_t Cin,
                         int32_t Cout, int32_t KH, int32_t KW, int32_t stride, int32_t pad_h, int32_t pad_w,
                         float* dw_dev, void* ws_dev, int64_t ws_bytes, void* stream);

/* Training forward conv (the conv of a conv -> BN-train pair: raw output,
 * no folded BN): y = conv(x, w, stride, pad) on the tcgen05 implicit-GEMM
 * path of the executor (one single-op launch), the filter packed to bf16
 * K-major from the device-resident fp32 master weights on every call (they
 * change every SGD step).  x: bf16 NHWC [N][H][W][Cin] (Cin % 8 == 0; TMA
 * im2col when Cin % 64 == 0, else the cp.async gather); w: fp32
 * [Cout][Cin][KH][KW]; y: bf16 NHWC [N][Ho][Wo][Cout] (Cout % 8 == 0).
 * Workspace: gacer_conv_fwd_workspace(...) bytes, 256-byte aligned. */
int64_t gacer_conv_fwd_workspace(int32_t N, int32_t H, int32_t W, int32_t Cin, int32_t Cout, int32_t KH, int32_t KW,
                                 int32_t stride, int32_t pad_h, int32_t pad_w);
int32_t gacer_conv_fwd(const void* x_dev, const float* w_dev, int32_t N, int32_t H, int32_t W, int32_t Cin,
                       int32_t Cout, int32_t KH, int32_t KW, int32_t stride, int32_t pad_h, int32_t pad_w, void* y_dev,
                       void* ws_dev, int64_t ws_bytes, void* stream);

/* Max-pool forward, NHWC bf16 (oracle_maxpool; padded taps never win). */
int32_t gacer_maxpool_fwd(const void* x_dev, int32_t N, int32_t H, int32_t W, int32_t C, int32_t KH, int32_t KW,
                          int32_t stride, int32_t ph, int32_t pw, int32_t Ho, int32_t Wo, void* y_dev, void* stream);

/* Residual add (oracle_add), then ReLU when relu != 0: y = a + b; bf16 [n],
 * n % 8 == 0; y may alias a or b. */
int32_t gacer_add(const void* a_dev, const void* b_dev, int64_t n, int32_t relu, void* y_dev, void* stream);

/* Global average pool forward (oracle_gap): y[n][c] = (1/HW) sum_p x[n][p][c],
 * fp32 sum in pixel order; x bf16 [N][HW][C], y bf16 [N][C]. */
int32_t gacer_gap_fwd(const void* x_dev, int32_t N, int32_t HW, int32_t C, void* y_dev, void* stream);

/* FC forward (oracle_linear): z[n][o] = b[o] + sum_k w[o][k] x[n][k]; x bf16
 * [N][K], w fp32 [O][K], b fp32 [O] (may be NULL), z fp32 [N][O] (logits).
 * One warp per output (lane-strided k, fixed butterfly: deterministic). */
int32_t gacer_linear_fwd(const void* x_dev, const float* w_dev, const float* b_dev, int32_t N, int32_t K, int32_t O,
                         float* z_dev, void* stream);

/* Mean softmax cross-entropy and its gradient (oracle_softmax_ce):
 *   loss = (1/N) sum_n [logsumexp(z_n) - z_n[label_n]],
 *   dz[n,j] = (softmax(z_n)_j - [j == label_n]) / N.
 * z, dz: fp32 [N][Cls] (dz may alias z); labels: int32 [N] in [0, Cls)
 * (out-of-range labels give loss = NaN for that row); loss: one fp32;
 * scratch: N floats (per-row losses, summed in row order in fp64). */
int32_t gacer_softmax_ce(const float* z_dev, const int32_t* labels_dev, int32_t N, int32_t Cls, float* loss_dev,
                         float* dz_dev, float* scratch_dev, void* stream);

/* SGD with momentum, PyTorch semantics (oracle_sgd_momentum):
 * buf = g (first != 0) else momentum * buf + g;  w -= lr * buf.
 * w, g, buf: fp32 [n], updated in place. */
int32_t gacer_sgd_momentum(float* w_dev, const float* g_dev, float* buf_dev, int64_t n, float lr, float momentum,
                           int32_t first, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GACER_TRAIN_H_ */
