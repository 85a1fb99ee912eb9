// Host-side launch API of the sm_100a kernels used by the executor.
// All tensors are fp32, NHWC (channels innermost), batch-major.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sn {

struct ConvShape {
  int N, H, W, C;   // input (C = stored channels; the DATA stem is padded to 4)
  int K, R, S;      // output channels, kernel rows, kernel cols
  int P, Q;         // output spatial
  int stride, pad;
};

// ---- tensor-core GEMM based ops (gemm_ops.cu) --------------------------------
// y[N*P*Q][K] = conv(x, w[K][R][S][C]) + bias.  stats (optional): BatchNorm
// statistics of y per M tile, [tiles][3][K] floats (conv_fwd_stats_tiles), for
// a BN consuming y (bn_stats_from_tiles) -- saves that BN's statistics pass.
cudaError_t conv_fwd(const ConvShape& s, const float* x, const float* w, const float* bias, float* y,
                     cudaStream_t st, float* stats = nullptr);
// Number of statistics tiles the forward (stem: conv_stem_fwd) emits, 0 if it
// cannot; *tile_rows = output rows per tile (the last tile may hold fewer), or
// 0 when each tile carries its own count (4 planes {shift, S1, S2, count}
// instead of 3).  The partial buffer needs tiles * 4 * K floats.
int conv_fwd_stats_tiles(const ConvShape& s, bool stem, int* tile_rows);
// dx[N*H*W][C] (+)= conv_transpose(dy, w); wt = scratch of K*R*S*C floats.
// prepped: wt already holds this layer's transformed dgrad weights (the
// executor prepares every layer's once per step, in one batched launch off the
// backward's dgrad chain: conv_dgrad_prep_job / conv_dgrad_prep_batch).
cudaError_t conv_dgrad(const ConvShape& s, const float* dy, const float* w, float* wt, float* dx,
                       int accumulate, cudaStream_t st, int prepped = 0);
// One layer's dgrad weight transform: the flipped / transposed filter or the
// sub-pixel blocks, exactly what conv_dgrad would launch first.
struct DgradPrepJob {
  const float* w;
  float* wt;
  int K, RS, C, flip, subpix;
};
// Fills *job for this shape's dgrad path under the current knobs; false when
// that path transforms its weights otherwise (the phase-decomposed strided dgrad).
bool conv_dgrad_prep_job(const ConvShape& s, const float* w, float* wt, DgradPrepJob* job);
// All jobs (device array) in one launch.
cudaError_t conv_dgrad_prep_batch(const DgradPrepJob* jobs, int njobs, cudaStream_t st);
// dw[K][R*S*C] = sum_pixels im2col(x)^T dy ; db[K] = column sums of dy (skipped if db is null).
// partial: scratch of splits*R*S*C*K floats (see conv_wgrad_splits).
// the halo weight-gradient kernels: their partial-slice count is fixed by the
// kernel (one per CTA or job), the im2col kernel's split count is free
bool conv_wgrad_splits_fixed(const ConvShape& s);
int conv_wgrad_splits(const ConvShape& s, int64_t partial_floats_cap);
cudaError_t conv_wgrad(const ConvShape& s, const float* x, const float* dy, float* dw, float* db,
                       float* partial, int splits, float* red_scratch, cudaStream_t st);
// kernels one conv_wgrad issues (bias: db not null); splitk_reduce's own count
int conv_wgrad_launches(const ConvShape& s, int splits, bool bias);
int splitk_reduce_launches(int splits, int M, int N);

// TMA-fed variants (conv_tma.cu); conv_fwd/conv_dgrad/conv_wgrad dispatch to
// them when the shapes allow (C % 32 == 0; dgrad stride 1) unless SN_CONV_TMA=0.
bool conv_tma_ok_fwd(const ConvShape& s);
bool conv_tma_ok_dgrad(const ConvShape& s);
bool conv_tma_ok_wgrad(const ConvShape& s);
cudaError_t conv_fwd_tma(const ConvShape& s, const float* x, const float* w, const float* bias, float* y,
                         float* stats, cudaStream_t st);
cudaError_t conv_dgrad_tma(const ConvShape& s, const float* dy, const float* wt_flip, float* dx, int accumulate,
                           cudaStream_t st);
cudaError_t conv_wgrad_tma(const ConvShape& s, const float* x, const float* dy, float* partial, int splits,
                           cudaStream_t st);
// D = sum of split-K partials [splits][M][N] (+bias) (+D), optionally transposed.
cudaError_t splitk_reduce(const float* P, int splits, int M, int N, float* D, const float* bias, int accumulate,
                          int transpose, cudaStream_t st);

// Stem convolution over the spatially padded C=4 image buffer (conv_tma.cu).
bool conv_stem_ok(const ConvShape& s);
int64_t stem_padded_floats(const ConvShape& s);
int64_t stem_weight_floats(const ConvShape& s);
int64_t stem_wgrad_partial_floats(const ConvShape& s);
cudaError_t stem_pad_input(const ConvShape& s, int H_raw, int W_raw, int C_raw, int pad, const float* raw, float* xp,
                           cudaStream_t st);
cudaError_t conv_stem_fwd(const ConvShape& s, const float* xp, const float* w, float* wp_scratch, const float* bias,
                          float* y, float* stats, cudaStream_t st);
// The stem BN's backward fused into the stem weight gradient: instead of the
// materialised BN dx, the kernel reads the BN input x and the BN's own dy g
// and forms dx on the fly (statistics / coefficients from bn_bwd's
// statistics pass); bit-identical to running bn_bwd's dx pass first.
struct StemBnFuse {
  const float* x;      // BN input (the stem CONV's output) [N][P][Q][K]
  const float* g;      // BN output gradient [N][P][Q][K] (ReLU mask applied here when relu)
  const float* stats;  // BN mean[K], invstd[K]
  const float* gamma;
  const float* beta;
  const float* coef;   // bn_bwd's {sum g, sum g xhat} (bn_coef_ptr)
  int64_t rows;
  int relu;
  // optional: g gathered instead from a following 3x3 / s2 / p1 max pool's
  // output gradient [N][pool_P][pool_Q][K] and saved argmax (g unused; the
  // pool backward need not run; coef from bn_bwd_pool_stats)
  const float* dy_pool = nullptr;
  const uint8_t* argmax = nullptr;
  int pool_P = 0, pool_Q = 0;
};
bool conv_stem_wgrad_rows_ok(const ConvShape& s);
bool stem_pool_gather_ok(const ConvShape& s, int pool_P, int pool_Q);
cudaError_t conv_stem_wgrad(const ConvShape& s, const float* xp, const float* dy, float* partial, float* wp_scratch,
                            float* dw, float* db, float* red, cudaStream_t st, const StemBnFuse* fuse = nullptr);
// Channel-pad raw NHWC images (C_raw -> Cs) for the generic path.
cudaError_t pad_channels(const float* raw, int C_raw, float* out, int Cs, int64_t pixels, cudaStream_t st);

// Halo-tiled stride-1 convolution (conv_halo.cu): one TMA box per 32-channel
// chunk serves every filter tap.  Variant 0 = not applicable to the shape.
// stride 2: the phase-mode kernel (four strided phase boxes per chunk).
int conv_halo_variant(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, int stride = 1);
int conv_halo_stats_tiles(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, int stride = 1);
cudaError_t conv_halo(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, const float* x,
                      const float* w, const float* bias, float* y, int accumulate, float* stats, cudaStream_t st,
                      int stride = 1);
void set_conv_halo(int mode);  // 0 off, 1 by shape (default; env SN_CONV_HALO=0), 2 whenever legal (tests)
// Halo-tiled weight gradient, C, K multiples of 64 (64 x 64 sub-problems of
// M = 64 MMAs, all taps per CTA): partial = conv_halo_wgrad_splits() * R*S*C*K
// floats, dw[K][R][S][C].
bool conv_halo_wgrad_ok(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q);
int conv_halo_wgrad_splits();
// C, K multiples of 128: one filter row x 128 channels x 128 k per CTA group,
// M = N = 128 MMAs; partial = conv_halo_wgrad128_splits(C, K, R) * R*S*C*K floats.
bool conv_halo_wgrad128_ok(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q);
int conv_halo_wgrad128_splits(int C, int K, int R);
cudaError_t conv_halo_wgrad128(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q,
                               const float* x, const float* dy, float* partial, float* dw, cudaStream_t st);
cudaError_t conv_halo_wgrad(int N, int H, int W, int C, int K, int R, int S, int pad, int P, int Q, const float* x,
                            const float* dy, float* partial, float* dw, cudaStream_t st);

bool conv_tma_ok_dgrad_strided(const ConvShape& s);
// 3x3 / stride 2 / pad 1 dgrad as one sub-pixel GEMM (conv_tma.cu); wt_scratch
// must hold 16*C*K floats (conv_dgrad_scratch_floats)
bool conv_dgrad_subpix_ok(const ConvShape& s);
cudaError_t conv_dgrad_subpix_tma(const ConvShape& s, const float* dy, const float* w, float* wt_scratch, float* dx,
                                  int accumulate, cudaStream_t st, int prepped = 0);
void set_conv_subpix(int on);          // 0: phase-decomposed strided dgrad (A/B, tests)
int conv_dgrad_launches(const ConvShape& s, int prepped = 0);  // kernels one conv_dgrad issues
int64_t conv_dgrad_scratch_floats(const ConvShape& s);  // wt scratch conv_dgrad needs
cudaError_t conv_dgrad_strided_tma(const ConvShape& s, const float* dy, const float* w, float* wt_scratch, float* dx,
                                   int accumulate, cudaStream_t st);
void set_conv_tma(int on);
// Numeric mode of every CONV / FC contraction: 0 = tf32 tensor-core math (the
// TMA / halo / pair kernels), 1 = fp32-faithful 3xTF32 split operands in the
// generic gather kernel (gemm_tc.cuh).  Process-wide; the executor sets it
// around its own launches (sn_exec_options.precision).
void set_precision(int p);
int precision();
// A/B measurement hook, SN_XSKIP bitmask.  Skipping bits (results are wrong,
// and operand values change the power draw, so read step times with care):
// 1 BN-backward finaliser, 2 BN dx bias finaliser, 4 BN-backward statistics
// pass, 8 BN dx pass, 16 halo wgrad64, 32 split-K reductions, 64 weight
// transposes, 128 BN forward tile statistics.  Doubling bits (idempotent
// launches issued twice: the step-time delta is their real cost in the graph):
// 512 every BN statistics finaliser, 1024 every weight transpose.
int xskip(int bit);
// CTA-pair (cta_group::2) conv kernels: 0 off, 1 when the shape keeps the
// pairs busy (default; env SN_CONV_PAIRS=0 turns them off), 2 always (tests).
void set_conv_pairs(int mode);
void set_conv_bn(int bn);  // im2col conv tile width override (0 = policy), for A/B timing
int conv_pairs_mode();
bool use_tma();
int conv_halo_mode();
int conv_bn_force();
int conv_subpix_mode();
// The kernel-variant knobs of the CONV dispatch above, as one value (read at
// launch; the executor applies a layer's measured choice around its launches).
struct ConvKnobs {
  int halo, pairs, bn, subpix;  // set_conv_halo / set_conv_pairs / set_conv_bn / set_conv_subpix
  bool operator==(const ConvKnobs& o) const {
    return halo == o.halo && pairs == o.pairs && bn == o.bn && subpix == o.subpix;
  }
};
ConvKnobs conv_knobs();
void set_conv_knobs(const ConvKnobs& k);
struct KnobScope {
  ConvKnobs saved;
  explicit KnobScope(const ConvKnobs& k) : saved(conv_knobs()) { set_conv_knobs(k); }
  ~KnobScope() { set_conv_knobs(saved); }
};

// FC: x[B][I], w[O][I], y[B][O]
int fc_splits(int B, int I, int O, int64_t partial_floats_cap);
int fc_fwd_launches(int B, int I, int O);  // kernels one fc_fwd issues
cudaError_t fc_fwd(int B, int I, int O, const float* x, const float* w, const float* bias, float* y,
                   float* partial, int splits, cudaStream_t st);
cudaError_t fc_dgrad(int B, int I, int O, const float* dy, const float* w, float* dx, int accumulate,
                     float* partial, int splits, cudaStream_t st, float* wt_scratch = nullptr);
// fc_wgrad_splits: split count for fc_wgrad's TMA path (0: not applicable)
int fc_wgrad_splits(int B, int I, int O, int64_t partial_floats_cap);
int fc_bwd_launches(int B, int I, int O, int wsplits, bool dgrad);  // kernels fc_wgrad (+ fc_dgrad) issue
cudaError_t fc_wgrad(int B, int I, int O, const float* x, const float* dy, float* dw, float* db,
                     float* red_scratch, cudaStream_t st, float* partial = nullptr,
                     int splits = 0);

// ---- memory-bound layer kernels (layers.cu) ------------------------------------
// Per-channel column reductions over a [rows][C] matrix need a scratch of
// kRedChunks*C*2 doubles.
constexpr int kRedChunks = 592;
int64_t red_scratch_floats(int C);

cudaError_t bias_grad(const float* dy, int64_t rows, int C, float* db, float* red_scratch, cudaStream_t st);
// db[c] = sum over blocks of part[block][0][c] (fixed order; part [nblocks][2][C] doubles)
cudaError_t bias_grad_from_partials(const double* part, int nblocks, int C, float* db, cudaStream_t st);
// where bn_bwd leaves its {sum g, sum g xhat} coefficients inside red_scratch
float* bn_coef_ptr(float* red_scratch, int C);

// BatchNorm (training statistics).  stats = {mean[C], invstd[C]} saved outside
// the arena; running = {mean[C], var[C]} updated only when update_running.
cudaError_t bn_fwd(const float* x, int64_t rows, int C, const float* gamma, const float* beta, float* y,
                   float* stats, float* running, float eps, float momentum, int compute_stats,
                   float* red_scratch, cudaStream_t st);
// Statistics from the producing convolution's per-tile partials
// ({shift, sum(y - shift), sum((y - shift)^2)} per tile and channel, tile t
// holding min(tile_rows, rows - t*tile_rows) rows, or with tile_rows == 0 a
// fourth plane holding each tile's row count); x = the BN input (row 0 is the
// global shift).  Same outputs as bn_fwd(compute_stats=1, y=null).
cudaError_t bn_stats_from_tiles(const float* tiles, int ntiles, int tile_rows, const float* x, int64_t rows, int C,
                                float* stats, float* running, float eps, float momentum, float* red_scratch,
                                cudaStream_t st);
// relu = 1 fuses the backward of the ReLU consuming this BN: dy is then the
// gradient w.r.t. the ReLU output and the mask bn(x) > 0 is recomputed from x
// (bit-identical to the forward's, see bn_affine in layers.cu).
// dbias (optional; dx not null, bn_bwd_bias_ok(C)): the column sums of this
// call's dx contribution -- the bias gradient of the CONV whose output only
// this BN consumes -- computed in the dx pass (saves that CONV's bias pass).
bool bn_bwd_bias_ok(int C);
cudaError_t bn_bwd(const float* x, const float* dy, int64_t rows, int C, const float* gamma, const float* beta,
                   const float* stats, int relu, float* dx, int accumulate, float* dgamma, float* dbeta,
                   float* red_scratch, cudaStream_t st, float* dbias = nullptr, float* copy_dst = nullptr,
                   int copy_acc = 0, float* copy2 = nullptr);
// Statistics pass of bn_bwd (dgamma, dbeta, and the coefficients at
// bn_coef_ptr) for a BN whose [ReLU'd] output feeds a 3x3 / s2 / p1 max pool
// with saved argmax, in 2 x 2 pixel-block order: dy gathered from the pool
// output's gradient and argmax (dy_mat null: the pool backward need not run)
// or read from the materialised pool-input gradient dy_mat -- same bits.
struct PoolShape;
// bn_bwd's dx pass alone, from coefficients a statistics pass left at bn_coef_ptr
cudaError_t bn_bwd_dx(const float* x, const float* dy, int64_t rows, int C, const float* gamma, const float* beta,
                      const float* stats, int relu, float* dx, int accumulate, float* red_scratch, cudaStream_t st,
                      float* dbias = nullptr);
bool pool_bn_stats_ok(const PoolShape& ps, int bn_C);
cudaError_t bn_bwd_pool_stats(const PoolShape& ps, const uint8_t* argmax, const float* dy_pool, const float* dy_mat,
                              const float* x, int C, const float* gamma, const float* beta, const float* stats,
                              int relu, float* dgamma, float* dbeta, float* red_scratch, cudaStream_t st);
// copy2 (optional, C % 4 == 0): the statistics pass also writes dy there and
// the dx pass reads dy from it (dx may then overlap the original dy).
// copy_dst (optional, C % 4 == 0): the fused backward of the 2-input JOIN
// feeding the ReLU: its gradient dy is also written (copy_acc: added) into the
// JOIN's other input's gradient buffer in the reduction pass.

// Fused BN apply + ReLU (+ 2-input JOIN) (C % 4 == 0): y = bn(x), y_relu =
// max(bn(x), 0), y_join = y_relu + join_other; null outputs are not written.
cudaError_t bn_apply_relu(const float* x, int64_t rows, int C, const float* gamma, const float* beta,
                          const float* stats, float* y, float* y_relu, cudaStream_t st,
                          const float* join_other = nullptr, float* y_join = nullptr);
// JOIN backward into two gradient buffers with one read of dy (n % 4 == 0).
cudaError_t grad_copy2(const float* src, float* d1, int acc1, float* d2, int acc2, int64_t n, cudaStream_t st);

cudaError_t relu_fwd(const float* x, float* y, int64_t n, cudaStream_t st);
cudaError_t relu_bwd_inplace(const float* y, float* g, int64_t n, cudaStream_t st);
// dx (+)= (y > 0) * dy: the backward of an ACT with its own gradient buffer
// (its producer forks; see the executor's side roots)
cudaError_t relu_bwd_to(const float* y, const float* dy, float* dx, int64_t n, int accumulate, cudaStream_t st);

struct PoolShape {
  int N, H, W, C, P, Q, K, stride, pad, mode;  // mode 0 max, 1 avg
};
// argmax (optional, pool_saves_argmax(s)): the forward also records, per output
// element, the first window position holding the maximum (one byte); the
// backward then gathers with it instead of re-deriving it from x and y.
bool pool_saves_argmax(const PoolShape& s);
cudaError_t pool_fwd(const PoolShape& s, const float* x, float* y, cudaStream_t st, uint8_t* argmax = nullptr);
// Max-pool backward recomputes each window's first argmax from x and y (the
// reference's backward reads) into a byte per output (executor scratch of
// pool_scratch_bytes), then gathers; avg-pool gathers directly.
int64_t pool_scratch_bytes(const PoolShape& s);
int pool_bwd_kernels(const PoolShape& s);  // launches one pool_bwd issues
// pool_bwd with a saved argmax reads neither x nor y (the gather kernel path)
bool pool_bwd_argmax_only(const PoolShape& s);
// BN (batch statistics) + ReLU + max pool in one pass over the BN input x:
// y = pool(relu(bn(x))), the argmax saved as pool_fwd does, the ReLU output
// written to y_relu when not null (pool_fwd_bn_relu_ok: k3 s2 pad 1, even
// input, C <= 512).
bool pool_fwd_bn_relu_ok(const PoolShape& s);
cudaError_t pool_fwd_bn_relu(const PoolShape& s, const float* x, const float* gamma, const float* beta,
                             const float* stats, float* y_relu, float* y, uint8_t* argmax, cudaStream_t st);
cudaError_t pool_bwd(const PoolShape& s, const float* x, const float* y, const float* dy, float* dx,
                     int accumulate, void* scratch, cudaStream_t st, const uint8_t* argmax = nullptr);

cudaError_t lrn_fwd(const float* x, float* y, int64_t pixels, int C, int size, float alpha, float beta,
                    float k, cudaStream_t st);
cudaError_t lrn_bwd(const float* x, const float* y, const float* dy, float* dx, int64_t pixels, int C,
                    int size, float alpha, float beta, float k, int accumulate, cudaStream_t st);

// Dropout: mask bit = hash(seed, layer, *iteration, index) >= rate * 2^32.
cudaError_t dropout_fwd(const float* x, float* y, int64_t n, float rate, uint64_t seed, int layer,
                        const uint32_t* iteration, cudaStream_t st);
cudaError_t dropout_bwd_inplace(float* g, int64_t n, float rate, uint64_t seed, int layer,
                                const uint32_t* iteration, cudaStream_t st);
cudaError_t dropout_bwd_to(const float* dy, float* dx, int64_t n, float rate, uint64_t seed, int layer,
                           const uint32_t* iteration, int accumulate, cudaStream_t st);

// Softmax over F features per row + cross entropy vs labels; loss_rows[B].
cudaError_t softmax_fwd(const float* x, float* y, int B, int F, const int32_t* labels, float* loss_rows,
                        cudaStream_t st);
cudaError_t softmax_ce_bwd(const float* y, const int32_t* labels, float* dx, int B, int F, int accumulate,
                           cudaStream_t st);
cudaError_t loss_reduce(const float* loss_rows, int B, float* loss, cudaStream_t st);

// y = sum_i inputs[i] (device array of n_in pointers), n elements.
cudaError_t join_fwd(const float* const* inputs, int n_in, float* y, int64_t n, cudaStream_t st);
// dst (+)= src
cudaError_t grad_copy(const float* src, float* dst, int64_t n, int accumulate, cudaStream_t st);
// k-way JOIN backward in ceil(k/8) passes over dy (n % 4 == 0; destinations distinct)
int grad_copy_multi_launches(int k);
cudaError_t grad_copy_multi(const float* src, float* const* dsts, const int* accs, int k, int64_t n, cudaStream_t st);
// Dense JOIN-chain backward step: r = (acc_r ? r + src : src), then dsts[t] =
// (accs[t] ? dsts[t] + r : r).  Bit-identical to adding src into every buffer
// one JOIN at a time (same additions, same order).
int grad_prefix_launches(int k);
cudaError_t grad_prefix(const float* src, float* r, int acc_r, float* const* dsts, const int* accs, int k, int64_t n,
                        cudaStream_t st);

cudaError_t sgd_update(float* params, const float* grads, int64_t n, float lr, float grad_scale,
                       cudaStream_t st);
// Same update, skipped on the device when *flag == 0 (graph-captured DP buckets).
cudaError_t sgd_update_flagged(float* params, const float* grads, int64_t n, float lr, float grad_scale,
                               const int* flag, cudaStream_t st);
cudaError_t bump_iteration(uint32_t* iteration, cudaStream_t st);
cudaError_t fill_zero(float* p, int64_t n, cudaStream_t st);

}  // namespace sn
