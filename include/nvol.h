/*
 * nvol.h — C ABI of libnvol.so, the B200 (sm_100a) implementation of the
 * hash-grid encoder + ReLU MLP training step, full-grid decode and macro-cell
 * ray marching of the arXiv 2207.11620 CPU reference
 * (/root/reference/pkg/src/neuralvol).
 *
 * Every entry point replaces one numba kernel (or one numpy step) of the
 * reference; the reference symbol is cited beside each declaration.  The
 * reference's "FFI" is numba's: caller-allocated arrays, no return value.  Here
 * every function takes plain device pointers + sizes, returns an int status
 * and runs asynchronously on the caller's stream:
 *
 *   NVOL_OK (0)            enqueued
 *   NVOL_EINVAL (1)        bad argument        -> ConfigError (errors.py:9-10)
 *   NVOL_ECUDA (2)         CUDA launch failure -> RuntimeError
 *
 * nvol_last_error() returns a static description of the last failure.
 *
 * Ownership: the caller owns every buffer (PyTorch allocates them); the
 * library allocates nothing except transient tensor memory (TMEM) inside
 * kernels.  Pointers are device pointers unless marked [host].  `stream` is a
 * cudaStream_t (0 = legacy default stream).  Calls are re-entrant per stream.
 *
 * Layouts (all little-endian, row-major, matching the reference):
 *   coords      f32/f64 [B,3] in [0,1)^3, x fastest              (sampler.py:33-38)
 *   params      encoder table, level-major / entry-major / feature-minor
 *               (encoding.py:145-169), followed in the flat training
 *               buffer by each W_i (out x in) row-major             (trainer.py:114-123)
 *   level_*     the four per-level arrays of GridEncoder.kernel_tables()
 *               (encoding.py:174-177) [host]
 *   volume      normalised f32 [Dz,Dy,Dx], x fastest                (volume.py:99-107)
 */
#ifndef NVOL_H
#define NVOL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NVOL_OK 0
#define NVOL_EINVAL 1
#define NVOL_ECUDA 2
#define NVOL_MAX_LEVELS 32

/* ------------------------------------------------------------------ library */

/* ABI version (bumped on any signature change; 2: the nvol_render camera parameter array gained
 * the image tile rows row0, nrows; 3: nvol_render path tracing block + 3 stats; 4: the training
 * pipeline's NaN state (nvol_train_fwd_bwd / nvol_adam_train_step / nvol_adam_encode_step). */
int nvol_abi_version(void);
/* Static string describing the last non-zero status (thread-local). */
const char *nvol_last_error(void);
/* 1 when the tcgen05 tensor-core MLP is compiled in and usable on `device`. */
int nvol_has_tcgen05(int device);

/* Ordered-reduction mode (SPEC bitwise-repeatability criterion): on != 0 makes
 * every reduction of the fp32 SIMT training engine (nvol_train_fwd_bwd mode 0:
 * split-K dW GEMMs, the loss sum, the encoder scatter) run in a fixed order,
 * so training is bitwise repeatable run to run.  Library-wide; default off. */
int nvol_set_deterministic(int32_t on);

/* ------------------------------------------------------------------ encoder */

/* _kernels.py:31-79 grid_encode_fwd (called from model.py:136-150).
 * dtype_bytes = 4 (f32 coords/params/out/w_cache) or 8 (f64 path of
 * encoding.py:203-213, used for gradient checks).  idx_cache (i64 [B,m,8],
 * flat element offset of each corner row) and w_cache ([B,m,8]) may be NULL.
 * Float32 results are bit-identical to the reference. */
int nvol_grid_encode_fwd(const void *coords, int64_t b, const void *params,
                         const int64_t *level_off, const int64_t *level_res,
                         const int64_t *level_entries, const uint8_t *level_dense,
                         int32_t n_levels, int32_t n_feat, int64_t *idx_cache, void *w_cache,
                         void *out, int32_t dtype_bytes, void *stream);

/* _kernels.py:82-92 grid_encode_bwd: grad_out[idx+f] += w * dl_dfeat[i, l*n+f]
 * (accumulating).  Float atomics: order-dependent in the last ulp. */
int nvol_grid_encode_bwd(const void *dl_dfeat, const int64_t *idx_cache, const void *w_cache,
                         int64_t b, int32_t n_levels, int32_t n_feat, void *grad_out,
                         int32_t dtype_bytes, void *stream);

/* encoding.py:215-226 encode_backward, recomputing corners from coords
 * (no caches).  deterministic != 0 reproduces the reference's serial scatter
 * order exactly (float32 only): bit-identical to _kernels.grid_encode_bwd. */
int nvol_grid_encode_bwd_coords(const void *coords, const void *dl_dfeat, int64_t b,
                                const int64_t *level_off, const int64_t *level_res,
                                const int64_t *level_entries, const uint8_t *level_dense,
                                int32_t n_levels, int32_t n_feat, void *grad_out,
                                int32_t dtype_bytes, int32_t deterministic, void *stream);

/* ------------------------------------------------------------------ MLP, loss, optimizer */

/* network.py:61-74 Mlp.forward.  weights[i] -> W_i (widths[i+1] x widths[i]);
 * acts[i] -> activation buffer i ([B, widths[i]]); acts[0] is the input and
 * acts[n_layers] the output.  [host] arrays of device pointers. */
int nvol_mlp_forward(int64_t b, int32_t n_layers, const int32_t *widths, const void *const *weights,
                     void *const *acts, int32_t relu_out, int32_t dtype_bytes, void *stream);

/* network.py:76-93 Mlp.backward.  dl_dout [B] (output width 1); grads[i] are
 * accumulated; dl_dinput [B, widths[0]]; scratch: two buffers of
 * B x max(widths) elements. */
int nvol_mlp_backward(int64_t b, int32_t n_layers, const int32_t *widths, const void *const *weights,
                      const void *const *acts, const void *dl_dout, void *const *grads,
                      void *dl_dinput, void *scratch0, void *scratch1, int32_t relu_out,
                      int32_t dtype_bytes, void *stream);

/* network.py:96-114 loss_and_grad.  kind 0 = L1, 1 = L2.  Differences in
 * f64; grad written in the pred dtype; *loss_sum (f64, device) receives the
 * sum of |d| (L1) or d^2 (L2) — accumulated, caller zeroes. */
int nvol_loss_and_grad(const void *pred, const void *target, int64_t b, int32_t kind,
                       void *grad, double *loss_sum, int32_t dtype_bytes, void *stream);

/* Same, with the gradient divided by b_global instead of b (data-parallel
 * shard of a global batch: network.py:108 grad = sign(d) / B_global). */
int nvol_loss_and_grad_scaled(const void *pred, const void *target, int64_t b, int64_t b_global,
                              int32_t kind, void *grad, double *loss_sum, int32_t dtype_bytes,
                              void *stream);

/* trainer.py:61-77 history bookkeeping on the device: losses[*step_counter - t0]
 * = *acc * inv_b, then *acc = 0 (CUDA-graph friendly). */
int nvol_loss_record(double *acc, double *losses, const int64_t *step_counter, int64_t t0,
                     int64_t cap, double inv_b, void *stream);

/* network.py:160-183 adam_step on one flat group; scalars are the
 * dtype-cast values the reference computes on the host (lr_at, c1, c2 ...).
 * Bit-identical to the reference; zeroes g. */
int nvol_adam_step(void *p, void *g, void *m, void *v, int64_t n, double lr, double beta1,
                   double one_minus_beta1, double beta2, double one_minus_beta2, double c1,
                   double c2, double eps, double l2, int32_t dtype_bytes, void *stream);

/* network.py:167-171: index of the first NaN in g (or -1), written to *first. */
int nvol_find_nan(const void *g, int64_t n, int64_t *first, int32_t dtype_bytes, void *stream);

/* ------------------------------------------------------------------ sampling, volumes, metrics */

/* sampler.py:54-74 sample_incore with the reference's numpy PCG64 stream:
 * coords are float32 draws u32_offset .. u32_offset+3B of default_rng(seed)
 * (initial (state, inc) passed as four u64 words); targets are the clamped
 * cell-centred trilinear reads of volume.py:148-164.  Bit-identical. */
int nvol_sample_incore(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                       uint64_t u32_offset, int64_t b, const float *volume, int64_t dx,
                       int64_t dy, int64_t dz, float *coords, float *targets, void *stream);

/* Same stream, step counter read from device memory (CUDA-graph friendly):
 * u32 offset = u32_base + (*step_counter - counter0) * 3 * b_global + 3 * row0
 * (rows [row0, row0+b) of a global batch of b_global: the data-parallel shard
 * of one rank reproduces exactly those rows of the single-process batch). */
/* sampler.py:224-253 BlockBuffer.sample (out-of-core, SURVEY 8 f item 2): the
 * caller draws slots (int32 [b], rng.integers(0, R)), voxel fractions u and raw
 * jitter (f32 [b,3] each, rng.random(float32)) with the reference's generator;
 * coordinates and the payload-local trilinear (nearest != 0: nearest) targets
 * are computed here, bit-exact.  origins / interiors int64 [R,3], payloads f32
 * [R][pz][py][px] with a one-voxel ghost border; all device pointers. */
int nvol_sample_outofcore(const int32_t *slots, const float *u, const float *jitter, int64_t b,
                          const int64_t *origins, const int64_t *interiors, const float *payloads, int64_t px,
                          int64_t py, int64_t pz, int64_t dx, int64_t dy, int64_t dz, int32_t nearest,
                          float *coords, float *targets, void *stream);

int nvol_sample_incore_dev(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                           uint64_t u32_base, const int64_t *step_counter, int64_t counter0, int64_t b_global,
                           int64_t row0, int64_t b,
                           const float *volume, int64_t dx, int64_t dy, int64_t dz, float *coords,
                           float *targets, void *stream);

/* nvol_sample_incore_dev with the online macro-cell update fused in
 * (macrocell.py:101-133 macrocell_update_online on each sampled row, as the
 * reference's live session does per training step, service.py:279): every
 * row's target widens value_lo / value_hi [gz][gy][gx] (cells of n_g voxels)
 * with exact int-ordered atomics.  mc_lo = NULL disables the update. */
int nvol_sample_incore_dev_mc(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                              uint64_t u32_base, const int64_t *step_counter, int64_t counter0,
                              int64_t b_global, int64_t row0, int64_t b, const float *volume, int64_t dx,
                              int64_t dy, int64_t dz, float *coords, float *targets, float *mc_lo, float *mc_hi,
                              int64_t gx, int64_t gy, int64_t gz, int64_t n_g, void *stream);

/* macrocell.py:101-133 macrocell_update_online for a batch already on the device
 * (coords f32 [n,3], targets f32 [n] in [0,1]); bit-exact with the reference. */
int nvol_macrocell_update_online(const float *coords, const float *targets, int64_t n, int64_t dx, int64_t dy,
                                 int64_t dz, float *lo, float *hi, int64_t gx, int64_t gy, int64_t gz,
                                 int64_t n_g, void *stream);

/* volume.py:167-171 sample_trilinear_many (no clamp). */
int nvol_trilinear(const float *volume, int64_t dx, int64_t dy, int64_t dz, const float *pts,
                   int64_t n, float *out, void *stream);

/* fields.py:67-88 rasterize: field 0 gauss, 1 blobs, 2 waves, 3 mlobb, f64
 * evaluation at voxel centres, clipped, stored as f32 (out_u8 = 0) or as
 * round(v*255) u8 (out_u8 = 1); rows [z0, z0+nz). */
int nvol_rasterize(int32_t field, int64_t dx, int64_t dy, int64_t dz, int64_t z0, int64_t nz,
                   void *out, int32_t out_u8, void *stream);

/* volume.py:197-207 mse numerator: *sum += sum((a-b)^2) over n normalised
 * values, f64 accumulation. */
int nvol_sq_err_sum(const float *a, const float *b, int64_t n, double *sum, void *stream);

/* ------------------------------------------------------------------ fused field evaluation / decode */

/* _kernels.py:154-176 field_eval_model == NeuralModel.eval_fused
 * (model.py:184-198): per-sample encode + serial float32 matvec chain,
 * bit-identical to the reference.  weights: flat concatenation of W_i. */
int nvol_field_eval_exact(const float *coords, int64_t b, const float *params,
                          const int64_t *level_off, const int64_t *level_res,
                          const int64_t *level_entries, const uint8_t *level_dense,
                          int32_t n_levels, int32_t n_feat, const float *weights,
                          const int32_t *widths, int32_t n_layers, int32_t relu_out,
                          float *out, void *stream);

/* Same evaluation on the tensor cores (tcgen05, fp16 operands / fp32
 * accumulate; north-star half-precision bar): the batched Phi evaluator of
 * the renderers (_render_kernels.py:518-540 phi_eval_staged). */
int nvol_field_eval_tc(const float *coords, int64_t b, const float *params,
                       const int64_t *level_off, const int64_t *level_res,
                       const int64_t *level_entries, const uint8_t *level_dense, int32_t n_levels,
                       int32_t n_feat, const float *weights, const int32_t *widths,
                       int32_t n_layers, int32_t relu_out, void *mlp_image, float *out,
                       void *stream);

/* Bytes of the device scratch `mlp_image` the tensor-core evaluators pack the
 * fp32 weights into (fp16 UMMA core-matrix tiles + fp32 output row). */
int64_t nvol_mlp_image_bytes(int32_t n_levels, int32_t n_feat, int32_t n_neurons, int32_t n_hidden);

/* trainer.py:80-106 decode_slabs over voxel-centre coordinates of the brick
 * [z0, z0+nz) of a (dx,dy,dz) grid: out[k] = Phi * (hi-lo) + lo (f64 then f32).
 * mode 0 = exact (serial fp32, == eval_fused), 1 = tensor-core (tcgen05,
 * fp16 operands / fp32 accumulate). */
int nvol_decode(const float *params, const int64_t *level_off, const int64_t *level_res,
                const int64_t *level_entries, const uint8_t *level_dense, int32_t n_levels,
                int32_t n_feat, const float *weights, const int32_t *widths, int32_t n_layers,
                int32_t relu_out, int64_t dx, int64_t dy, int64_t dz, int64_t z0, int64_t nz,
                double lo, double hi, float *out, int32_t mode, void *mlp_image, void *stream);

/* ------------------------------------------------------------------ fused training step */

/* One NeuralModel.train_step (model.py:154-174) as a device-resident pipeline
 * over a flat parameter buffer [enc | pad | W_0 | W_1 ... ] (and equally
 * laid-out grad, m, v buffers), where W_0 starts at the encoder parameter
 * count rounded up to a multiple of 4 floats (16-byte aligned):  encode -> MLP -> loss -> backprop -> encoder scatter.  The
 * Adam update is a separate call (nvol_adam_step over the flat buffer) so a
 * data-parallel caller can all-reduce `grads` in between.
 * coords/targets: [b] rows of this rank; grad_scale = 1/B_global (L1 sign
 * gradient, network.py:108).  loss_sum (f64) accumulates sum |pred-target|.
 * mode 0 = SIMT fp32, 1 = tcgen05 (fp16 operands, fp32 accumulate), optionally
 * or-ed with NVOL_TRAIN_PREENCODED / NVOL_TRAIN_ENCODE_ONLY (below).
 * nan_state (nullable): NaN detection + halt, see "NaN contract" below. */
int nvol_train_fwd_bwd(const float *coords, const float *targets, int64_t b, int64_t b_global,
                       const float *params, float *grads, const int64_t *level_off,
                       const int64_t *level_res, const int64_t *level_entries,
                       const uint8_t *level_dense, int32_t n_levels, int32_t n_feat,
                       int32_t n_neurons, int32_t n_hidden, int32_t relu_out, int32_t loss_kind,
                       double *loss_sum, void *workspace, int64_t workspace_bytes, int32_t mode,
                       int64_t *nan_state, void *stream);

/* Profiling hook (bench.py): with n >= 4 cudaEvent_t handles set,
 * nvol_train_fwd_bwd mode 1 runs unchunked on the caller's stream and records
 * events[0..3] before encode / after encode / after MLP / after scatter, so
 * each stage kernel is timed with CUDA events on its launching stream.
 * n = 0 disables.  [host] array of event handles. */
int nvol_set_stage_events(void *const *events, int32_t n);

/* Pipeline hook (trainer.StepPipeline): while set, nvol_train_fwd_bwd mode 1
 * records this cudaEvent_t right after the step's encoder launch (before the
 * MLP), so the caller forks the next step's sampling there -- it then runs
 * beside the latency-bound MLP instead of the L2-bound encoder.  NULL disables.
 * No reference counterpart (trainer.py:61-77 samples serially). */
int nvol_set_fork_event(void *event);

/* Data-parallel exchange over peer memory (distributed.PeerExchange; NVOL_DP_PEER=1): the sharded
 * optimizer's reduce-scatter -> Adam on this rank's slice -> all-gather as ONE kernel per rank that
 * reads / writes the other ranks' flat buffers through their CUDA-IPC (NVLink P2P) mappings.
 * Replaces dist.reduce_scatter + adam_step (network.py:160-183) + dist.all_gather of the NCCL
 * path; the step's loss is the rank-ordered sum of the ranks' loss sums and the NaN limit their
 * minimum.  Arrays of `world` device addresses (host int64): flat gradients, flat parameters,
 * loss sums (double), NaN states (int64[2]) and step flags (int64[2]: ready, done) of every rank;
 * [lo, hi) is this rank's slice of the flat buffer, m / v its own moment buffers.
 *   nvol_dp_signal: own ready flag = step + 1 (after this rank's scatter);
 *   nvol_dp_wait:   before a step, every rank's done flag >= step; zeroes the own loss sum. */
int nvol_dp_signal(int64_t *own_flags, const int64_t *step_counter, const int64_t *nan_state, void *stream);
int nvol_dp_wait(int32_t world, const int64_t *flags, const int64_t *step_counter, double *own_loss_acc,
                 const int64_t *nan_state, void *stream);
int nvol_dp_fused_adam(int32_t world, int32_t rank, const int64_t *grads, const int64_t *params,
                       const int64_t *loss_accs, const int64_t *nan_states, const int64_t *flags, int64_t lo,
                       int64_t hi, float *m, float *v, const float *sched, int64_t sched_len,
                       int64_t *step_counter, float beta1, float one_minus_beta1, float beta2,
                       float one_minus_beta2, float eps, float l2, int64_t *nan_state, double *losses,
                       int64_t t0, int64_t cap, double inv_b, uint32_t *ticket, void *stream);

/* Parity hooks for the tcgen05 training engine (tests only; all null in
 * production).  While set, nvol_train_fwd_bwd mode 1 additionally writes
 * feat  [b][n_levels*n_feat] f32: the hot encoder's fp32 features
 *       (encode_tiles_kernel, before the fp16 split; reference
 *       _kernels.py:31-79 grid_encode_fwd `out`),
 * pred  [b] f32: the per-sample MLP output of mlp_tc_kernel
 *       (network.py:61-74 Mlp.forward),
 * dfeat [n_levels*n_feat][b] f32: the feature-major dL/dfeat the MLP hands to
 *       the scatter (network.py:76-93 Mlp.backward return value). */
int nvol_train_tc_debug(float *feat, float *pred, float *dfeat);

/* The tcgen05 engine's encoder-backward kernel on its own (the launch
 * nvol_train_fwd_bwd mode 1 makes after the MLP), fed a caller-provided
 * feature-major dL/dfeat [n_levels*n_feat][stride]; accumulates into grads
 * (the flat buffer's encoder region).  Replaces grid_encode_bwd
 * (_kernels.py:82-92) with the corners recomputed from coords. */
int nvol_train_tc_scatter(const float *coords, const float *dfeat, int64_t b, int64_t stride,
                          const int64_t *level_off, const int64_t *level_res,
                          const int64_t *level_entries, const uint8_t *level_dense,
                          int32_t n_levels, int32_t n_feat, float *grads, void *stream);

/* L2 set-aside for persisting lines (cudaLimitPersistingL2CacheSize): the
 * training step keeps its flat gradient L2-resident between Adam and the
 * encoder-backward scatter (evict_last policies).  Requests `bytes`, clamped
 * to the device maximum; returns the bytes set (>= 0) or -1 on error.
 * Device-wide setting.  No reference counterpart (GPU residency control). */
int64_t nvol_l2_persist(int64_t bytes);

/* Diagnostic: L2 peaks for the L2-bound kernels' rooflines.  out[0] = streaming
 * read GB/s of an L2-resident 48 MB buffer, out[1] = random 8-byte gathers G/s,
 * out[2] = random float2 REDs G/s.  Synchronous; allocates 48 MB transiently.
 * No reference counterpart (measurement). */
int nvol_l2_probe(double *out);

/* 1 if the tcgen05 training engine (nvol_train_fwd_bwd mode 1) takes this
 * grid / MLP shape (n_neurons in {16, 32, 64}, 1..8 hidden layers, encoder
 * width <= 2 * n_neurons, shared-memory and TMEM budgets), else 0. */
int nvol_train_tc_supported(int32_t n_levels, int32_t n_feat, int32_t n_neurons, int32_t n_hidden);

/* Workspace bytes nvol_train_fwd_bwd needs for batch b. */
int64_t nvol_train_workspace_bytes(int64_t b, int32_t n_levels, int32_t n_feat, int32_t n_neurons,
                                   int32_t n_hidden, int32_t mode);

/* Flat-buffer Adam step reading the step counter from device memory (for
 * CUDA-graph replay) and a per-step scalar table sched[t] = {lr, c1, c2} as
 * f32 cast on the host exactly like network.py:163-181; increments
 * *step_counter.  nan_flag (u32, nullable) is set when any g is NaN. */
int nvol_adam_flat_dev(float *p, float *g, float *m, float *v, int64_t n, const float *sched,
                       int64_t sched_len, int64_t *step_counter, float beta1, float one_minus_beta1,
                       float beta2, float one_minus_beta2, float eps, float l2, uint32_t *nan_flag,
                       void *stream);

/* The training pipeline's step tail in one launch: nvol_adam_flat_dev's
 * update, then (last block to finish, via the zero-initialised u32 *ticket)
 * losses[*step_counter - t0] = *loss_acc * inv_b (if 0 <= index < cap),
 * *loss_acc = 0 and ++*step_counter — i.e. nvol_loss_record + Adam + counter
 * advance of trainer.py:61-77 / network.py:160-183 without extra launches.
 * nan_state (nullable): the pipeline's NaN state, see "NaN contract" below. */
int nvol_adam_train_step(float *p, float *g, float *m, float *v, int64_t n, const float *sched,
                         int64_t sched_len, int64_t *step_counter, float beta1, float one_minus_beta1,
                         float beta2, float one_minus_beta2, float eps, float l2, int64_t *nan_state,
                         double *loss_acc, double *losses, int64_t t0, int64_t cap, double inv_b,
                         uint32_t *ticket, void *stream);

/* NaN contract of the training pipeline (network.py:160-183 adam_step checks
 * every parameter group for a NaN gradient BEFORE updating it and raises
 * FloatingPointError(group, flat index) without advancing t).  nan_state is a
 * device int64[2], initialised to {INT64_MAX, 0}:
 *   [0] the flat index where the first parameter group holding a NaN gradient
 *       starts (INT64_MAX: none).  Set by the tcgen05 MLP kernel (NaN in
 *       dL/dfeat -> encoder group 0; NaN in dW_j -> W_j's start) or by
 *       nvol_nan_scan (SIMT engine); lowered by nvol_adam_train_step for a NaN
 *       it meets itself.
 *   [1] halted.  nvol_adam_train_step updates only q < [0] (the groups in front
 *       of the offending one, as the reference) and, when [0] is set, halts
 *       instead of recording the loss and advancing the step counter; the
 *       training kernels (encode / MLP / scatter / Adam) of a halted pipeline
 *       return at entry.  The host raises FloatingPointError with the group
 *       and the first NaN's flat index (nvol_find_nan over that group). */
int nvol_nan_scan(const float *g, int64_t n, const int64_t *group_starts, int32_t n_groups,
                  int64_t *nan_state, void *stream);

/* nvol_train_fwd_bwd mode flags (tcgen05 engine, mode 1 only). */
#define NVOL_TRAIN_PREENCODED 16  /* the workspace's tile buffer already holds this batch's encoding */
#define NVOL_TRAIN_ENCODE_ONLY 32 /* run the encoder forward into the tile buffer and stop */

/* nvol_adam_train_step fused with the NEXT step's encoder forward: one
 * persistent launch whose CTAs split into an Adam sweep over the flat buffers
 * (table order) and the encoding of next_coords [b,3] into the tcgen05 tile
 * buffer of `workspace` (the nvol_train_fwd_bwd mode-1 workspace for batch b);
 * level l is encoded as soon as the sweep has updated level l's table.  The
 * next nvol_train_fwd_bwd then runs with mode 1 | NVOL_TRAIN_PREENCODED.
 * work: zero-initialised u32[2 + NVOL_MAX_LEVELS], re-armed by the kernel.
 * Same results as nvol_adam_train_step followed by the encode of next_coords
 * with the updated parameters (trainer.py:61-77, network.py:160-183,
 * _kernels.py:31-79). */
int nvol_adam_encode_step(float *p, float *g, float *m, float *v, int64_t n, const float *sched,
                          int64_t sched_len, int64_t *step_counter, float beta1, float one_minus_beta1,
                          float beta2, float one_minus_beta2, float eps, float l2, int64_t *nan_state,
                          double *loss_acc, double *losses, int64_t t0, int64_t cap, double inv_b,
                          uint32_t *work, const float *next_coords, int64_t b, const int64_t *level_off,
                          const int64_t *level_res, const int64_t *level_entries,
                          const uint8_t *level_dense, int32_t n_levels, int32_t n_feat, int32_t n_neurons,
                          int32_t n_hidden, void *workspace, int64_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------ rendering */

/* Workspace bytes nvol_render needs for an image of n_pixels and batch K. */
int64_t nvol_render_workspace_bytes(int64_t n_pixels, int32_t k_batch);

/* One frame of the ray marcher: camera.py:117-143 pixel rays, render.py:225-243
 * slab test + compaction, then either the sample-streaming wavefront loop
 * (architecture 0 = render_wavefront, render.py:383-454: rm_coord ->
 * batched Phi (eval_mode 0 exact / 1 tcgen05) -> rm_shade -> compaction) or
 * the in-shader mega-kernel (architecture 1 = render_reference,
 * render.py:347-380).  [host] cam_params[18] = eye[3], fwd[3], right[3],
 * up[3] (camera.py:44-56 basis, float64), tan_half, aspect, width, height,
 * row0, nrows (the image tile rendered: rows [row0, row0+nrows) of the frame;
 * multi-GPU renders give each rank a tile);
 * [host] render_params[29] = mode_shadow, use_mc, skip_empty, k_batch, s1,
 * s2, pexp, termination, ambient, density_scale, n_g, -light[3],
 * background[3], Dx, Dy, Dz, then path tracing (mode "pathtrace",
 * _render_kernels.py:566-878: delta tracking, NEE, Russian roulette):
 * pathtrace, seed low 32 bits, seed high 32 bits, frame, rr_depth,
 * light radiance[3], global majorant (f32-rounded).  TF tables as TransferFunction.tables
 * (transfer.py:43-47) [host].  mu: device macro-cell majorants (gz,gy,gx)
 * (a 1x1x1 dummy without macro-cells).  Field: a dense normalised grid
 * (use_grid) or the hash-grid model (tables [host], params/weights device).
 * img: device (nrows*W*3) float32.  stats_out [host]: {field evaluations,
 * iterations, majorant violations}; alive_hist [host]: rays alive per iteration (up to max_hist). */
int nvol_render(const double *cam_params, const double *render_params, const float *tf_cv,
                const float *tf_crgb, int32_t ncv, const float *tf_ov, const float *tf_oa,
                int32_t nov, const float *mu, int64_t gx, int64_t gy, int64_t gz, int32_t use_grid,
                const float *norm, int64_t ndx, int64_t ndy, int64_t ndz, const float *params,
                const int64_t *level_off, const int64_t *level_res, const int64_t *level_entries,
                const uint8_t *level_dense, int32_t n_levels, int32_t n_feat, const float *weights,
                const int32_t *widths, int32_t n_layers, int32_t relu_out, int32_t architecture,
                int32_t eval_mode, void *mlp_image, float *img, void *workspace,
                int64_t workspace_bytes, int64_t *stats_out, int32_t *alive_hist, int32_t max_hist,
                void *stream);

/* macrocell.py:63-76 _ranges_from_array: bordered per-cell min/max of a
 * (dz,dy,dx) float32 array (clip != 0: values clipped to [0,1] first, as
 * macrocell_from_model does). */
int nvol_macrocell_ranges(const float *vals, int64_t dx, int64_t dy, int64_t dz, int64_t ng,
                          int32_t clip, float *lo, float *hi, void *stream);

/* tracking.py adaptive_step / correct_opacity: the marcher's own device formulas over n
 * inputs x.  which 0: adaptive step, x = majorant mu, (a, b, c) = (s1, s2, p)
 * (_render_kernels.py:244-253); which 1: opacity correction 1 - (1 - x)^(a / b), a = s-bar,
 * b = s1 (_render_kernels.py:364-392).  Device arrays. */
int nvol_march_formula(int32_t which, const float *x, int64_t n, float a, float b, float c, float *out,
                       void *stream);

/* rng.py RngStream.uniform / _render_kernels.py:26-49 _u01: the path tracer's counter
 * stream (SplitMix64-style avalanche of (seed, frame, pixel, event), 24-bit float32 in
 * [0, 1)) for n keys: out[i] = u01(seed, frame, pixel[i], event[i]).  Device arrays. */
int nvol_rng_u01(uint64_t seed, uint64_t frame, const int64_t *pixel, const int64_t *event, int64_t n,
                 float *out, void *stream);

/* macrocell.py:159-181 dda_traverse (_render_kernels.py:153-188 dda_collect): the macro-cell
 * cells a float64 ray [host] ray = {ox, oy, oz, dx, dy, dz} walks over [t0, t1] with cell size
 * ng on a gx x gy x gz grid: cells (cap x 3, int64) and (s_enter, s_exit) pairs (cap x 2,
 * float64), *count records; zero-length grazes dropped.  Device outputs. */
int nvol_dda_collect(const double *ray, double t0, double t1, double ng, int64_t gx, int64_t gy,
                     int64_t gz, int64_t cap, int64_t *cells, double *ts, int64_t *count, void *stream);

/* macrocell.py:136-156 macrocell_set_tf: mu = max TF opacity over [lo,hi]
 * (np.interp semantics, float64) * density_scale; untouched cells -> 0.
 * op_v / op_a [host]: opacity control points. */
int nvol_macrocell_set_tf(const float *lo, const float *hi, int64_t ncell, const double *op_v,
                          const double *op_a, int32_t nop, double density_scale, float *mu,
                          void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NVOL_H */
