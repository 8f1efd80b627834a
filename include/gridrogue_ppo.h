/* gridrogue_ppo.h -- the PPO learner's fused minibatch objective (not part of
 * the env-step boundary in gridrogue_b200.h; the reference ships no learner,
 * SPEC.md:16).  Same library: libgridrogue_b200.so.
 *
 * One launch on `stream` computes, for a minibatch of `batch` rows, the
 * clipped PPO surrogate with minibatch-normalised advantages, the clipped
 * value loss and the policy entropy (the purejaxrl objective of PAPER.md's
 * Craftax-1B PPO), and writes the gradients of
 *     loss = pg + vf_coef * vl - ent_coef * entropy
 * with respect to the logits [batch, n_actions] and the values [batch].
 * out[4] (float, device, zeroed by the caller) receives
 * [loss, pg, vl, entropy].  All pointers are device pointers.
 * Returns 0, or -1 for an unsupported n_actions (17 and 43 are built) /
 * batch <= 0, -2 for a CUDA launch error.
 */
#ifndef GRIDROGUE_PPO_H
#define GRIDROGUE_PPO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

int grp_ppo_loss(const float* logits, const float* values, const int64_t* actions, const float* logp_old,
                 const float* advantages, const float* values_old, const float* returns, int32_t batch,
                 int32_t n_actions, float clip_eps, float vf_coef, float ent_coef, float* dlogits,
                 float* dvalues, float* out, void* stream);

/* One rollout step's action sampling, one launch on `stream`: actions ~
 * Categorical(softmax(logits[n, n_actions])) by Gumbel-max with
 * counter-based uniforms keyed by (seed, *counter, t, env, action) -- no
 * generator state, so the call replays inside a CUDA graph; writes the
 * actions to actions_a (and actions_b if not null), log p(action) to logp
 * and values[env * ld_values] to value; when reward_out is not null also
 * copies prev_reward -> reward_out and prev_done (uint8) -> done_out (float).
 * logits / values are bf16 (bf16 != 0) or float32, row strides ld_*.
 * Returns 0, -1 (unsupported n_actions / n <= 0), -2 (launch error). */
int grp_sample_actions(const void* logits, const void* values, int32_t bf16, int32_t n, int32_t n_actions,
                       int64_t ld_logits, int64_t ld_values, uint64_t seed, const unsigned long long* counter,
                       uint32_t t, int64_t* actions_a, int64_t* actions_b, float* logp, float* value,
                       const float* prev_reward, const uint8_t* prev_done, float* reward_out, float* done_out,
                       void* stream);


/* grp_ppo_loss over bf16 logits / values with row strides, the gradients
 * written as bf16 (what the head GEMMs of a bf16 learner consume): d loss /
 * d logits into dlogits[row * ld_dlogits + j] for j < n_actions and zeros for
 * n_actions <= j < n_pad (a head padded to n_pad outputs), d loss / d value
 * into dvalues[row * ld_dvalues].  out[4] as for grp_ppo_loss.  index: null,
 * or int64[batch] -- row i's actions / logp_old / advantages / values_old /
 * returns are entry index[i] of those arrays (the minibatch gather fused).
 * Returns 0, -1 (unsupported n_actions, batch <= 0, n_pad < n_actions), -2. */
int grp_ppo_loss_bf16(const void* logits, int64_t ld_logits, const void* values, int64_t ld_values,
                      const int64_t* actions, const float* logp_old, const float* advantages,
                      const float* values_old, const float* returns, int32_t batch, int32_t n_actions,
                      float clip_eps, float vf_coef, float ent_coef, void* dlogits, int64_t ld_dlogits,
                      int32_t n_pad, void* dvalues, int64_t ld_dvalues, float* out, const int64_t* index,
                      void* stream);

/* One layer of the learner's hand-written backward (bf16 activations /
 * gradients, row-major): with dy[i, j] = dy_a[i * ld_a + j] for j < split and
 * dy_b[i * ld_b + j - split] otherwise,
 *   y != NULL: dz[i * cols + j] = bf16(dy[i, j] * (1 - y[i * ld_y + j]^2))   (tanh backward)
 *   db[j] = sum over rows of dz[i, j] (or of dy when y == NULL), fp32.
 * batch > 1 (split == cols): entry b reads y + b * bs_y, dy_a + b * bs_a, writes
 * dz + b * bs_dz and db + b * cols (the actor's and critic's layers at once).
 * work: float[batch * row_chunks * cols]; counters: unsigned[batch *
 * ceil(cols / 64)], zero before the first call (each call leaves them zero).
 * The sum order is fixed by row_chunks: results are deterministic.
 * 0, -1 (bad arguments), -2. */
int grp_bias_grad(const void* y, int64_t ld_y, const void* dy_a, int64_t ld_a, const void* dy_b, int64_t ld_b,
                  int32_t split, int32_t rows, int32_t cols, void* dz, float* db, float* work,
                  int32_t row_chunks, unsigned* counters, int32_t batch, int64_t bs_y, int64_t bs_a,
                  int64_t bs_dz, void* stream);

/* z[b, i, j] = bf16(tanh(z[b, i, j] + bias[b, j])) in place; z a contiguous
 * bf16 [batch, rows, cols] tensor, bias bf16 [batch, cols]; cols % 8 == 0,
 * both 16-byte aligned.  0, -1 (bad arguments), -2. */
int grp_bias_tanh(void* z, const void* bias, int32_t batch, int32_t rows, int32_t cols, void* stream);

/* torch.nn.utils.clip_grad_norm_(max_norm) of grads * grad_scale, then one
 * torch.optim.Adam step (no weight decay; *lr and *step live on the device,
 * *step is incremented) over n flat fp32 parameters, and params_bf16 = bf16
 * (params) for the next forward.  grads are not modified.  work:
 * float[4 + 296] (work[0..3] = gradient multiplier, step size, sqrt of the
 * second bias correction, pre-clip norm); counter: one unsigned, zero before
 * the first call.  fp32 buffers 16-byte aligned, params_bf16 8-byte aligned.
 * Two launches on `stream`.  0, -1 (bad arguments), -2. */
int grp_clip_adam(float* params, const float* grads, float* exp_avg, float* exp_avg_sq, void* params_bf16,
                  int64_t n, const float* lr, float* step, float beta1, float beta2, float eps, float grad_scale,
                  float max_norm, float* work, unsigned* counter, void* stream);

/* dst[i * ld_dst + j] = bf16(src[i * width + j]) (round to nearest even) for
 * rows i and j < width: a batch's float32 observations into a bf16 rollout
 * buffer with padded rows (ld_dst >= width; vectorised when width and ld_dst
 * are multiples of 4, src 16-byte and dst 8-byte aligned).
 * 0, -1 (bad arguments), -2. */
int grp_rows_to_bf16(const float* src, int64_t rows, int32_t width, void* dst, int64_t ld_dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif
