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

#ifdef __cplusplus
}
#endif
#endif
