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

#ifdef __cplusplus
}
#endif
#endif
