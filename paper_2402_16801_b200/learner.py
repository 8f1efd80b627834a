"""The graphed PPO learner's minibatch update without autograd (SURVEY.md
8(f) f1; the learner is not on the env-step boundary).

``ppo._train_graphed`` with ``PPOConfig.manual_backward`` (the default) runs
each minibatch of the actor-critic update through this module instead of
autocast + autograd + ``clip_grad_norm_`` + fused ``torch.optim.Adam``:

* forward in bf16 on cuBLAS (``addmm`` with the bias in the GEMM epilogue,
  ``tanh_`` in place) over weights that live as one flat bf16 buffer;
* the PPO objective and its logits / value gradients in one kernel
  (``grp_ppo_loss_bf16``), the action head padded to a multiple of 8 outputs
  (43 -> 48: cuBLAS then runs the head GEMMs on its tensor-core kernels
  instead of the unaligned SIMT fallbacks; the pad rows start at zero, their
  gradients are exactly zero, so they stay zero and the softmax never sees
  them);
* the backward written out layer by layer: for each layer one kernel forms the
  tanh backward and the bias gradient (``grp_bias_grad``: a deterministic
  column sum), cuBLAS the weight gradient straight into the fp32 gradient
  buffer (``mm`` with ``out_dtype=float32``) and the input gradient;
* global-norm clipping and Adam over the flat fp32 parameters in two launches
  (``grp_clip_adam``), which also refresh the bf16 copy the next forward and
  the rollout read.

The arithmetic is the autocast learner's (bf16 GEMM inputs and activations,
fp32 accumulation, fp32 master weights and optimizer state); the test
``tests/test_gpu.py::test_manual_learner_matches_autograd`` compares the
gradients with autograd's and the update with torch's clip + Adam.
"""

from __future__ import annotations

from ._lib import lib

ALIGN = 8                 # parameter offsets in elements: 16-byte aligned bf16 and fp32 views
ROW_CHUNKS = 32           # grp_bias_grad row chunks (fixes the summation order)
SQ_CTAS = 296             # grp_clip_adam's partial-sum CTAs (gr_ppo.cu)


def pad_actions(n_actions: int) -> int:
    return (n_actions + 7) // 8 * 8


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc})")


class ManualLearner:
    """Flat parameter / gradient / Adam-state buffers for a FusedActorCritic
    (ppo.make_fused_model) and its minibatch forward + backward + step.

    The module's parameters become views of the flat fp32 buffer (their
    ``.grad`` views of the flat gradient buffer), so ``model(x)`` still
    evaluates the current weights and a multi-GPU all-reduce covers every
    gradient in one call (``self.G``).
    """

    def __init__(self, model, n_actions: int, rows: int, device, betas=(0.9, 0.999), eps: float = 1e-5):
        import torch
        import torch.nn as nn
        self.torch = torch
        self.model = model
        self.n_actions = int(n_actions)
        self.rows = int(rows)
        self.betas, self.eps = betas, float(eps)
        self.L = model.layer
        self.first = model.first
        self.actor = [m for m in model.actor if isinstance(m, nn.Linear)]
        self.critic = [m for m in model.critic if isinstance(m, nn.Linear)]
        self.a_pad = self.actor[-1].out_features
        if self.a_pad % 8 or self.a_pad < self.n_actions:
            raise ValueError(f"the action head must have a multiple of 8 outputs >= {n_actions}, got {self.a_pad}")
        params = list(model.parameters())
        offs, n = [], 0
        for p in params:
            offs.append(n)
            n += (p.numel() + ALIGN - 1) // ALIGN * ALIGN
        f32 = dict(dtype=torch.float32, device=device)
        self.n = n
        self.P = torch.zeros(n, **f32)
        self.G = torch.zeros(n, **f32)
        self.M = torch.zeros(n, **f32)
        self.V = torch.zeros(n, **f32)
        self.Pb = torch.zeros(n, dtype=torch.bfloat16, device=device)
        with torch.no_grad():
            for p, o in zip(params, offs):
                k = p.numel()
                self.P[o:o + k].copy_(p.detach().reshape(-1))
                p.data = self.P[o:o + k].view_as(p)
                p.grad = self.G[o:o + k].view_as(p)
            self.Pb.copy_(self.P)
        self.params = params
        self._w = {id(p): self.Pb[o:o + p.numel()].view_as(p) for p, o in zip(params, offs)}
        self._g = {id(p): p.grad for p in params}
        self.step_t = torch.zeros(1, **f32)
        self.adam_work = torch.zeros(4 + SQ_CTAS, **f32)
        self.adam_ctr = torch.zeros(1, dtype=torch.int32, device=device)
        # activations and gradients of one minibatch
        bf = dict(dtype=torch.bfloat16, device=device)
        R, L = self.rows, self.L
        self.h0 = torch.empty((R, 2 * L), **bf)
        self.ha = [torch.empty((R, L), **bf) for _ in self.actor[:-1]]
        self.hc = [torch.empty((R, L), **bf) for _ in self.critic[:-1]]
        self.logits = torch.empty((R, self.a_pad), **bf)
        self.value = torch.empty((R, self.critic[-1].out_features), **bf)
        self.dlogits = torch.empty((R, self.a_pad), **bf)
        self.dvalue = torch.empty_like(self.value)
        self.dz = torch.empty((R, L), **bf)
        self.dya = torch.empty((R, L), **bf)
        self.dyc = torch.empty((R, L), **bf)
        self.dz0 = torch.empty((R, 2 * L), **bf)
        self.bg_work = torch.zeros(ROW_CHUNKS * max(2 * L, self.a_pad), **f32)
        self.bg_ctr = torch.zeros((2 * L + 63) // 64 + 1, dtype=torch.int32, device=device)

    # --- views -------------------------------------------------------------
    def w(self, lin):
        """bf16 (weight, bias) of a Linear: views of the flat bf16 buffer."""
        return self._w[id(lin.weight)], self._w[id(lin.bias)]

    def grads(self, lin):
        return self._g[id(lin.weight)], self._g[id(lin.bias)]

    def bf16_weights(self):
        """bf16 views of every parameter, module order (the rollout's weights)."""
        return [self._w[id(p)] for p in self.params]

    # --- forward -------------------------------------------------------------
    def forward(self, x):
        """x: [rows, obs_pad] bf16 -> (logits [rows, a_pad], value [rows, 1]) bf16."""
        torch = self.torch
        L = self.L
        w, b = self.w(self.first)
        torch.addmm(b, x, w.t(), out=self.h0).tanh_()
        for lins, hs, inp in ((self.actor, self.ha, self.h0[:, :L]), (self.critic, self.hc, self.h0[:, L:])):
            for lin, h in zip(lins[:-1], hs):
                w, b = self.w(lin)
                torch.addmm(b, inp, w.t(), out=h).tanh_()
                inp = h
            w, b = self.w(lins[-1])
            torch.addmm(b, inp, w.t(), out=self.logits if lins is self.actor else self.value)
        return self.logits, self.value

    # --- backward --------------------------------------------------------------
    def _bias_grad(self, y, dy_a, dy_b, split, cols, dz, db):
        torch = self.torch
        rows = self.rows
        ld = lambda t: t.stride(0) if t is not None else 0
        p = lambda t: t.data_ptr() if t is not None else None
        _check(lib().grp_bias_grad(p(y), ld(y), p(dy_a), ld(dy_a), p(dy_b), ld(dy_b), split, rows, cols, p(dz),
                                   db.data_ptr(), self.bg_work.data_ptr(), ROW_CHUNKS, self.bg_ctr.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream), "grp_bias_grad")

    def _branch_backward(self, lins, hs, inp0, dout, dy_buf):
        """Backward through one head's Linear stack (the last Linear without
        an activation); the gradient of its input (inp0) ends in dy_buf."""
        torch = self.torch
        inputs = [inp0] + hs   # input of lins[k] is inputs[k]
        # the head: dz = dout
        gw, gb = self.grads(lins[-1])
        self._bias_grad(None, dout, None, dout.shape[1], dout.shape[1], None, gb)
        torch.mm(dout.t(), inputs[-1], out_dtype=torch.float32, out=gw)
        torch.mm(dout, self.w(lins[-1])[0], out=dy_buf)
        for k in range(len(lins) - 2, -1, -1):
            gw, gb = self.grads(lins[k])
            self._bias_grad(hs[k], dy_buf, None, self.L, self.L, self.dz, gb)
            torch.mm(self.dz.t(), inputs[k], out_dtype=torch.float32, out=gw)
            torch.mm(self.dz, self.w(lins[k])[0], out=dy_buf)

    def backward(self, x):
        """Gradients of the loss whose d/d logits and d/d value are in
        self.dlogits / self.dvalue (grp_ppo_loss_bf16) into self.G."""
        torch = self.torch
        L = self.L
        self._branch_backward(self.actor, self.ha, self.h0[:, :L], self.dlogits, self.dya)
        self._branch_backward(self.critic, self.hc, self.h0[:, L:], self.dvalue, self.dyc)
        gw, gb = self.grads(self.first)
        self._bias_grad(self.h0, self.dya, self.dyc, L, 2 * L, self.dz0, gb)
        torch.mm(self.dz0.t(), x, out_dtype=torch.float32, out=gw)

    def loss(self, actions, logp_old, adv, v_old, ret, clip_eps, vf_coef, ent_coef, stats, index=None):
        """The PPO objective of the last forward; stats (float[4], zeroed
        here) <- [loss, pg, vl, entropy]; gradients into dlogits / dvalue.
        index (int64[rows], optional): row i's per-sample inputs are entry
        index[i] of the given arrays (the minibatch gather in the kernel)."""
        torch = self.torch
        stats.zero_()
        _check(lib().grp_ppo_loss_bf16(
            self.logits.data_ptr(), self.logits.stride(0), self.value.data_ptr(), self.value.stride(0),
            actions.data_ptr(), logp_old.data_ptr(), adv.data_ptr(), v_old.data_ptr(), ret.data_ptr(), self.rows,
            self.n_actions, float(clip_eps), float(vf_coef), float(ent_coef), self.dlogits.data_ptr(),
            self.dlogits.stride(0), self.a_pad, self.dvalue.data_ptr(), self.dvalue.stride(0), stats.data_ptr(),
            None if index is None else index.data_ptr(), torch.cuda.current_stream().cuda_stream), f"grp_ppo_loss_bf16 (n_actions {self.n_actions})")

    # --- optimizer -------------------------------------------------------------
    def clip_adam(self, lr_t, max_norm: float, grad_scale: float = 1.0):
        """clip_grad_norm_(max_norm) of G * grad_scale, one Adam step on P
        (lr from the device scalar lr_t), Pb <- bf16(P)."""
        torch = self.torch
        b1, b2 = self.betas
        _check(lib().grp_clip_adam(self.P.data_ptr(), self.G.data_ptr(), self.M.data_ptr(), self.V.data_ptr(),
                                   self.Pb.data_ptr(), self.n, lr_t.data_ptr(), self.step_t.data_ptr(), b1, b2,
                                   self.eps, float(grad_scale), float(max_norm), self.adam_work.data_ptr(),
                                   self.adam_ctr.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "grp_clip_adam")
