"""The graphed PPO learner's minibatch update without autograd (SURVEY.md
8(f) f1; the learner is not on the env-step boundary).

``ppo._train_graphed`` with ``PPOConfig.manual_backward`` (the default) runs
each minibatch of the actor-critic update through this module instead of
autocast + autograd + ``clip_grad_norm_`` + fused ``torch.optim.Adam``:

* forward in bf16 on cuBLAS over weights that live as one flat bf16 buffer:
  the first layer and the heads as ``addmm`` (bias in the GEMM epilogue),
  the actor's and critic's hidden layers as one batched GEMM per depth
  followed by a bias + tanh kernel (``grp_bias_tanh``);
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
    gradient in one call (``self.G``).  In the flat buffer the actor's and the
    critic's k-th hidden weights (and biases) sit next to each other, so each
    pair is one [2, L, L] (or [2, L]) tensor: the two hidden stacks run as
    batched GEMMs, two entries per launch.
    """

    def __init__(self, model, n_actions: int, rows: int, device, betas=(0.9, 0.999), eps: float = 1e-5):
        import torch
        import torch.nn as nn
        self.torch = torch
        self.model = model
        self.n_actions = int(n_actions)
        self.rows = int(rows)
        self.betas, self.eps = betas, float(eps)
        self.L = L = model.layer
        self.first = model.first
        self.actor = [m for m in model.actor if isinstance(m, nn.Linear)]
        self.critic = [m for m in model.critic if isinstance(m, nn.Linear)]
        self.a_pad = self.actor[-1].out_features
        if self.a_pad % 8 or self.a_pad < self.n_actions:
            raise ValueError(f"the action head must have a multiple of 8 outputs >= {n_actions}, got {self.a_pad}")
        if len(self.actor) != len(self.critic) or any(
                a.weight.shape != (L, L) or c.weight.shape != (L, L) for a, c in zip(self.actor[:-1], self.critic[:-1])):
            raise ValueError("the actor and critic need the same [L, L] hidden stacks")
        if L % 8:
            raise ValueError("layer size must be a multiple of 8")
        self.n_hidden = len(self.actor) - 1
        # flat layout: first layer, then per hidden layer (actor w, critic w,
        # actor b, critic b), then the two heads
        order = [self.first.weight, self.first.bias]
        for a, c in zip(self.actor[:-1], self.critic[:-1]):
            order += [a.weight, c.weight, a.bias, c.bias]
        order += [self.actor[-1].weight, self.actor[-1].bias, self.critic[-1].weight, self.critic[-1].bias]
        params = list(model.parameters())
        assert len(order) == len(params) and {id(p) for p in order} == {id(p) for p in params}
        off, n = {}, 0
        for p in order:
            off[id(p)] = n
            n += (p.numel() + ALIGN - 1) // ALIGN * ALIGN
        f32 = dict(dtype=torch.float32, device=device)
        self.n = n
        self.P = torch.zeros(n, **f32)
        self.G = torch.zeros(n, **f32)
        self.M = torch.zeros(n, **f32)
        self.V = torch.zeros(n, **f32)
        self.Pb = torch.zeros(n, dtype=torch.bfloat16, device=device)
        with torch.no_grad():
            for p in params:
                o, k = off[id(p)], p.numel()
                self.P[o:o + k].copy_(p.detach().reshape(-1))
                p.data = self.P[o:o + k].view_as(p)
                p.grad = self.G[o:o + k].view_as(p)
            self.Pb.copy_(self.P)
        self.params = params   # module order
        self._w = {id(p): self.Pb[off[id(p)]:off[id(p)] + p.numel()].view_as(p) for p in params}
        self._g = {id(p): p.grad for p in params}

        def pair(buf, a, shape):   # the [2, ...] view starting at the actor entry
            o = off[id(a)]
            return buf[o:o + 2 * a.numel()].view(2, *shape)
        self.hw = [pair(self.Pb, a.weight, (L, L)) for a in self.actor[:-1]]      # bf16 [2, L, L]
        self.hb = [pair(self.Pb, a.bias, (L,)) for a in self.actor[:-1]]          # bf16 [2, L]
        self.hgw = [pair(self.G, a.weight, (L, L)) for a in self.actor[:-1]]      # fp32 [2, L, L]
        self.hgb = [pair(self.G, a.bias, (L,)) for a in self.actor[:-1]]          # fp32 [2, L]
        self.step_t = torch.zeros(1, **f32)
        self.adam_work = torch.zeros(4 + SQ_CTAS, **f32)
        self.adam_ctr = torch.zeros(1, dtype=torch.int32, device=device)
        # activations and gradients of one minibatch
        bf = dict(dtype=torch.bfloat16, device=device)
        R = self.rows
        self.acts = self.make_acts(R)
        self.h0, self.h0_pair, self.hs = self.acts.h0, self.acts.h0_pair, self.acts.hs
        self.logits, self.value = self.acts.logits, self.acts.value
        self.dlogits = torch.empty((R, self.a_pad), **bf)
        self.dvalue = torch.empty_like(self.value)
        self.dy = torch.empty((2, R, L), **bf)
        self.dz = torch.empty((2, R, L), **bf)
        self.dz0 = torch.empty((R, 2 * L), **bf)
        self.bg_work = torch.zeros(2 * ROW_CHUNKS * max(2 * L, self.a_pad), **f32)
        self.bg_ctr = torch.zeros(2 * ((2 * L + 63) // 64 + 1), dtype=torch.int32, device=device)

    def make_acts(self, rows: int):
        """Activation buffers of a forward over `rows` rows (the minibatch's
        are self.acts; the rollout keeps its own set)."""
        import types
        torch = self.torch
        bf = dict(dtype=torch.bfloat16, device=self.P.device)
        L = self.L
        a = types.SimpleNamespace(rows=rows)
        a.h0 = torch.empty((rows, 2 * L), **bf)
        a.h0_pair = a.h0.view(rows, 2, L).transpose(0, 1)   # [2, rows, L] view: actor / critic halves
        a.hs = [torch.empty((2, rows, L), **bf) for _ in range(self.n_hidden)]
        a.logits = torch.empty((rows, self.a_pad), **bf)
        a.value = torch.empty((rows, self.critic[-1].out_features), **bf)
        return a

    # --- views -------------------------------------------------------------
    def w(self, lin):
        """bf16 (weight, bias) of a Linear: views of the flat bf16 buffer."""
        return self._w[id(lin.weight)], self._w[id(lin.bias)]

    def grads(self, lin):
        return self._g[id(lin.weight)], self._g[id(lin.bias)]

    def bf16_weights(self):
        """bf16 views of every parameter, module order (the rollout's weights)."""
        return [self._w[id(p)] for p in self.params]

    def _stream(self):
        return self.torch.cuda.current_stream().cuda_stream

    # --- forward -------------------------------------------------------------
    def forward(self, x, acts=None):
        """x: [rows, obs_pad] bf16 -> (logits [rows, a_pad], value [rows, 1])
        bf16, in `acts` (make_acts; default the minibatch's buffers)."""
        torch = self.torch
        a = acts or self.acts
        w, b = self.w(self.first)
        torch.addmm(b, x, w.t(), out=a.h0).tanh_()
        inp = a.h0_pair
        for k in range(self.n_hidden):   # actor and critic layer k: one batched GEMM, then bias + tanh
            torch.bmm(inp, self.hw[k].transpose(1, 2), out=a.hs[k])
            _check(lib().grp_bias_tanh(a.hs[k].data_ptr(), self.hb[k].data_ptr(), 2, a.rows, self.L,
                                       self._stream()), "grp_bias_tanh")
            inp = a.hs[k]
        w, b = self.w(self.actor[-1])
        torch.addmm(b, inp[0], w.t(), out=a.logits)
        w, b = self.w(self.critic[-1])
        torch.addmm(b, inp[1], w.t(), out=a.value)
        return a.logits, a.value

    # --- backward --------------------------------------------------------------
    def _bias_grad(self, y, dy_a, dy_b, split, cols, dz, db, batch=1):
        """grp_bias_grad over [rows, cols] operands (batch 1) or [2, rows,
        cols] ones (the actor / critic pair, one source)."""
        ld = lambda t: t.stride(-2) if t is not None else 0
        bs = lambda t: t.stride(0) if (t is not None and batch > 1) else 0
        p = lambda t: t.data_ptr() if t is not None else None
        _check(lib().grp_bias_grad(p(y), ld(y), p(dy_a), ld(dy_a), p(dy_b), ld(dy_b), split, self.rows, cols, p(dz),
                                   db.data_ptr(), self.bg_work.data_ptr(), ROW_CHUNKS, self.bg_ctr.data_ptr(),
                                   batch, bs(y), bs(dy_a), bs(dz), self._stream()), "grp_bias_grad")

    def backward(self, x):
        """Gradients of the loss whose d/d logits and d/d value are in
        self.dlogits / self.dvalue (grp_ppo_loss_bf16) into self.G."""
        torch = self.torch
        L = self.L
        last = self.hs[-1] if self.n_hidden else self.h0_pair
        # the heads (no activation): dz = the loss gradient
        for lin, dout, e in ((self.actor[-1], self.dlogits, 0), (self.critic[-1], self.dvalue, 1)):
            gw, gb = self.grads(lin)
            self._bias_grad(None, dout, None, dout.shape[1], dout.shape[1], None, gb)
            torch.mm(dout.t(), last[e], out_dtype=torch.float32, out=gw)
            torch.mm(dout, self.w(lin)[0], out=self.dy[e])
        # hidden layers, actor and critic batched
        for k in range(self.n_hidden - 1, -1, -1):
            inp = self.hs[k - 1] if k > 0 else self.h0_pair
            self._bias_grad(self.hs[k], self.dy, None, L, L, self.dz, self.hgb[k], batch=2)
            torch.bmm(self.dz.transpose(1, 2), inp, out_dtype=torch.float32, out=self.hgw[k])
            torch.bmm(self.dz, self.hw[k], out=self.dy)
        gw, gb = self.grads(self.first)
        self._bias_grad(self.h0, self.dy[0], self.dy[1], L, 2 * L, self.dz0, gb)
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
            None if index is None else index.data_ptr(), self._stream()),
            f"grp_ppo_loss_bf16 (n_actions {self.n_actions})")

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
