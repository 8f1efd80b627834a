"""PPO host logic without a GPU: the advantage estimator and the model shapes."""

import numpy as np
import pytest
import torch

from paper_2402_16801_b200.ppo import PPOConfig, gae, make_model


def _gae_loop(r, v, d, last, gamma, lam):
    T, N = r.shape
    adv = np.zeros((T, N))
    for n in range(N):
        running = 0.0
        for t in reversed(range(T)):
            nxt = last[n] if t == T - 1 else v[t + 1, n]
            nonterm = 1.0 - d[t, n]
            delta = r[t, n] + gamma * nxt * nonterm - v[t, n]
            running = delta + gamma * lam * nonterm * running
            adv[t, n] = running
    return adv


def test_gae_matches_plain_loop():
    rng = np.random.default_rng(0)
    T, N = 17, 5
    r = rng.normal(size=(T, N))
    v = rng.normal(size=(T, N))
    d = (rng.random((T, N)) < 0.2).astype(np.float64)
    last = rng.normal(size=N)
    adv, ret = gae(torch.tensor(r), torch.tensor(v), torch.tensor(d), torch.tensor(last), 0.99, 0.8)
    ref = _gae_loop(r, v, d, last, 0.99, 0.8)
    assert np.allclose(adv.numpy(), ref, atol=1e-12)
    assert np.allclose(ret.numpy(), ref + v, atol=1e-12)


def test_model_shapes_and_init():
    m = make_model(8268, 43, 512)
    logits, v = m(torch.zeros(3, 8268))
    assert logits.shape == (3, 43) and v.shape == (3,)
    # policy head initialised near-uniform (orthogonal gain 0.01)
    assert float(m.actor[-1].weight.abs().max()) < 0.05


def test_paper_hyperparameters():
    c = PPOConfig()
    assert (c.n_envs, c.n_steps, c.n_minibatches, c.update_epochs, c.layer_size) == (1024, 64, 8, 4, 512)
    assert (c.lr, c.gamma, c.gae_lambda, c.clip_eps, c.vf_coef, c.ent_coef) == (2e-4, 0.99, 0.8, 0.2, 0.5, 0.01)
