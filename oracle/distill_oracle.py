"""CPU fp64 oracle for united-expert distillation (BrownoutServe §4.2, Eq. 4).

TEST INFRASTRUCTURE ONLY.  Only ``tests/`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this module; the product
path (``paper_2507_17133_b200``) shares no code with it.

Paper (§4.2 "United Expert Model"): the m experts of a layer are cut
into ceil(m/k) groups; for group j the k original experts are the
teacher and the united expert UE_j the student; the training target is
the originals' hidden states and the loss is Eq. 4:

    L^j_MSE = (1/k) * sum_{i=0}^{k-1} || H^j_u - H^{j*k+i}_o ||^2

Readings (D21-D24):
  D21  Eq. 4 has no token dimension: the squared norm is summed over the
       hidden dimension and AVERAGED over the N training tokens (SPEC's
       decision); k is the group's actual size (ragged last group, D15).
  D22  Optimiser: plain gradient descent with a fixed learning rate (the paper
       names none); fp32 master weights on the GPU, fp64 here.
  D23  Training tokens: synthetic N(0, 1) rows with the bias channel (the
       paper's teacher inputs come from real traffic); the same N tokens train
       every group (each teacher sees every token).
  D24  Expert form: the SwiGLU FFN of D13, so H(x) = Wd (silu(Wg x) * (Wu x)).

The gradient is the plain derivative of L^j with respect to the united
weights, written out by the chain rule in the order of the forward pass (no
reformulation): it is pinned against central finite differences.
"""
from __future__ import annotations

import numpy as np


def group_members(j: int, m: int, way: int) -> list:
    """Experts of group j: [j*k, min((j+1)*k, m)) (ragged last group, D15)."""
    return list(range(j * way, min((j + 1) * way, m)))


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def expert_ffn(X, Wg, Wu, Wd):
    """H(x) = Wd (silu(Wg x) * (Wu x)) for every row of X [N, d] (D24)."""
    X, Wg, Wu, Wd = _f64(X), _f64(Wg), _f64(Wu), _f64(Wd)
    a = X @ Wg.T
    b = X @ Wu.T
    h = a / (1.0 + np.exp(-a)) * b
    return h @ Wd.T


def teacher_outputs(X, experts, members):
    """H_o^{j*k+i}: the hidden states of each original expert of the group."""
    Wg, Wu, Wd = experts
    return [expert_ffn(X, Wg[e], Wu[e], Wd[e]) for e in members]


def group_loss(Hu, Ho):
    """Eq. 4 with the per-token mean of D21:
    (1/N) sum_t (1/k) sum_i ||Hu_t - Ho^i_t||^2."""
    Hu = _f64(Hu)
    k = len(Ho)
    N = Hu.shape[0]
    tot = 0.0
    for Hi in Ho:
        tot += float(((Hu - _f64(Hi)) ** 2).sum())
    return tot / k / N


def variance_floor(Ho):
    """The part of Eq. 4 no student can remove: (1/N)(1/k) sum_t sum_i ||mean_i Ho - Ho^i||^2."""
    k = len(Ho)
    mean = sum(_f64(H) for H in Ho) / k
    return group_loss(mean, Ho)


def united_grads(X, UWg, UWu, UWd, Ho):
    """dL^j / d(UWg, UWu, UWd) by the chain rule through the forward pass.

    forward:  a = X UWg^T, b = X UWu^T, s = sigmoid(a), h = a s b, y = h UWd^T
    loss:     L = (1/N)(1/k) sum_i sum_t ||y_t - Ho^i_t||^2
    backward: dL/dy   = (2/(N k)) sum_i (y - Ho^i)
              dL/dUWd = (dL/dy)^T h
              dL/dh   = (dL/dy) UWd
              dL/da   = dL/dh * b * (s + a s (1 - s))      (d silu / da)
              dL/db   = dL/dh * a s
              dL/dUWg = (dL/da)^T X,  dL/dUWu = (dL/db)^T X
    Returns (loss, dUWg, dUWu, dUWd)."""
    X, UWg, UWu, UWd = _f64(X), _f64(UWg), _f64(UWu), _f64(UWd)
    N = X.shape[0]
    k = len(Ho)
    a = X @ UWg.T
    b = X @ UWu.T
    s = 1.0 / (1.0 + np.exp(-a))
    h = a * s * b
    y = h @ UWd.T
    loss = group_loss(y, Ho)
    dy = np.zeros_like(y)
    for Hi in Ho:
        dy += y - _f64(Hi)
    dy *= 2.0 / (N * k)
    dUWd = dy.T @ h
    dh = dy @ UWd
    da = dh * b * (s + a * s * (1.0 - s))
    db = dh * a * s
    dUWg = da.T @ X
    dUWu = db.T @ X
    return loss, dUWg, dUWu, dUWd


def sgd_step(weights, grads, lr):
    """Plain gradient descent (D22): W <- W - lr dL/dW."""
    return tuple(_f64(w) - lr * _f64(g) for w, g in zip(weights, grads))


def distill_group(X, experts, members, init, lr, steps):
    """Train one united expert for `steps` full-batch GD steps.
    Returns (weights, losses) where losses[s] is Eq. 4 before step s and
    losses[steps] after the last one."""
    Ho = teacher_outputs(X, experts, members)
    W = tuple(_f64(w) for w in init)
    losses = []
    for _ in range(steps):
        loss, *g = united_grads(X, *W, Ho)
        losses.append(loss)
        W = sgd_step(W, g, lr)
    losses.append(group_loss(expert_ffn(X, *W), Ho))
    return W, losses
