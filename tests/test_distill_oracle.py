"""Pins of the distillation oracle (oracle/distill_oracle.py, Eq. 4)
against what the mathematics fixes: finite differences, a closed-form
decomposition, zero-loss special cases, symmetry and monotone descent."""
import numpy as np
import pytest

from oracle import distill_oracle as D


def _rand(seed, d=6, f=5, m=4, N=7, scale=0.5):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, d))
    ex = (rng.standard_normal((m, f, d)) * scale, rng.standard_normal((m, f, d)) * scale,
          rng.standard_normal((m, d, f)) * scale)
    uw = (rng.standard_normal((f, d)) * scale, rng.standard_normal((f, d)) * scale,
          rng.standard_normal((d, f)) * scale)
    return X, ex, uw


def test_group_members_paper_examples():
    """P:149 / Fig. 2: m = 8, k = 2 -> 4 groups; k = 3 -> sizes 3, 3, 2."""
    assert [D.group_members(j, 8, 2) for j in range(4)] == [[0, 1], [2, 3], [4, 5], [6, 7]]
    assert [len(D.group_members(j, 8, 3)) for j in range(3)] == [3, 3, 2]
    assert D.group_members(0, 8, 8) == list(range(8))


def test_expert_ffn_matches_per_row_loop():
    X, ex, _ = _rand(0)
    got = D.expert_ffn(X, ex[0][1], ex[1][1], ex[2][1])
    for t in range(X.shape[0]):     # per-row scalar loop of Wd (silu(Wg x) * Wu x)
        a = [sum(ex[0][1][r, j] * X[t, j] for j in range(X.shape[1])) for r in range(ex[0].shape[1])]
        b = [sum(ex[1][1][r, j] * X[t, j] for j in range(X.shape[1])) for r in range(ex[1].shape[1])]
        h = [a[r] / (1 + np.exp(-a[r])) * b[r] for r in range(len(a))]
        y = [sum(ex[2][1][c, r] * h[r] for r in range(len(h))) for c in range(ex[2].shape[1])]
        assert np.allclose(got[t], y, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_gradient_matches_central_finite_differences(seed):
    X, ex, uw = _rand(seed)
    Ho = D.teacher_outputs(X, ex, [0, 1, 2])
    loss, *g = D.united_grads(X, *uw, Ho)
    rng = np.random.default_rng(seed + 10)
    eps = 1e-6
    for wi in range(3):
        for _ in range(6):
            idx = tuple(rng.integers(0, s) for s in uw[wi].shape)
            wp = [w.copy() for w in uw]
            wm = [w.copy() for w in uw]
            wp[wi][idx] += eps
            wm[wi][idx] -= eps
            fd = (D.group_loss(D.expert_ffn(X, *wp), Ho) - D.group_loss(D.expert_ffn(X, *wm), Ho)) / (2 * eps)
            assert abs(fd - g[wi][idx]) <= 1e-6 * max(1.0, abs(fd))
    assert loss == pytest.approx(D.group_loss(D.expert_ffn(X, *uw), Ho), rel=1e-12)


def test_loss_decomposes_into_bias_and_variance_floor():
    """(1/k) sum_i ||u - h_i||^2 = ||u - mean||^2 + (1/k) sum_i ||mean - h_i||^2 per token:
    the floor is a lower bound reached exactly at the pointwise mean."""
    X, ex, uw = _rand(4)
    Ho = D.teacher_outputs(X, ex, [0, 1, 2, 3])
    Hu = D.expert_ffn(X, *uw)
    mean = sum(Ho) / 4
    lhs = D.group_loss(Hu, Ho)
    bias = ((Hu - mean) ** 2).sum() / X.shape[0]
    assert lhs == pytest.approx(bias + D.variance_floor(Ho), rel=1e-12)
    assert lhs >= D.variance_floor(Ho)
    assert D.group_loss(mean, Ho) == pytest.approx(D.variance_floor(Ho), rel=1e-12)


def test_zero_loss_cases():
    """k = 1 with the united expert a copy of its original: loss 0 and gradient 0;
    k = 2 identical originals, united = copy: loss 0 (SPEC examples, TRIVIAL)."""
    X, ex, _ = _rand(5)
    Ho = D.teacher_outputs(X, ex, [2])
    loss, *g = D.united_grads(X, ex[0][2], ex[1][2], ex[2][2], Ho)
    # zero up to the rounding of a*sigmoid(a) vs a/(1+exp(-a))
    assert loss <= 1e-28 and all(np.abs(gi).max() <= 1e-14 for gi in g)
    same = tuple(np.stack([w[1], w[1]]) for w in ex)
    Ho2 = D.teacher_outputs(X, same, [0, 1])
    assert D.group_loss(D.expert_ffn(X, ex[0][1], ex[1][1], ex[2][1]), Ho2) == 0.0
    assert D.variance_floor(Ho2) <= 1e-28      # (h + h) / 2 rounds back to h up to one ulp


def test_loss_symmetric_in_the_group_members():
    """Eq. 4 is a symmetric sum over the k originals."""
    X, ex, uw = _rand(6)
    Hu = D.expert_ffn(X, *uw)
    a = D.group_loss(Hu, D.teacher_outputs(X, ex, [0, 1, 3]))
    b = D.group_loss(Hu, D.teacher_outputs(X, ex, [3, 0, 1]))
    assert a == pytest.approx(b, rel=1e-14)


def test_gradient_descent_decreases_loss_towards_floor():
    """Small-step GD is monotone and approaches the floor from above; with
    identical originals (floor 0) it drives the loss towards 0 (SPEC example)."""
    X, ex, uw = _rand(7, N=64, d=4, f=4, scale=0.4)
    _, losses = D.distill_group(X, ex, [0, 1], uw, lr=0.05, steps=200)
    assert all(b <= a + 1e-15 for a, b in zip(losses, losses[1:]))
    floor = D.variance_floor(D.teacher_outputs(X, ex, [0, 1]))
    assert losses[-1] >= floor and losses[-1] < 0.5 * losses[0]
    same = tuple(np.stack([w[0], w[0]]) for w in ex)
    _, l2 = D.distill_group(X, same, [0, 1], uw, lr=0.1, steps=2000)
    assert all(b <= a + 1e-15 for a, b in zip(l2, l2[1:]))
    assert l2[-1] < 2e-2 * l2[0]
