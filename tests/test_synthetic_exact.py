"""CPU pin of the exactly-representable router inputs the GPU routing-parity
tests rely on (synthetic.make_exact_router_inputs): Eq. 8 computed in
fp32 in three different summation orders equals the fp64 product bit for bit,
so a GPU router that accumulates in fp32 in any order must reproduce the fp64
logits exactly (no clear-margin filter needed)."""
import numpy as np
import pytest
import torch

import synthetic as S


@pytest.mark.parametrize("ties", [True, False])
@pytest.mark.parametrize("cfg", [S.CONFIGS["tiny"], S.with_(S.CONFIGS["qwen3_30b_a3b_prefill"], T=64),
                                 S.with_(S.CONFIGS["mixtral_prefill"], T=32)], ids=lambda c: c.name)
def test_exact_inputs_sum_exactly_in_fp32(cfg, ties):
    x, Wr = S.make_exact_router_inputs(cfg, ties=ties)
    assert S.exactness_bound(x, Wr) < 2.0 ** 11
    ref = x.double() @ Wr.double().T
    xf, wf = x.float().numpy(), Wr.float().numpy()
    fwd = np.zeros(ref.shape, dtype=np.float32)
    for j in range(cfg.d):                      # sequential fp32 accumulation, ascending k
        fwd += np.outer(xf[:, j], wf[:, j]).astype(np.float32)
    bwd = np.zeros(ref.shape, dtype=np.float32)
    for j in reversed(range(cfg.d)):            # descending k
        bwd += np.outer(xf[:, j], wf[:, j]).astype(np.float32)
    pair = (xf[:, None, :] * wf[None, :, :]).astype(np.float32)
    while pair.shape[-1] > 1:                   # pairwise tree
        if pair.shape[-1] % 2:
            pair = np.concatenate([pair, np.zeros(pair.shape[:-1] + (1,), np.float32)], -1)
        pair = (pair[..., 0::2] + pair[..., 1::2]).astype(np.float32)
    for got in (fwd, bwd, pair[..., 0]):
        assert np.array_equal(got.astype(np.float64), ref.numpy())
    if ties:   # exact ties between experts are common
        L = ref.numpy()
        assert any(len(set(row)) < len(row) for row in L)


def test_exact_inputs_are_seeded():
    c = S.CONFIGS["tiny"]
    a = S.make_exact_router_inputs(c)
    b = S.make_exact_router_inputs(c)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
