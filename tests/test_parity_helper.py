"""The element-wise parity helper (tests/parity.py) on a bf16-faithful CPU emulation of the GPU path:
it must accept the honest result and reject a corrupted tile, row or element (CPU only)."""
import numpy as np
import pytest
import torch

import tl_inputs as TI
from oracle import tl_oracle as O
from parity import parity_report

W, M, H, I = 4, 512, 512, 1024


def _bf(x):
    return x.to(torch.bfloat16).to(torch.float32)


@pytest.fixture(scope="module")
def case():
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=3)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    ref = np.concatenate(O.mlp_forward([TI.to_f64(t) for t in Xs], [TI.to_f64(t) for t in W1s],
                                       [TI.to_f64(t) for t in W2s], TI.ACT_SILU_MUL), 0)
    # the GPU path's arithmetic (DESIGN R8): fp32 accumulation, Z rounded to bf16, partials to bf16,
    # own partial fp32 + slots in ascending rank order, one final bf16 rounding
    x = torch.cat(Xs).float()
    il = I // W
    parts = []
    for r in range(W):
        y = x @ W1s[r].float().T
        z = _bf(torch.nn.functional.silu(y[:, :il]) * y[:, il:])
        parts.append(z @ W2s[r].float().T)
    out = torch.zeros(M, H)
    mr = M // W
    for o in range(W):
        acc = parts[o][o * mr:(o + 1) * mr].clone()
        for s in range(W):
            if s != o:
                acc += _bf(parts[s][o * mr:(o + 1) * mr])
        out[o * mr:(o + 1) * mr] = _bf(acc)
    return out.double().numpy(), ref


def test_honest_result_passes(case):
    got, ref = case
    rep = parity_report(got, ref)
    assert rep["ok"], rep
    assert 1e-3 < rep["global"] < 4e-3        # the bf16 budget of SURVEY §8(c)


@pytest.mark.parametrize("scale", [1.01, 0.99])
def test_one_corrupted_tile_fails(case, scale):
    got, ref = case
    bad = got.copy()
    bad[128:256, 256:512] *= scale           # one 128 x 256 CTA tile off by 1 %
    rep = parity_report(bad, ref)
    assert not rep["ok"] and rep["worst_tile"] == (128, 256)
    assert rep["global"] < 5e-3               # ... which the global norm alone would have accepted


def test_one_bad_element_fails(case):
    got, ref = case
    bad = got.copy()
    bad[300, 17] = ref[300, 17] + 0.1 * np.sqrt((ref[300] ** 2).mean())
    rep = parity_report(bad, ref)
    assert not rep["ok"] and rep["elements_over_bound"] == 1 and rep["first_over"][:2] == (300, 17)


def test_swapped_rows_fail(case):
    got, ref = case
    bad = got.copy()
    bad[[5, 6]] = bad[[6, 5]]
    assert not parity_report(bad, ref)["ok"]
