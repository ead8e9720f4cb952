"""evaluateSharing on the GPU path (evaluate.py; frontend/src/evaluate.ts:16-50)
vs the fp32 Llama oracle: base cache for the first m = min(ceil(r n), n-1)
positions, the decode module recomputes the tail on top of it, greedy
prediction from its last-position logits. Predictions must agree wherever
the oracle's top-1/top-2 margin exceeds 2e-2 * max|logit| (bf16 path)."""

import numpy as np
import pytest
import torch

LOGIT_RTOL = 2e-2


def test_shared_prefix_length_contract():
    from paper_2602_12029_b200.evaluate import shared_prefix_length
    assert [shared_prefix_length(r, 10) for r in (0, 0.25, 0.5, 1, 0.99)] == [0, 3, 5, 9, 9]
    for bad in (-0.1, 1.5, float("nan")):
        with pytest.raises(ValueError):
            shared_prefix_length(bad, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("ratio", [0.0, 0.3, 0.5, 1.0])
def test_evaluate_sharing_matches_oracle(ratio):
    from oracle.model import LlamaOracle
    from paper_2602_12029_b200.evaluate import SharingEvaluator, evaluate_sharing, shared_prefix_length
    from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights
    cfg = LlamaConfig.tiny()
    base = ModuleWeights(cfg, 3, with_head=False)
    dec = ModuleWeights(cfg, 4)
    torch.cuda.synchronize()
    base_o, dec_o = LlamaOracle(cfg, base.reference_layout()), LlamaOracle(cfg, dec.reference_layout())
    rng = np.random.default_rng(int(ratio * 10))
    n, B = 45, 6
    prompts = [rng.integers(0, cfg.vocab, n).tolist() for _ in range(B)]
    ev = SharingEvaluator(cfg, B, n)
    pred = ev.predictions(dec, base, ratio, prompts)
    m = shared_prefix_length(ratio, n)
    want, flips = [], 0
    for p, got in zip(prompts, pred):
        past = None
        if m > 0:
            past = [(k.to(torch.bfloat16).float(), v.to(torch.bfloat16).float()) for k, v in base_o.prefill(p[:m])]
        lg = dec_o.forward(p[m:], past)[0][-1]
        w = int(torch.argmax(lg))
        want.append(w)
        if int(got) != w:
            top2 = torch.topk(lg, 2).values
            assert float(top2[0] - top2[1]) <= LOGIT_RTOL * float(lg.abs().max()), (got, w)
            flips += 1
    assert flips <= 1
    acc = evaluate_sharing(dec, base, ratio, prompts, want, evaluator=ev)
    assert acc >= (B - flips) / B
