"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Restatements of the reference algorithms on the hot path, used by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
as the checker. Nothing in paper_2602_12029_b200/ imports this package; the
product path fails loudly without its CUDA extension.

  oracle/pool.py    src/prefillsim/kvstore.py BlockPool restated (argmin-scan
                    LRU as tests/reference_pool.py). Pinned against the
                    reference itself: tests/golden/pool_streams.json.gz was
                    produced by running prefillsim.kvstore.BlockPool
                    (tests/golden/make_golden.py).
  oracle/model.py   fp32 Llama restatement of the kernels' semantics with the
                    control flow of frontend/src/model.ts:246-412 (pinned
                    against transformers' LlamaForCausalLM on the same weights,
                    tests/golden/llama_tiny.npz); layer_forward() is one layer,
                    used whole-model and weight-streamed per layer by the
                    full-size parity test; bf16_storage=True is its bf16
                    precision model.
  oracle/tinylm.py  literal restatement of the reference TinyLM
                    (frontend/src/model.ts:112-331, rng.ts splitmix64 /
                    Box-Muller init; RNG pinned by rng.test.ts:5-13), with the
                    reference's KV-cache property tests mirrored; the checker of
                    the GPU TinyLM (paper_2602_12029_b200/tinylm.py). Tensor
                    parity is unpinned at the tfjs boundary (no node in the
                    image; the reference publishes no tensor golden values).

The router and workload generator have no separate oracle module: the
product's own router.py / workload.py are compared directly with traces the
reference produced (tests/golden/router_traces.json, workload.json).
"""
