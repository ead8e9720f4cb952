"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Restatements of the reference algorithms on the hot path, used by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
as the checker. Nothing in paper_2602_12029_b200/ imports this package; the
product path fails loudly without its CUDA extension.

  oracle/pool.py   — src/prefillsim/kvstore.py BlockPool (pinned against the
                     reference itself: tests/golden/pool_*.json were produced
                     by running prefillsim.kvstore.BlockPool, see
                     tests/golden/make_golden.py)
  oracle/router.py — src/prefillsim/router.py (pinned by golden routing
                     traces from the reference)
  oracle/model.py  — fp32 Llama restatement of the kernels' semantics (pinned
                     against transformers' LlamaForCausalLM on the same
                     weights, tests/golden/llama_tiny.npz) and a literal
                     TinyLM restatement of frontend/src/model.ts:246-331
                     (parity unpinned at the tfjs boundary: the reference
                     publishes no tensor golden values; its property tests are
                     mirrored instead)
  oracle/rng.py    — splitmix64 / mixSeed / Rng (frontend/src/rng.ts;
                     pinned by the seed-0 vectors of rng.test.ts:5-13 and
                     test_workload.py:12-17)
"""
