"""ORACLE — test infrastructure only.

CPU restatement (numpy) of the reference algorithm of the Instant-NVR render
back-end hot path, used as the parity checker of the CUDA product and as the
CPU baseline of bench.py. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package; the product
(paper_2304_03184_b200) never does and has no CPU fallback.

Parity pinning:
  * deform.py (stage 1: k-NN, DQB warps, KnnField, LBS) restates
    capfields/{transforms,edgraph,knnfield,skeleton}.py in the same float64
    evaluation order and is PINNED against golden vectors produced by the real
    reference (tests/golden/make_golden.py, run in the builder container) —
    tests/test_oracle_golden.py.
  * nrf.py (stages 2-4: hash encode, MLPs, march/composite) restates SPEC.md
    (nrf module). The reference has no code and no tests for
    these stages, so their parity is "unpinned" by the reference; they are
    pinned only by SPEC.md's worked examples (SPEC.md:369-371, 386-389,
    409-413), which tests/test_oracle_nrf.py checks.
"""
