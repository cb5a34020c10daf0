"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatements of the reference's migration path, used as the checker by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg.  The product package (paper_2501_06709_b200) never imports this package.

  planner.py          plan_hybrid & co. (migration.py), parity pinned against
                      tests/golden/*.json generated from the reference itself.
  kvmig_oracle.c      the byte path (migrate / allocate / re-prefill) in C;
                      the reference moves no bytes, so the byte layout is frozen
                      by this repo and pinned by identity / known-answer
                      properties and by recorded outputs of vLLM 0.22's
                      swap_blocks (tests/golden/thirdparty_vectors.json); the
                      re-prefill by HF transformers' Llama projections (see the
                      C header and tests/test_oracle_cpu.py).
  kvmig_oracle.py     ctypes wrapper over liboracle_kvmig.so (built by Makefile).
  attention_ref.py    fp32 torch paged-decode reference (checker of kvm_paged_decode),
                      pinned by recorded flashinfer 0.6 decode outputs.
"""
