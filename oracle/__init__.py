"""CPU oracle for the HODLR QR hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product path (``paper_1809_10585_b200``) never
imports it and fails loudly when its CUDA library is missing.

Parity pinned: ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors produced by the reference package itself
(``tests/golden/make_golden.py``, committed outputs in ``tests/golden/``) and
against the reference tests' known-answer examples.
"""
