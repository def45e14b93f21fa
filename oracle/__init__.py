"""CPU oracle for the MoE-MPMC hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only as
the checker or the timed CPU baseline. The product path
(``paper_2605_11537_b200``) never imports it and has no CPU fallback.

Parity is pinned: ``tests/golden/`` holds vectors produced by running the
reference package itself (``tests/golden/make_golden.py``), and
``tests/test_oracle_golden.py`` checks this restatement against them.
"""
