"""CPU parity oracle for the alternating-NNLS hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` arm may import this package.  The product package
``paper_1506_08938_b200`` never imports it: there is no CPU fallback.

* ``nnls_oracle.c``  -- C restatement of ``nmfkit/kernels.py`` (bit-exact).
* ``nmf_oracle.py``  -- numpy restatement of ``nmfkit/{nmf,parallel,nqp,matrix}.py``.
* ``generators.py``  -- pinned synthetic inputs for BASELINE.json configs 1-5.

Parity is pinned: ``tests/golden/make_golden.py`` ran the reference itself
(imported from /root/reference in the build container) and committed its
outputs under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks the
oracle against them.
"""
