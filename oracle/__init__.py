"""CPU oracle for the Bloch event-stream hot path — TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it.  The product path
(``paper_1305_6861_b200``) never imports, calls or falls back to anything
here; it fails loudly when its CUDA library is missing.

Contents
--------
``bloch_oracle``  float64 numpy restatement of the reference's hot path
                  (``mrsim.engine.precompute_sequence_tables`` /
                  ``compute_block`` and the moment / pulse helpers they call),
                  each function citing the reference file:line it follows.
``cpu_pool``      the reference's multiprocess block dispatch restated
                  (``engine._run_pool``), used as the timed CPU baseline.

Parity pin: the restatement is checked against golden vectors produced by
running the *reference itself* in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.
"""
