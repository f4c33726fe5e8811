"""CPU oracle for the FlashTTS beam-step hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2509_00195_b200``) never imports it and shares no code
with it; the only common module is ``synth`` (seeded inputs, no method
arithmetic).

What it computes (the plain definition of the result):

* ``select``      -- PRM top-K survivor selection by a full sort
                     (PAPER.md 3.1 P:181 "selects the top-K candidates
                     globally with a static branching factor"; ties to the
                     lower index; ordering ledger C3-C5).
* ``block_table`` -- a sequential paged block-table simulator with a
                     lowest-free-page allocator (heap), refcounts = number of
                     live tables containing a page, eager
                     copy-on-write of partial last pages at fork (ledger C6-C8).
* ``beams``       -- per-beam explicit token lists, deep-copied at fork
                     ("Top-scoring paths are then replicated").
* ``attention``   -- fp64 softmax attention of each beam's query over its own
                     materialised K/V copy (textbook definition, ledger
                     C10/C11), plus the partial-state (m, l, o) merge used to
                     pin the cascade identity.
* ``run``         -- drives a whole configuration through the schedule of
                     ``synth.workload`` and records every fork and sampled
                     attention outputs.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): SPEC worked examples, the
hand-derived C1 trace, brute-force subset enumeration, library
sort and fp64 SDPA cross-checks, closed forms, invariants.
"""
