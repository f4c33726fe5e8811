"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no attention, selection, fork
or allocation logic). It only produces inputs:

* ``rng``      -- a counter-based generator (lowbias32 hash) evaluated with
                  integer torch ops, so it gives bit-identical bf16 values on
                  CPU (oracle side) and on CUDA (device-side input staging).
* ``workload`` -- the BASELINE.json configurations C1..C5 (shapes, step
                  lengths, score streams) and the per-iteration schedule
                  (which beams are active, which requests end a step).

Both ``oracle/`` and the product path may import it; neither imports the
other.
"""
from . import rng, workload  # noqa: F401
