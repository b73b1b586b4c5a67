"""CPU oracle for the B200 RSS engine — TEST INFRASTRUCTURE ONLY.

A numpy restatement (three parties co-resident, "trio" form) of the
reference `mpc3` package's hot path: AES-CTR PRF streams, the float-limb
ring bilinear engine, the replicated-sharing protocols and the layer
schedule of private inference/training.  Every function cites the reference
file:line it restates (paths relative to /root/reference/pkg/src/mpc3/).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import this package, and only as the checker or
the timed CPU reference.  The product (`paper_2104_10949_b200`) never imports
it; it fails loudly when its CUDA library is missing.

Parity pin: `tests/golden/make_golden.py` runs the real reference (importable
in the build container) and commits its outputs — per-party shares included —
as fixtures under `tests/golden/`; `tests/test_oracle.py` checks this oracle
against them bit-for-bit.
"""
