"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This module holds NO arithmetic of the method (no MMH, no MH, no reduction,
no transforms).  It only produces:

* the workload table (n, r, m) of BASELINE.json ``configs`` and its seeds;
* the synthetic reconciled key: i.i.d. Bernoulli(0.5) bits (PAPER.md:168,
  "x in X is chosen uniformly at random"), drawn from numpy's Philox4x64-10
  as little-endian 64-bit words truncated to ceil(n/8) bytes, MSB-first bit
  order within each byte;
* structured special keys (all-zero, all-one, alternating, single bits).

Both the oracle (``oracle/``) and the CUDA product path consume these bytes;
neither imports the other.
"""
from .workloads import CONFIGS, PAPER_CONFIGS, PaperWorkload, Workload, get_workload, key_bytes, special_key  # noqa: F401
