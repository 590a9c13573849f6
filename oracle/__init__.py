"""CPU ORACLE for the MMH-MH privacy-amplification hash (arXiv 2105.13678).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``include/``,
``paper_2105_13678_b200/``) may import, call, link or execute anything under
``oracle/``.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it.  It shares no code, no
headers, no tables and no constant generators with the CUDA path; the only
module both sides consume is ``synth/`` (seeded input bytes, no arithmetic).

Contents
--------
``oracle.mersenne``   Mersenne-prime field Z_p, p = 2^gamma - 1 (PAPER.md:129-132,
                      SPEC.md:25-103): exponent table, fold reduction, field ops.
``oracle.hashes``     MMH (Eq. 1-2), MH (Eq. 3-4),
                      Algorithm 1 in the paper's own shape
                      (gamma-bit blocks with reload) and in the r-bit-block shape
                      the B200 library computes (readings A1-A10 of DESIGN.md).
``oracle.seeds``      hash-key expansion a_i, b, c from a 64-bit seed (reading A7).
``oracle.toeplitz``   Toeplitz-hashing PA over GF(2), the NEXT-4 comparator,
                      readings A14 (index convention) and A15 (seeded diagonal).
``oracle.params``     NEXT-1 parameter derivation (security coefficient, block count,
                      gamma selection), exact rational scans.
``oracle.security``   brute-force universality / composition checks
                      (Appendix A, Lemma 2).
``oracle.schoolbook`` plain C schoolbook big-integer version of the same pipeline
                      (``oracle/schoolbook.c``), for larger sizes and the CPU
                      baseline timing.

Parity status: every function is pinned by ``tests/test_oracle_*.py``
(``-m "not gpu"``); see DESIGN.md "Oracle pins".  No function is
"parity unpinned".
"""
