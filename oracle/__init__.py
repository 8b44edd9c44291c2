"""CPU oracle for the all-pairs hot path -- TEST INFRASTRUCTURE ONLY.

Plain numpy / pure-Python restatements of the reference's algorithms, each
citing the reference file:line it follows.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
this package, and only as the checker or the timed CPU baseline -- never as
the product path (which lives in ``paper_2009_04755_b200`` and fails loudly
without its CUDA library).

Pinning status ("Oracle"):
  * rng / synthetic / scheduler / cv / slot cache: pinned against golden
    vectors generated from the reference itself (tests/golden/make_golden.py)
    and the reference tests' known answers.
  * pce / ncc / gmm: parity UNPINNED by the reference, which contains no
    PRNU, NCC or GMM arithmetic; pinned instead by
    known-answer tests (shift -> peak location, identical items -> NCC = 1,
    same-camera vs different-camera separation) and cross-checks against
    scipy.fft.
"""
