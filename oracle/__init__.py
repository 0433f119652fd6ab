"""CPU oracle for the plane-wave FGT hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (/root/reference/pkg/src/fgt and the
Alg 2 contract of /root/reference/SPEC.md:361-444), written from the reference's
behaviour, not copied from it.  Each function cites the reference file:line it
follows.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its
`cpu_baseline` leg and `--impl reference`) may import this package, and only as the
checker / CPU baseline -- never as the product path.

Pinning: `tests/golden/make_golden.py` runs the real reference package (importable
from /root/reference/pkg/src in the build container) and commits its outputs as
fixtures; `tests/test_oracle_golden.py` checks this oracle against them (tree box
sets and leaf lists bit-exact, kernels and NUFFTs to roundoff, Table 1/2 parameters
exactly).  The end-to-end driver (the reference ships none) is additionally pinned
against exact O(NM) sums at <= 10 eps.
"""
