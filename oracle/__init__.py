"""CPU oracle for the l1-filtering hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithm of /root/reference/pkg/src/
l1pcp for the path the CUDA library accelerates (each function cites the reference
file:line it follows).  It exists to CHECK the product:

  * only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference-arm legs
    may import it;
  * the product package (paper_1108_5359_b200) never imports, calls or links anything here
    and fails loudly when its CUDA library is missing.

Pinning: tests/golden/*.npz hold inputs and outputs of the reference itself (generated in
the build container by tests/golden/make_golden.py, which imports /root/reference), and
tests/test_oracle_golden.py checks this oracle against every one of them.  The Philox
generator restatement (philox_gen.py) is pinned against numpy.random.Philox, a
third-party implementation of Philox4x64-10.
"""
