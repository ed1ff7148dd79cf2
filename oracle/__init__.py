"""CPU oracle for the ctprev preview data-reduction path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import anything from here, and only as the checker
or the timed CPU reference.  The product package ``paper_2311_15038_b200`` never
imports it (a test asserts that).

* ``oracle.ctp_oracle``  -- numpy restatement of the reference functions
  (``/root/reference/pkg/src/ctprev/{volume,mask,slicemap,render}.py``), each
  citing the file:line it follows.  Pinned against golden vectors produced by
  the reference itself (``tests/golden/make_golden.py``) and against the known
  answers in the reference's own tests.
* ``oracle/ctp_oracle_c.c`` -- the same arithmetic in plain C (gcc, OpenMP over
  z-slabs / image rows) for the raycaster and as the multi-core CPU baseline.
"""
