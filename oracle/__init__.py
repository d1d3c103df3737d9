"""CPU oracle for the PipeGCN training step (arXiv 2203.10428) -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything in this package.  The
product path (`paper_2203_10428_b200/`) never imports it; the two share no code.

Plain, slow, obviously-correct NumPy/SciPy in float64, following the paper:

* `hashmask`  -- the dropout mask definition (reading R5; App. F)
* `partition` -- Alg. 1 lines 1-5: V_i, B_i, S_{i,j}, S_{j,i}, P_i
* `sage`      -- O1: full-graph GraphSAGE-mean (Eq. 1-3; App. A.1
                 PAPER.md:637-657), loss and its gradient, SGD (Alg. 1 l.32) and Adam (Table 3)
* `pipegcn`   -- O2 vanilla partition-parallel training (Fig. 1(a)) and
                 O3 PipeGCN (Alg. 1; Eq. 3-4; matrix form
                 PAPER.md:659-677) with the smoothing of Sec. 3.4

Pins (tests/test_oracle_*.py, `-m "not gpu"`): SplitMix64 published vectors, brute-force set
definitions and dense-P brute force on tiny graphs, hand-derived golden values
(tests/golden/), float64 central finite differences, O2 == O1, O3(t=1) == O1 on P_in,
O3 == O2 once eta = 0 halos settle, EMA gamma=0 identity and geometric convergence, the
EMA-F / EMA-G transients against the recursion's closed form at eta = 0,
Adam against torch.optim.Adam.  Readings of ambiguous passages: DESIGN.md "Readings".
Parity unpinned: exact per-step values of O3 in the eta > 0 transient beyond the pins
above, and zero-init EMA-G (R12).
"""
