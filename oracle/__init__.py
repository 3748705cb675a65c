"""CPU oracle for arXiv 2409.04202 (GenModel + GenTree) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import or execute anything under `oracle/`.  The product path
(`paper_2409_04202_b200`, the C-ABI library) never imports it and shares no code with it:
this package is plain, slow, obviously-correct Python (numpy for elementwise fp32 adds,
`fractions.Fraction` for exact costs), written directly from the paper's text.

Citation convention: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n.
Readings of ambiguous/garbled passages are the Q-numbered register in DESIGN.md
(SURVEY.md §8(c)).

Modules
  topology  — tree topology, parse/validate, servers, convergence ratio
  plans     — plan data model, natural RS builders of every Fig. 1 plan type (P:136-145,
              P:446-478), AG = reversed RS, ACPS, tag verifier
  genmodel  — GenModel exact (Fraction) and fixed-order float64 evaluation,
              Table 1/2 closed forms, optimality bounds (Thm 1)
  gentree   — Algorithm 1 and 2, sub-plan composition
  simulate  — step-by-step data simulation in the plan's exact summation order (fp32/bf16)
  theorems  — brute-force enumeration of reduce trees: Eq. 12-14, Theorems 1 and 2
  fit       — §3.4 fitting via NNLS with a w_t scan; Eq. 6 fan-in fit

Parity status: every function is pinned by a `-m "not gpu"` test (tests/test_oracle_*.py)
except where its docstring says "parity unpinned".
"""
