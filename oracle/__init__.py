"""CPU oracle for the AA hot path of arXiv 2110.09667 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg / ``--impl reference`` arm may import anything under ``oracle/``.  The product
path (``paper_2110_09667_b200``, libaa) never imports, links or calls it; the two
share no code.  Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n.

Two layers, plain numpy in fp64:

* O1 ``aa_definition`` — Alg. 1 with gamma the least-squares
  minimiser computed by an unpivoted Householder QR (``numpy.linalg.qr``) of the
  explicit window matrix F_i, then back-substitution.
* O2 ``aa_variant`` — the same driver, gamma from the paper's incremental QR:
  QRAdd_MGS / _ICWY / _CGS2 / _DCGS2 (Algs. 3-6), Givens QRDelete
  (P:111), the ICWY correction-matrix rebuild after a
  delete, and the LSP solve (Alg. 2), with a ledger that
  counts global reductions by phase.

Pins (tests/test_oracle_*.py): AA == GMRES on linear G, exact-rational
normal equations, Householder QR equivalence, the sync-count formulas
(P:536-540), the loss-of-orthogonality classes, and the
SPEC worked examples in tests/golden/.  Parity status of each function is
listed in DESIGN.md §"Oracle pins"; the only "parity unpinned" items are the
paper's iteration counts at paper scale and DCGS-2-inside-AA trajectories,
which the paper itself does not fix.
"""
from .qr import (EPS, Ledger, QRState, Reducer, back_substitution,  # noqa: F401
                 forward_substitution_unit_lower, icwy_rebuild_T, icwy_update_T_small,
                 loss_of_orthogonality,
                 qradd, qrdelete_givens, lsp_solve, VARIANTS)
from .aa import aa_definition, aa_variant, AAResult  # noqa: F401
