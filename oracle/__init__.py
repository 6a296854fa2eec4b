"""GIST CPU oracle -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, FP64 (numpy/scipy) implementation of what the
GIST hot path computes, written from /root/reference/PAPER.md (arXiv 2102.10424).
It shares no code with the CUDA product path (`paper_2102_10424_b200/`), and the
product never imports it.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.

Citations use `PAPER.md:<line>` plus the section/equation they fall in.
Readings where the paper is silent are numbered R1..R18 and listed in DESIGN.md
(they follow SURVEY.md section 8(c)).

Parity status per function: every public function is pinned by a `-m "not gpu"`
test in tests/test_oracle_*.py except `eval_full` accuracy against real data
(parity unpinned: synthetic labels only).
"""
from .gist_oracle import *  # noqa: F401,F403
