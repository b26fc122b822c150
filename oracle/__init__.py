"""Checker-side package: the CPU restatement of the reference semantics and the
reference's own emitted CPU path.

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2509_25605_b200) never imports, loads or calls anything here.
"""
