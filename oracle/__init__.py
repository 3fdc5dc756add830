"""ORACLE package — CPU restatements of the reference's hot path.

TEST INFRASTRUCTURE ONLY: importable from ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs, as the checker.
The product package (``paper_2310_18481_b200``) never imports it.
"""
