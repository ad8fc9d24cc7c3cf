"""CPU oracle for the ACDC hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import anything from this package, and only as a
checker or as the timed CPU baseline.  The product path
(``paper_1511_05946_b200``) never imports it and has no CPU fallback.
"""
