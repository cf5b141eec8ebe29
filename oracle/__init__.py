"""CPU oracle for the SKP-PME reciprocal path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the CPU baseline,
never as the thing measured or shipped. The product package
``paper_2601_18838_b200`` never imports it.
"""
